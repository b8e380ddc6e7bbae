// recurrent.cu -- recurrent (decode) path: run_recurrent (recurrent.cpp:65-115)
// with the memory state carried in place (RecurrentOptions::initial_state,
// recurrent.hpp:23-27), folding step_exp / step_sig (recurrent.cpp:9-63):
//   exp: m' = max(logsig(f) + m, i);  fg = exp(logsig(f) + m - m');  ig = exp(i - m')
//   sig: fg = sigmoid(f);             ig = sigmoid(i)
//   C' = fg C + ig k v^T ;  n' = fg n + ig k (exp)
//   h  = C'^T q / sqrt(d) / max(|n'.q / sqrt(d)|, exp(-m'))   (exp; sig: no divide)
//
// Decode is HBM-bound on the state (C is dqk x dhv fp32 per head): one CTA
// owns a 64-column slice of one head's C in registers (256 threads: 64
// columns x 4 row groups of dqk/4 rows), so C is read once and written once
// per launch however many steps T the launch folds. The step inputs are
// staged in shared memory 16 steps at a time; h is reduced over the 4 row
// groups. n and q.n (exp) are carried redundantly by every column slice of a
// head (thread t < dqk owns n[t]).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>

#include "kernels.h"
#include "stab.cuh"

namespace tfla_k {
namespace {

constexpr int kCols = 64;
constexpr int kThreads = 256;

__device__ __forceinline__ float logsigf(float x) { return fminf(x, 0.f) - log1pf(expf(-fabsf(x))); }
__device__ __forceinline__ float sigmf(float x) {
    if (x >= 0.f) return 1.f / (1.f + expf(-x));
    const float e = expf(x);
    return e / (1.f + e);
}

// Step-input staging: up to kTB steps' q / k (fp32, all dqk), this slice's v
// columns and the gate pre-activations are loaded into shared memory in one
// pass, so a step costs shared-memory reads and one barrier (the h partials
// and the q.n warp sums are double-buffered by step parity).
constexpr int kTB = 16;

// kCluster: the column-slice CTAs of a head form a cluster (dhv / 64 <= 8);
// every CTA reads the initial n / m, arrives on the cluster barrier, and slice
// 0 writes the final n / m in place only after the barrier's wait -- no CTA can
// observe another's update and no copy of n / m is needed. Otherwise the host
// passes launch-private copies (n_in / m_in).
template <int R, bool kCluster>  // rows of C per thread = dqk / 4
__global__ void __launch_bounds__(kThreads, 2) recurrent_kernel(RecurrentArgs a) {
    constexpr int dqk = 4 * R;
    __shared__ __align__(16) float qs[kTB][dqk], ks[kTB][dqk], vs[kTB][kCols], gi[kTB], gf[kTB], gm[kTB];
    __shared__ float red[2][4][kCols], nqw[2][8];
    const int dhv = a.dhv, T = a.T;
    const int bh = blockIdx.y, x0 = blockIdx.x * kCols;
    const int t = threadIdx.x, xl = t & (kCols - 1), pg = t >> 6;
    const bool is_exp = a.variant == 0;
    const float rs = rsqrtf(static_cast<float>(dqk));

    float c[R];
    float* C = a.c_state + static_cast<size_t>(bh) * dqk * dhv + x0 + xl;
#pragma unroll
    for (int r = 0; r < R; ++r) c[r] = C[static_cast<size_t>(pg * R + r) * dhv];
    const float* n_src = kCluster ? a.n_state : a.n_in;
    const float* m_src = kCluster ? a.m_state : a.m_in;
    float n_reg = (is_exp && t < dqk && n_src) ? n_src[static_cast<size_t>(bh) * dqk + t] : 0.f;  // thread t owns n[t]
    float m = (is_exp && m_src) ? m_src[bh] : 0.f;
    if (kCluster) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");  // n / m read

    StabLocal sl;
    for (int s0 = 0; s0 < T; s0 += kTB) {
        const int nb = min(kTB, T - s0);
        const size_t row0 = static_cast<size_t>(bh) * T + s0;
        if (s0 > 0) __syncthreads();  // the previous block's steps are done with the staging
        // 16-B loads, all issued before any use (one latency per block)
        constexpr int kQ4 = dqk / 8;                                   // uint4 per q / k row
        constexpr int kLd = (kTB * kQ4 + kThreads - 1) / kThreads;     // per thread and array
        uint4 qv[kLd], kv[kLd], vv;
#pragma unroll
        for (int j = 0; j < kLd; ++j) {
            const int i = t + j * kThreads;
            if (i < nb * kQ4) {
                qv[j] = *reinterpret_cast<const uint4*>(a.q + (row0 + i / kQ4) * dqk + (i % kQ4) * 8);
                kv[j] = *reinterpret_cast<const uint4*>(a.k + (row0 + i / kQ4) * dqk + (i % kQ4) * 8);
            }
        }
        const bool v_ld = t < nb * (kCols / 8);
        if (v_ld) vv = *reinterpret_cast<const uint4*>(a.v + (row0 + t / (kCols / 8)) * dhv + x0 + (t % (kCols / 8)) * 8);
        auto put8 = [](float* dst, const uint4& u) {
            const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(b2[e]);
                dst[2 * e] = f.x;
                dst[2 * e + 1] = f.y;
            }
        };
#pragma unroll
        for (int j = 0; j < kLd; ++j) {
            const int i = t + j * kThreads;
            if (i < nb * kQ4) {
                put8(&qs[i / kQ4][(i % kQ4) * 8], qv[j]);
                put8(&ks[i / kQ4][(i % kQ4) * 8], kv[j]);
            }
        }
        if (v_ld) put8(&vs[t / (kCols / 8)][(t % (kCols / 8)) * 8], vv);
        // the block's gates (one warp, the scalar m recurrence in order):
        // gi <- input gate, gf <- forget gate, gm <- exp(-m) of each step
        if (t < 32) {
            const float ip = t < nb ? a.i_pre[row0 + t] : 0.f, fp = t < nb ? a.f_pre[row0 + t] : 0.f;
            float fg = 0.f, ig = 0.f;
            if (!is_exp && t < nb) {
                fg = sigmf(fp);
                ig = sigmf(ip);
            }
            if (is_exp) {  // warp 0 runs the scalar m recurrence over the block's steps (lane st keeps step st)
                for (int st = 0; st < nb; ++st) {
                    const float ips = __shfl_sync(0xffffffffu, ip, st), fps = __shfl_sync(0xffffffffu, fp, st);
                    const float f_log = logsigf(fps) + m;
                    const float m_new = fmaxf(f_log, ips);
                    if (a.stab && t == 0 && blockIdx.x == 0) {  // stab::exp_guarded at recurrent.cpp:17-18
                        sl.note((f_log - m_new) * 1.4426950408889634f);
                        sl.note((ips - m_new) * 1.4426950408889634f);
                    }
                    if (t == st) {
                        fg = expf(f_log - m_new);
                        ig = expf(ips - m_new);
                    }
                    m = m_new;
                    if (t == st) gm[st] = expf(-m_new);
                }
            }
            if (t < nb) {
                gi[t] = ig;
                gf[t] = fg;
            }
        }
        __syncthreads();  // (m is carried by warp 0 only: thread 0 writes m_state at the end)
        for (int st = 0; st < nb; ++st) {
            const int s = s0 + st, par = s & 1;
            const float ig = gi[st], fg = gf[st];
            const float iv = ig * vs[st][xl];
            float hq[4] = {0.f, 0.f, 0.f, 0.f};  // four independent partial dot chains
            // the 32 lanes of a warp share the row group: broadcast 16-B reads
            const float4* k4 = reinterpret_cast<const float4*>(&ks[st][pg * R]);
            const float4* q4 = reinterpret_cast<const float4*>(&qs[st][pg * R]);
#pragma unroll
            for (int r4 = 0; r4 < R / 4; ++r4) {
                const float4 kk = k4[r4], qq = q4[r4];
                const float kv[4] = {kk.x, kk.y, kk.z, kk.w}, qv[4] = {qq.x, qq.y, qq.z, qq.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int r = 4 * r4 + e;
                    c[r] = fmaf(fg, c[r], iv * kv[e]);
                    hq[e] = fmaf(c[r], qv[e], hq[e]);
                }
            }
            const float hp = (hq[0] + hq[1]) + (hq[2] + hq[3]);
            red[par][pg][xl] = hp;
            if (is_exp && t < dqk) {
                n_reg = fmaf(fg, n_reg, ig * ks[st][t]);
                float nq = n_reg * qs[st][t];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) nq += __shfl_xor_sync(0xffffffffu, nq, o);
                if ((t & 31) == 0) nqw[par][t >> 5] = nq;
            }
            __syncthreads();
            if (t < kCols) {
                float h = (red[par][0][t] + red[par][1][t] + red[par][2][t] + red[par][3][t]) * rs;
                if (is_exp) {
                    float nq = 0.f;
#pragma unroll
                    for (int w = 0; w < (dqk + 31) / 32; ++w) nq += nqw[par][w];
                    h /= fmaxf(fabsf(nq * rs), gm[st]);
                }
                a.h[(row0 + st) * dhv + x0 + t] = __float2bfloat16_rn(h);
            }
        }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) C[static_cast<size_t>(pg * R + r) * dhv] = c[r];
    if (a.stab && t == 0) sl.flush(a.stab);
    if (kCluster) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");  // every slice read n / m
    if (blockIdx.x == 0 && is_exp) {
        if (t < dqk && a.n_state) a.n_state[static_cast<size_t>(bh) * dqk + t] = n_reg;
        if (t == 0 && a.m_state) a.m_state[bh] = m;
    }
}

}  // namespace

bool recurrent_supported(int dqk, int dhv) {
    return (dqk == 64 || dqk == 128 || dqk == 256) && dhv % kCols == 0 && dhv > 0;
}

bool recurrent_cluster(int dhv) { return dhv / kCols <= 8; }

template <int R>
static void launch_r(const RecurrentArgs& a, int BH, cudaStream_t st) {
    const dim3 grid(a.dhv / kCols, BH);
    if (recurrent_cluster(a.dhv)) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(kThreads);
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = a.dhv / kCols;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, recurrent_kernel<R, true>, a);
    } else {
        recurrent_kernel<R, false><<<grid, kThreads, 0, st>>>(a);
    }
}

void launch_recurrent(const RecurrentArgs& a, int BH, int dqk, cudaStream_t st) {
    if (dqk == 256) launch_r<64>(a, BH, st);
    else if (dqk == 128) launch_r<32>(a, BH, st);
    else launch_r<16>(a, BH, st);
}

}  // namespace tfla_k
