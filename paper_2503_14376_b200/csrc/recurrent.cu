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
// per launch however many steps T the launch folds. Per step the q/k/v
// vectors are staged in shared memory; h is reduced over the 4 row groups.
// n and q.n (exp) are carried redundantly by every column slice of a head.
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

template <int R>  // rows of C per thread = dqk / 4
__global__ void __launch_bounds__(kThreads) recurrent_kernel(RecurrentArgs a) {
    __shared__ float qs[4 * R], ks[4 * R], vs[kCols], ns[4 * R];
    __shared__ float red[4][kCols], nqw[8];
    const int dqk = 4 * R, dhv = a.dhv, T = a.T;
    const int bh = blockIdx.y, x0 = blockIdx.x * kCols;
    const int t = threadIdx.x, xl = t & (kCols - 1), pg = t >> 6;
    const bool is_exp = a.variant == 0;
    const float rs = rsqrtf(static_cast<float>(dqk));

    float c[R];
    float* C = a.c_state + static_cast<size_t>(bh) * dqk * dhv + x0 + xl;
#pragma unroll
    for (int r = 0; r < R; ++r) c[r] = C[static_cast<size_t>(pg * R + r) * dhv];
    // n / m are read from the launch-private copies (n_in / m_in): the column
    // slices of a head run in any order, and slice 0 overwrites n_state / m_state
    if (t < dqk) ns[t] = (is_exp && a.n_in) ? a.n_in[static_cast<size_t>(bh) * dqk + t] : 0.f;
    float m = (is_exp && a.m_in) ? a.m_in[bh] : 0.f;

    StabLocal sl;
    for (int s = 0; s < T; ++s) {
        const size_t row = static_cast<size_t>(bh) * T + s;
        if (t < dqk) {
            qs[t] = __bfloat162float(a.q[row * dqk + t]);
            ks[t] = __bfloat162float(a.k[row * dqk + t]);
        }
        if (t < kCols) vs[t] = __bfloat162float(a.v[row * dhv + x0 + t]);
        const float ip = a.i_pre[row], fp = a.f_pre[row];
        float fg, ig;
        if (is_exp) {
            const float f_log = logsigf(fp) + m;
            const float m_new = fmaxf(f_log, ip);
            if (a.stab && t == 0 && blockIdx.x == 0) {  // stab::exp_guarded at recurrent.cpp:17-18
                sl.note((f_log - m_new) * 1.4426950408889634f);
                sl.note((ip - m_new) * 1.4426950408889634f);
            }
            fg = expf(f_log - m_new);
            ig = expf(ip - m_new);
            m = m_new;
        } else {
            fg = sigmf(fp);
            ig = sigmf(ip);
        }
        __syncthreads();
        const float iv = ig * vs[xl];
        float hp = 0.f;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int p = pg * R + r;
            c[r] = fmaf(fg, c[r], iv * ks[p]);
            hp = fmaf(c[r], qs[p], hp);
        }
        red[pg][xl] = hp;
        if (is_exp) {
            float nq = 0.f;
            if (t < dqk) {
                const float n = fmaf(fg, ns[t], ig * ks[t]);
                ns[t] = n;
                nq = n * qs[t];
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) nq += __shfl_xor_sync(0xffffffffu, nq, o);
            if ((t & 31) == 0) nqw[t >> 5] = nq;
        }
        __syncthreads();
        if (t < kCols) {
            float h = (red[0][t] + red[1][t] + red[2][t] + red[3][t]) * rs;
            if (is_exp) {
                float nq = 0.f;
                for (int w = 0; w < (dqk + 31) / 32; ++w) nq += nqw[w];
                h /= fmaxf(fabsf(nq * rs), expf(-m));
            }
            a.h[row * dhv + x0 + t] = __float2bfloat16_rn(h);
        }
        __syncthreads();  // q / k / v / red / nqw are rewritten by the next step
    }
#pragma unroll
    for (int r = 0; r < R; ++r) C[static_cast<size_t>(pg * R + r) * dhv] = c[r];
    if (a.stab && t == 0) sl.flush(a.stab);
    if (blockIdx.x == 0 && is_exp) {
        if (t < dqk && a.n_state) a.n_state[static_cast<size_t>(bh) * dqk + t] = ns[t];
        if (t == 0 && a.m_state) a.m_state[bh] = m;
    }
}

}  // namespace

bool recurrent_supported(int dqk, int dhv) {
    return (dqk == 64 || dqk == 128 || dqk == 256) && dhv % kCols == 0 && dhv > 0;
}

void launch_recurrent(const RecurrentArgs& a, int BH, int dqk, cudaStream_t st) {
    dim3 grid(a.dhv / kCols, BH);
    if (dqk == 256) recurrent_kernel<64><<<grid, kThreads, 0, st>>>(a);
    else if (dqk == 128) recurrent_kernel<32><<<grid, kThreads, 0, st>>>(a);
    else recurrent_kernel<16><<<grid, kThreads, 0, st>>>(a);
}

}  // namespace tfla_k
