// state_scan2.cu -- K1 / K3 for wide heads: the inter-chunk state recurrence
// with the running state resident in TMEM.
//
//   fwd (state_recurrence_head, chunkwise.cpp:13-68):
//       C_{k+1} = gbar_k C_k + (a_bar o K_k)^T V_k,   n_{k+1} = gbar_k n_k + K_k^T a_bar
//   bwd (backward_state_pass_head, chunkwise.cpp:196-237):
//       dC_k = gbar_k dC_{k+1} + (w o Q_k)^T dH_k,    d_g[k] = gbar_k <C_k, dC_{k+1}>
//
// CTA = (256-column x half, 128-row p tile, head); two CTAs per SM, so one
// CTA's state update overlaps the other's MMAs. Unlike state_scan.cu (64-column
// tiles, state in registers, gate applied to the 64-column B operand), the
// state lives in TMEM (256 fp32 columns) and the tensor core accumulates
// (a_bar o K)^T V straight into it: per chunk the epilogue warps read C_k once
// (bf16 operand copy + optional fp32 reference-layout state + the backward's
// d_g dot) and scale it by gbar_k in place, then the MMAs of chunk k add the
// chunk's contribution. The gate sits on the contraction dim and is applied to
// the 128-column A operand (K / Q rows) in shared memory, a quarter of the
// bytes the 64-column design transformed per state element; the N = 256 MMAs
// read 96 B/clk of shared memory instead of 192 (N = 64). Requires d_qk % 128
// == 0, d_hv % 256 == 0, L % 32 == 0.
// Warps: 0 TMA producer, 1 tcgen05 issuer (+ TMEM owner), 2-3 gate transform
// (+ n increments), 4-11 state epilogue (TMEM lane quarter warp % 4, column
// half (warp - 4) / 4).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "host_util.h"
#include "kernels.h"
#include "tc.cuh"

namespace tfla_k {
namespace {

constexpr int kRows = 32;                 // sequence rows per stage
constexpr int kStages = 4;
constexpr int kA = kRows * 128 * 2;       // 8 KB: 32 rows x 128 p (two 64-p atoms)
constexpr int kB = kRows * 256 * 2;       // 16 KB: 32 rows x 256 x (four 64-x atoms)
constexpr int kStage = kA + kB;           // 24 KB
constexpr int kTr = 64;                   // transform threads
constexpr int kEpi = 256;                 // epilogue threads
constexpr int kThreads = 64 + kTr + kEpi;  // 384
constexpr int kOffRed = kStages * kStage;                  // u partial exchange [4][128] f32
constexpr int kOffDg = kOffRed + 4 * 128 * 4;              // d_g exchange [2][8] f32
constexpr int kOffBar = kOffDg + 2 * 8 * 4;
constexpr int kSmemBytes = kOffBar + 256;

template <bool kBwd>
__global__ void __launch_bounds__(kThreads, 2)
    state_scan2_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                       ScanArgs args, __nv_bfloat16* __restrict__ states_out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* stages = smem;
    float* ured = reinterpret_cast<float*>(smem + kOffRed);
    float* dgred = reinterpret_cast<float*>(smem + kOffDg);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
    uint64_t* full = bars;
    uint64_t* tfull = full + kStages;
    uint64_t* empty = tfull + kStages;
    uint64_t* cfull = empty + kStages;     // chunk's MMAs done: the next state is in TMEM
    uint64_t* cscaled = cfull + 1;         // state emitted and scaled by gbar: MMAs may add
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cscaled + 1);

    const Geom& G = args.g;
    const int T = G.T, L = G.L, NC = G.NC, dqk = G.dqk, dhv = G.dhv;
    const int xt = blockIdx.x, pt = blockIdx.y, bh = blockIdx.z;
    const int x0 = xt * 256, p0 = pt * 128;
    const int nsb = L / kRows;
    const int total = NC * nsb;
    const int warp = tc::warp_id();

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&tfull[s], kTr);
            tc::mbar_init(&empty[s], 1);
        }
        tc::mbar_init(cfull, 1);
        tc::mbar_init(cscaled, kEpi);
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, 256);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (tc::elect_one()) {
            for (int gi = 0; gi < total; ++gi) {
                const int it = gi / nsb, sb = gi % nsb;
                const int c = kBwd ? NC - 1 - it : it;
                const int row = c * L + sb * kRows;
                const int s = gi % kStages;
                tc::mbar_wait(&empty[s], ((gi / kStages) & 1) ^ 1);
                uint8_t* sa = stages + s * kStage;
                tc::mbar_arrive_expect_tx(&full[s], kStage);
                for (int a = 0; a < 2; ++a) tc::tma_load_3d(sa + a * 4096, &mapA, &full[s], p0 + 64 * a, row, bh);
                for (int a = 0; a < 4; ++a)
                    tc::tma_load_3d(sa + kA + a * 4096, &mapB, &full[s], x0 + 64 * a, row, bh);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ tcgen05 issuer
        const uint32_t idesc = tc::idesc_bf16(128, 256, 1, 1);
        for (int it = 0; it < NC; ++it) {
            tc::mbar_wait(cscaled, it & 1);
            tc::tc_fence_after();
            for (int sb = 0; sb < nsb; ++sb) {
                const int gi = it * nsb + sb;
                const int s = gi % kStages;
                tc::mbar_wait(&tfull[s], (gi / kStages) & 1);
                tc::tc_fence_after();
                const uint32_t sa = tc::smem_u32(stages + s * kStage);
                if (tc::elect_one()) {
#pragma unroll
                    for (int ks = 0; ks < kRows / 16; ++ks)
                        tc::mma_bf16(tmem, tc::mnmajor_desc(sa, kRows, ks), tc::mnmajor_desc(sa + kA, kRows, ks),
                                     idesc, 1u);
                    tc::mma_commit(&empty[s]);
                    if (sb == nsb - 1) tc::mma_commit(cfull);
                }
                __syncwarp();
            }
        }
    } else if (warp < 4) {
        // ------------------------------------------------ gate transform warps 2..3
        // Scale the rows of every landed A stage (32 rows x 128 p, two SW128
        // atoms) by w (the gate on the contraction dim); (fwd, x half 0)
        // accumulate the n increments u_k[p] = sum_j a_bar_j k_j[p] in fp32.
        const int tt = threadIdx.x - 64;  // 0..63
        const int pc = tt & 15;           // this thread's 8-wide p chunk (fixed)
        const int atom = pc >> 3, c8 = pc & 7;
        const bool do_n = !kBwd && args.u_part != nullptr && xt == 0;
        const float* wv = args.w + static_cast<size_t>(bh) * T;
        float np[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) np[e] = 0.f;
        float wn[8];
        auto load_w = [&](int gi) {
            if (gi >= total) return;
            const int it2 = gi / nsb, sb2 = gi % nsb;
            const int c2 = kBwd ? NC - 1 - it2 : it2;
            const float* wk = wv + c2 * L + sb2 * kRows;
#pragma unroll
            for (int m = 0; m < 8; ++m) wn[m] = __ldg(wk + (tt >> 4) + 4 * m);
        };
        load_w(0);
        for (int gi = 0; gi < total; ++gi) {
            const int it = gi / nsb, sb = gi % nsb;
            const int c = kBwd ? NC - 1 - it : it;
            const int s = gi % kStages;
            float wr[8];
#pragma unroll
            for (int m = 0; m < 8; ++m) wr[m] = wn[m];
            load_w(gi + 1);
            tc::mbar_wait(&full[s], (gi / kStages) & 1);
            uint8_t* sa = stages + s * kStage + atom * 4096;
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int r = (tt >> 4) + 4 * m;
                uint4* ptr = reinterpret_cast<uint4*>(sa + r * 128 + ((c8 ^ (r & 7)) << 4));
                uint4 val = *ptr;
                __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&val);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 f = __bfloat1622float2(h2[e]);
                    const float a0 = f.x * wr[m], a1 = f.y * wr[m];
                    if (do_n) {
                        np[2 * e] += a0;
                        np[2 * e + 1] += a1;
                    }
                    h2[e] = __floats2bfloat162_rn(a0, a1);
                }
                *ptr = val;
            }
            tc::fence_proxy_async_smem();
            tc::mbar_arrive(&tfull[s]);
            if (do_n && sb == nsb - 1) {  // u_c for this p tile (n_xtiles = 1)
#pragma unroll
                for (int e = 0; e < 8; ++e) ured[(tt >> 4) * 128 + pc * 8 + e] = np[e];
                tc::named_bar_sync(2, kTr);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int p = tt + 64 * h;
                    const float u = ured[p] + ured[128 + p] + ured[256 + p] + ured[384 + p];
                    if (p0 + p < dqk) args.u_part[(static_cast<size_t>(bh) * NC + c) * dqk + p0 + p] = u;
                }
                tc::named_bar_sync(2, kTr);
#pragma unroll
                for (int e = 0; e < 8; ++e) np[e] = 0.f;
            }
        }
    } else {
        // ------------------------------------------------ state epilogue warps 4..11
        const int ep = threadIdx.x - 128;              // 0..255
        const int row = (warp & 3) * 32 + tc::lane_id();  // TMEM lane == p within the tile
        const int hx = (warp - 4) >> 2;                 // column half (128 columns)
        const int col0 = hx * 128;
        const uint32_t trow = tc::tmem_row_addr(tmem) + col0;
        const float* gb = args.gbar + static_cast<size_t>(bh) * NC;
        const bool p_ok = p0 + row < dqk;
        const size_t prow = static_cast<size_t>(p0 + row) * dhv + x0 + col0;  // offset inside one state
        const bool do_dg = kBwd && args.dg_part != nullptr;
        const int ntiles = gridDim.x * gridDim.y;

        // process the state S held in TMEM (first: the initial state, in
        // registers) -- emit it, (bwd) its d_g dot, scale it by g and store it back
        auto process = [&](int k, bool from_tmem, bool scale_store) {
            // fwd: S = C_k (emit slot k);  bwd: S = dC_{c+1}, c = NC-1-k (emit slot c)
            const int c = kBwd ? NC - 1 - k : k;
            const bool emit = k < NC;
            const float g = emit ? __ldg(gb + c) : 0.f;
            float dg = 0.f;
            const size_t slot = emit ? (static_cast<size_t>(bh) * NC + c) * dqk * dhv : 0;
            __nv_bfloat16* so = states_out + slot + prow;
            const __nv_bfloat16* cs = (do_dg && emit) ? args.c_saved + slot + prow : nullptr;
            float* f32 = nullptr;  // fp32 reference-layout state [BH][NC+1][dqk][dhv]
            if (!kBwd && args.c_states) f32 = args.c_states + (static_cast<size_t>(bh) * (NC + 1) + k) * dqk * dhv;
            if (kBwd && args.dc_states)
                f32 = args.dc_states + (static_cast<size_t>(bh) * (NC + 1) + (NC - k)) * dqk * dhv;
#pragma unroll 1
            for (int piece = 0; piece < 4; ++piece) {
                uint4 cur[4];  // (bwd) this piece of C_c, loads in flight under the TMEM load
                if (cs && p_ok)
#pragma unroll
                    for (int q = 0; q < 4; ++q) cur[q] = __ldg(reinterpret_cast<const uint4*>(cs + piece * 32) + q);
                float v[32];
                if (from_tmem) {
                    tc::tmem_ld32(trow + piece * 32, v);
                    tc::tmem_ld_wait();
                } else {
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] = 0.f;
                    if (!kBwd && args.c_init && p_ok) {
                        const float* src = args.c_init + static_cast<size_t>(bh) * dqk * dhv + prow + piece * 32;
#pragma unroll
                        for (int e = 0; e < 32; e += 4) {
                            const float4 f = *reinterpret_cast<const float4*>(src + e);
                            v[e] = f.x, v[e + 1] = f.y, v[e + 2] = f.z, v[e + 3] = f.w;
                        }
                    }
                }
                if (p_ok) {
                    if (emit) {
                        uint4* dst = reinterpret_cast<uint4*>(so + piece * 32);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            uint4 w;
                            w.x = tc::pack_bf16(v[8 * q], v[8 * q + 1]);
                            w.y = tc::pack_bf16(v[8 * q + 2], v[8 * q + 3]);
                            w.z = tc::pack_bf16(v[8 * q + 4], v[8 * q + 5]);
                            w.w = tc::pack_bf16(v[8 * q + 6], v[8 * q + 7]);
                            dst[q] = w;
                        }
                    }
                    if (f32) {
                        float* d = f32 + prow + piece * 32;
#pragma unroll
                        for (int e = 0; e < 32; e += 4)
                            *reinterpret_cast<float4*>(d + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
                    }
                    if (!kBwd && k == NC && args.c_final) {
                        float* d = args.c_final + static_cast<size_t>(bh) * dqk * dhv + prow + piece * 32;
#pragma unroll
                        for (int e = 0; e < 32; e += 4)
                            *reinterpret_cast<float4*>(d + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
                    }
                    if (cs) {  // d_g: <C_c, dC_{c+1}> over this piece (C_c from the forward's bf16 copy)
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&cur[q]);
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const float2 f = __bfloat1622float2(h2[e]);
                                dg = fmaf(f.x, v[8 * q + 2 * e], dg);
                                dg = fmaf(f.y, v[8 * q + 2 * e + 1], dg);
                            }
                        }
                    }
                }
                if (scale_store) {
                    uint32_t w[32];
#pragma unroll
                    for (int e = 0; e < 32; ++e) w[e] = __float_as_uint(g * v[e]);
                    tc::tmem_st32(trow + piece * 32, w);
                }
            }
            if (scale_store) {
                tc::tmem_st_wait();
                tc::tc_fence_before();
                tc::mbar_arrive(cscaled);
            }
            if (do_dg && emit) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) dg += __shfl_xor_sync(0xffffffffu, dg, o);
                float* red = dgred + (k & 1) * 8;
                if (tc::lane_id() == 0) red[warp - 4] = dg;
                tc::named_bar_sync(3, kEpi);
                if (ep == 0) {
                    float sdg = 0.f;
#pragma unroll
                    for (int w8 = 0; w8 < 8; ++w8) sdg += red[w8];
                    args.dg_part[(static_cast<size_t>(bh) * NC + c) * ntiles + pt * gridDim.x + xt] = sdg;
                }
            }
        };

        process(0, false, true);  // the initial state (C_0 / dC_NC = 0)
        for (int k = 1; k <= NC; ++k) {
            tc::mbar_wait(cfull, (k - 1) & 1);
            tc::tc_fence_after();
            // k < NC: emit + scale the state entering chunk k; k == NC: the final
            // state (fwd: c_states[NC] / c_final; bwd: dC_0 into dc_states[0])
            const bool last = k == NC;
            if (!last) {
                process(k, true, true);
            } else if ((!kBwd && (args.c_states || args.c_final)) || (kBwd && args.dc_states)) {
                process(k, true, false);
            }
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(tmem, 256);
}

}  // namespace

bool scan2_supported(const Geom& g) {
    return g.dqk % 128 == 0 && g.dhv % 256 == 0 && g.L % kRows == 0 && !tfla_host::env_flag("TFLA_NO_SCAN2");
}

// Measured (B200, 7B head shape, profiles/r02_*): the per-chunk state update
// is serial with the chunk's MMAs, so the TMEM-resident scan wins where the
// chunk is long -- forward K1 at L >= 512 (0.39 vs 0.48 ms) -- and loses where
// the update dominates: the backward's d_g reads of C_k sit on that serial
// path (L = 128: 1.04 vs 0.56 ms). TFLA_SCAN2=1 forces it for both passes.
bool scan2_use(const Geom& g, bool bwd) {
    if (!scan2_supported(g)) return false;
    if (tfla_host::env_flag("TFLA_SCAN2")) return true;
    // and only with at least one CTA per SM: its (head, p, x-half) grid is a
    // quarter of state_scan.cu's, which is a chain-latency disaster at long
    // context (B=1, NH=8: 32 CTAs; 1.87 vs 0.75 ms at L=512)
    const long ctas = static_cast<long>(g.dhv / 256) * (g.dqk / 128) * g.BH;
    return !bwd && g.L >= 512 && ctas >= tfla_host::num_sms();
}

int launch_state_scan2(bool bwd, const void* a_src, const void* b_src, void* states_out, const ScanArgs& a,
                       cudaStream_t st) {
    using namespace tfla_host;
    const Geom& g = a.g;
    CUtensorMap ma, mb;
    if (!make_tmap_bf16_3d(&ma, a_src, g.BH, g.T, g.dqk, 64, kRows) ||
        !make_tmap_bf16_3d(&mb, b_src, g.BH, g.T, g.dhv, 64, kRows))
        return 4;
    dim3 grid(g.dhv / 256, g.dqk / 128, g.BH);
    auto* out = static_cast<__nv_bfloat16*>(states_out);
    if (bwd) {
        ensure_smem_attr(reinterpret_cast<const void*>(state_scan2_kernel<true>), kSmemBytes);
        state_scan2_kernel<true><<<grid, kThreads, kSmemBytes, st>>>(ma, mb, a, out);
    } else {
        ensure_smem_attr(reinterpret_cast<const void*>(state_scan2_kernel<false>), kSmemBytes);
        state_scan2_kernel<false><<<grid, kThreads, kSmemBytes, st>>>(ma, mb, a, out);
    }
    return 0;
}

}  // namespace tfla_k
