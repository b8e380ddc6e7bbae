// state_scan.cu -- K1 (recurrent forward) and K3 (recurrent backward) on tcgen05.
//
// Forward  (state_recurrence_head, chunkwise.cpp:13-68):
//     C_{k+1} = gbar_k C_k + (a_bar o K_k)^T V_k,   n_{k+1} = gbar_k n_k + K_k^T a_bar
// Backward (backward_state_pass_head, chunkwise.cpp:196-237):
//     dC_k = gbar_k dC_{k+1} + (w o Q_k)^T dH_k,    w_i = b_bar_i / (h_denom_i sqrt(d_qk))
//     d_g[k] = gbar_k * sum(C_k o dC_{k+1})
// Both are "state_in -> emit; state = gbar * state + A^T diag(w) B" sweeps, so one
// kernel serves both directions.
//
// CTA = (x tile of N columns of d_hv, p tile of 128 rows of d_qk, head). Warp
// roles: warp 0 = TMA producer, warp 1 = tcgen05 issuer (+TMEM owner), warps
// 2..5 = transform / epilogue (128 threads, one accumulator row each).
// Per chunk: TMA streams 64-row k-blocks of A (MN-major, M = p) and B (MN-major,
// N = x) into a ring; the epilogue warps scale the B rows by w (the contraction
// dim carries the gate, so it must be applied to an operand); the MMA warp
// accumulates D_k = A^T diag(w) B into one of two TMEM buffers; the epilogue
// folds D_k into the fp32 register-resident state while the next chunk's MMA
// runs, and streams the state out as bf16 (TMA store) for the parallel kernels.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "host_util.h"
#include "kernels.h"
#include "tc.cuh"

namespace tfla_k {
namespace {

constexpr int kStages = 4;
constexpr int kAStage = 128 * 64 * 2;  // 2 MN atoms of 64 p x 64 rows

template <int N>
struct ScanSmem {
    static constexpr int kBStage = N * 64 * 2;
    static constexpr int kStage = kAStage + kBStage;
    static constexpr int kStaging = 128 * N * 2;
    static constexpr int kBytes = kStages * kStage + kStaging + 1024 /*align*/ + 512 /*bars*/;
};

template <bool kBwd, int N>
__global__ void __launch_bounds__(192, 1)
    state_scan_kernel(const __grid_constant__ CUtensorMap mapA,
                      const __grid_constant__ CUtensorMap mapB,
                      const __grid_constant__ CUtensorMap mapS, ScanArgs args) {
    using SM = ScanSmem<N>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint8_t* stages = smem;
    uint8_t* staging = smem + kStages * SM::kStage;
    uint64_t* bars = reinterpret_cast<uint64_t*>(staging + SM::kStaging);
    uint64_t* full = bars;
    uint64_t* tfull = full + kStages;
    uint64_t* empty = tfull + kStages;
    uint64_t* accfull = empty + kStages;  // [2]
    uint64_t* accempty = accfull + 2;     // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + 2);
    float* red = reinterpret_cast<float*>(tmem_slot + 4);

    const Geom& G = args.g;
    const int T = G.T, L = G.L, NC = G.NC, dqk = G.dqk, dhv = G.dhv;
    const int xt = blockIdx.x, pt = blockIdx.y, bh = blockIdx.z;
    const int x0 = xt * N, p0 = pt * 128;
    const int nA = (dqk - p0) >= 128 ? 2 : 1;
    const int nkb = L / 64;
    const int total = NC * nkb;
    const int warp = tc::warp_id();

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&tfull[s], 128);
            tc::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&accfull[b], 1);
            tc::mbar_init(&accempty[b], 128);
        }
        tc::fence_barrier_init();
    }
    if (nA == 1) {  // d_qk tail: the second MN atom of A is never loaded -> zeros
        for (int i = threadIdx.x; i < kStages * 512; i += blockDim.x) {
            const int s = i / 512, u = i % 512;
            reinterpret_cast<uint4*>(stages + s * SM::kStage + 8192)[u] = make_uint4(0, 0, 0, 0);
        }
        tc::fence_proxy_async_smem();
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, 2 * N);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (tc::elect_one()) {
            const uint32_t bytes = nA * 8192 + N * 128;
            for (int gi = 0; gi < total; ++gi) {
                const int it = gi / nkb, kb = gi % nkb;
                const int c = kBwd ? NC - 1 - it : it;
                const int row = c * L + kb * 64;
                const int s = gi % kStages;
                const uint32_t ph = (gi / kStages) & 1;
                tc::mbar_wait(&empty[s], ph ^ 1);
                uint8_t* sa = stages + s * SM::kStage;
                uint8_t* sb = sa + kAStage;
                tc::mbar_arrive_expect_tx(&full[s], bytes);
                for (int a = 0; a < nA; ++a)
                    tc::tma_load_3d(sa + a * 8192, &mapA, &full[s], p0 + 64 * a, row, bh);
                for (int a = 0; a < N / 64; ++a)
                    tc::tma_load_3d(sb + a * 8192, &mapB, &full[s], x0 + 64 * a, row, bh);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ tcgen05 issuer
        const uint32_t idesc = tc::idesc_bf16(128, N, 1, 1);
        for (int it = 0; it < NC; ++it) {
            const int buf = it & 1;
            tc::mbar_wait(&accempty[buf], ((it >> 1) & 1) ^ 1);
            tc::tc_fence_after();
            for (int kb = 0; kb < nkb; ++kb) {
                const int gi = it * nkb + kb;
                const int s = gi % kStages;
                tc::mbar_wait(&tfull[s], (gi / kStages) & 1);
                tc::tc_fence_after();
                const uint32_t sa = tc::smem_u32(stages + s * SM::kStage);
                const uint32_t sb = sa + kAStage;
                if (tc::elect_one()) {
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks)
                        tc::mma_bf16(tmem + buf * N, tc::mnmajor_desc(sa, 64, ks),
                                     tc::mnmajor_desc(sb, 64, ks), idesc, (kb | ks) ? 1u : 0u);
                    tc::mma_commit(&empty[s]);
                    if (kb == nkb - 1) tc::mma_commit(&accfull[buf]);
                }
                __syncwarp();
            }
        }
    } else {
        // ------------------------------------------------ transform + epilogue
        const int et = threadIdx.x - 64;                      // 0..127
        const int row = (warp & 3) * 32 + tc::lane_id();      // TMEM lane == p within tile
        const bool row_ok = row < dqk - p0;
        const bool do_n = !kBwd && xt == 0 && args.n_states != nullptr;
        const float* wv = args.w + static_cast<size_t>(bh) * T;
        const float* gb = args.gbar + static_cast<size_t>(bh) * NC;
        const uint32_t trow = tc::tmem_row_addr(tmem);

        float st[N];
#pragma unroll
        for (int i = 0; i < N; ++i) st[i] = 0.f;
        float nst = 0.f, npart_cur = 0.f, npart_nxt = 0.f;

        // Scale the B rows of every k-block stage of chunk `it` by w; (fwd,
        // x tile 0) also accumulate the n-state partial sum_j w_j k_j[p].
        auto transform = [&](int it) -> float {
            const int c = kBwd ? NC - 1 - it : it;
            float np = 0.f;
            for (int kb = 0; kb < nkb; ++kb) {
                const int gi = it * nkb + kb;
                const int s = gi % kStages;
                tc::mbar_wait(&full[s], (gi / kStages) & 1);
                uint8_t* sa = stages + s * SM::kStage;
                uint8_t* sb = sa + kAStage;
                const float* wk = wv + c * L + kb * 64;
#pragma unroll 4
                for (int u = et; u < N * 8; u += 128) {
                    const int atom = u >> 9, r = (u >> 3) & 63, ch = u & 7;
                    uint4* ptr = reinterpret_cast<uint4*>(sb + atom * 8192 + r * 128 + ch * 16);
                    uint4 val = *ptr;
                    const float wr = __ldg(wk + r);
                    __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&val);
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        float2 f = __bfloat1622float2(h2[e]);
                        h2[e] = __floats2bfloat162_rn(f.x * wr, f.y * wr);
                    }
                    *ptr = val;
                }
                if (do_n && row_ok) {
                    const int atom = row >> 6, pc = row & 63;
                    const __nv_bfloat16* a16 = reinterpret_cast<const __nv_bfloat16*>(sa + atom * 8192);
#pragma unroll 8
                    for (int r = 0; r < 64; ++r) {
                        const int off = r * 64 + ((((pc >> 3) ^ (r & 7)) << 3) | (pc & 7));
                        np += __ldg(wk + r) * __bfloat162float(a16[off]);
                    }
                }
                tc::fence_proxy_async_smem();
                tc::mbar_arrive(&tfull[s]);
            }
            return np;
        };

        // Emit the incoming state of chunk c: bf16 operand copy (TMA store),
        // optional fp32 reference-layout states, n, and (bwd) the d_g partial.
        auto emit = [&](int c, bool final_state) {
            if (!kBwd && args.c_states && row_ok) {
                float* dst = args.c_states +
                             ((static_cast<size_t>(bh) * (NC + 1) + c) * dqk + p0 + row) * dhv + x0;
#pragma unroll
                for (int i = 0; i < N; i += 4)
                    *reinterpret_cast<float4*>(dst + i) = make_float4(st[i], st[i + 1], st[i + 2], st[i + 3]);
            }
            if (!kBwd && final_state) {
                if (args.c_final && row_ok) {
                    float* dst = args.c_final + (static_cast<size_t>(bh) * dqk + p0 + row) * dhv + x0;
#pragma unroll
                    for (int i = 0; i < N; i += 4)
                        *reinterpret_cast<float4*>(dst + i) =
                            make_float4(st[i], st[i + 1], st[i + 2], st[i + 3]);
                }
                if (do_n && row_ok && args.n_final)
                    args.n_final[static_cast<size_t>(bh) * dqk + p0 + row] = nst;
            }
            if (do_n && row_ok)
                args.n_states[(static_cast<size_t>(bh) * (NC + 1) + c) * dqk + p0 + row] = nst;
            if (final_state) return;
            if (kBwd) {
                float acc = 0.f;
                if (row_ok) {
                    const __nv_bfloat16* cs =
                        args.c_saved + ((static_cast<size_t>(bh) * NC + c) * dqk + p0 + row) * dhv + x0;
#pragma unroll
                    for (int i = 0; i < N; i += 8) {
                        uint4 raw = *reinterpret_cast<const uint4*>(cs + i);
                        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            float2 f = __bfloat1622float2(h2[e]);
                            acc += f.x * st[i + 2 * e] + f.y * st[i + 2 * e + 1];
                        }
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                if (tc::lane_id() == 0) red[warp & 3] = acc;
            }
            if (et == 0) tc::tma_store_wait_read<0>();
            tc::named_bar_sync(1, 128);
            if (kBwd && et == 0) {
                const int ntiles = gridDim.x * gridDim.y;
                args.dg_part[(static_cast<size_t>(bh) * NC + c) * ntiles + pt * gridDim.x + xt] =
                    red[0] + red[1] + red[2] + red[3];
            }
#pragma unroll
            for (int c8 = 0; c8 < N / 8; ++c8) tc::sw128_store8(staging, row, c8, 128, st + 8 * c8);
            tc::fence_proxy_async_smem();
            tc::named_bar_sync(1, 128);
            if (et == 0) {
                for (int a = 0; a < N / 64; ++a)
                    tc::tma_store_3d(&mapS, staging + a * 16384, x0 + 64 * a, p0, bh * NC + c);
                tc::tma_store_commit();
            }
        };

        npart_cur = transform(0);
        for (int it = 0; it < NC; ++it) {
            const int c = kBwd ? NC - 1 - it : it;
            emit(c, false);
            if (it + 1 < NC) npart_nxt = transform(it + 1);
            const int buf = it & 1;
            tc::mbar_wait(&accfull[buf], (it >> 1) & 1);
            tc::tc_fence_after();
            const float gbar = __ldg(gb + c);
#pragma unroll
            for (int j = 0; j < N / 32; ++j) {
                float v[32];
                tc::tmem_ld32(trow + buf * N + j * 32, v);
                tc::tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 32; ++i) st[j * 32 + i] = fmaf(gbar, st[j * 32 + i], v[i]);
            }
            tc::tc_fence_before();
            tc::mbar_arrive(&accempty[buf]);
            nst = fmaf(gbar, nst, npart_cur);
            npart_cur = npart_nxt;
        }
        if (!kBwd) emit(NC, true);
        if (et == 0) tc::tma_store_wait_all<0>();
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(tmem, 2 * N);
}

template <bool kBwd, int N>
int launch_impl(const void* a_src, const void* b_src, void* states_out, const ScanArgs& a,
                cudaStream_t st) {
    using namespace tfla_host;
    const Geom& g = a.g;
    CUtensorMap ma, mb, ms;
    if (!make_tmap_bf16_3d(&ma, a_src, g.BH, g.T, g.dqk, 64, 64) ||
        !make_tmap_bf16_3d(&mb, b_src, g.BH, g.T, g.dhv, 64, 64) ||
        !make_tmap_bf16_3d(&ms, states_out, static_cast<uint64_t>(g.BH) * g.NC, g.dqk, g.dhv, 64,
                           128))
        return 4;
    const int smem = ScanSmem<N>::kBytes;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(state_scan_kernel<kBwd, N>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr_set = true;
    }
    dim3 grid(g.dhv / N, (g.dqk + 127) / 128, g.BH);
    state_scan_kernel<kBwd, N><<<grid, 192, smem, st>>>(ma, mb, ms, a);
    return 0;
}

}  // namespace

int launch_state_scan(bool bwd, const void* a_src, const void* b_src, void* states_out,
                      const ScanArgs& a, cudaStream_t st) {
    if (a.ntile == 128) {
        return bwd ? launch_impl<true, 128>(a_src, b_src, states_out, a, st)
                   : launch_impl<false, 128>(a_src, b_src, states_out, a, st);
    }
    return bwd ? launch_impl<true, 64>(a_src, b_src, states_out, a, st)
               : launch_impl<false, 64>(a_src, b_src, states_out, a, st);
}

}  // namespace tfla_k
