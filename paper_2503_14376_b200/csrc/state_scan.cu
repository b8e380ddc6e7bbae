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
// CTA = (x tile of N columns of d_hv, p tile of 128 rows of d_qk, head).
// Warp roles: warp 0 = TMA producer, warp 1 = tcgen05 issuer (+TMEM owner),
// warps 2..9 = transform / epilogue (256 threads; TMEM lane quarter warp%4, and
// the two warps sharing a quarter split the N columns).
// Per chunk: TMA streams 64-row k-blocks of A (MN-major, M = p) and B (MN-major,
// N = x) into a ring; the epilogue warps scale the B rows by w in shared memory
// (the gate sits on the contraction dim, so it must be applied to an operand);
// the MMA warp accumulates D_k = A^T diag(w) B into one of kNB TMEM buffers; the
// epilogue folds D_k into the fp32 register-resident state while the next
// chunks' MMAs run, and streams the state out as bf16 (double-buffered TMA
// store) for the parallel kernels. The backward's d_g needs C_k: its bf16 tile
// is TMA-prefetched by the producer into a double buffer.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "host_util.h"
#include "kernels.h"
#include "tc.cuh"

namespace tfla_k {
namespace {

#ifndef TFLA_SCAN_DEEP_BWD_STAGES
#define TFLA_SCAN_DEEP_BWD_STAGES 3
#endif
#ifndef TFLA_SCAN_DEEP_NCB
#define TFLA_SCAN_DEEP_NCB 4
#endif
constexpr int kNB = 4;               // TMEM D buffers
constexpr int kEpi = 256;            // transform (128) + update (128) threads
constexpr int kTr = 128;             // transform threads
constexpr int kUp = 128;             // update / emit threads
constexpr int kThreads = 64 + kEpi;

// N = 64 runs two CTAs per SM (two independent chunk chains per SM hide the
// per-chunk TMA / MMA / epilogue latency); N = 128 runs one.
// kDeep (grids of at most one CTA per SM, e.g. the long-context config's 128
// chains): one CTA per SM with an 8-stage ring -- the scan is bound by TMA
// latency over the bytes a CTA keeps in flight (stage interval = (latency +
// transform + MMA) / stages, profiles/r02_scan_traces.txt), and a grid that
// cannot fill two CTAs per SM gains nothing from the 2-CTA smem split.
// kR: rows (tokens) per stage. The TMA engine's rate is per box, not per byte,
// up to ~70 B/cycle/SM (profiles/r02_ubench_tma.txt: one issuer streams an
// L2-resident 64x64 box in ~230 cycles, a 64x128 box in about the same), so
// 128-row stages double the ingest ceiling wherever the smem fits them.
template <bool kBwd, int N, bool kDeep = false, int kR = 64>
struct ScanSmem {
    static constexpr int kMinBlocks = (N <= 64 && !kDeep) ? 2 : 1;
    // deep backward: 3 stages so that 4 C_k tiles fit -- the C_k prefetch (2
    // chunks ahead, still ~0.8k cycles of wait per chunk), not the stage ring,
    // bounded its chunk interval at long context: bwd scan 0.635 -> 0.55 ms
    // (3 tiles: 0.571); a second staging tile for the deep forward: no change
    static constexpr int kStages = kR == 128 ? (kDeep ? (kBwd ? TFLA_SCAN_DEEP_BWD_STAGES : 4) : 2)
                                             : (kDeep ? 8 : (kBwd ? 3 : 4));
    static constexpr int kAStage = 128 * kR * 2;  // 2 MN atoms of 64 p x kR rows
    // bwd, N = 64: the two C_k tiles double as the emit staging (the d_g dot
    // consumes C_k before the state tile is written over it), so C_{k+2} is
    // prefetched two chunks ahead in the smem a separate staging tile took:
    // the C_k TMA latency under load (~3.8k cycles, profiles/r02_scan_traces.txt)
    // no longer stalls the update warps every chunk
    static constexpr bool kShare = kBwd && N <= 64;
    static constexpr int kNSt = kShare ? 0 : (N <= 64 ? 1 : 2);  // staging buffers
    static constexpr int kNCb = kBwd ? ((kShare && kDeep && kR == 128) ? TFLA_SCAN_DEEP_NCB : 2) : 0;  // C_k tiles (bwd d_g)
    static constexpr int kBStage = N * kR * 2;
    static constexpr int kStage = kAStage + kBStage;
    static constexpr int kTile = 128 * N * 2;  // one bf16 state tile
    static constexpr int kOffStaging = kStages * kStage;
    static constexpr int kOffC = kOffStaging + kNSt * kTile;
    static constexpr int kOffVec = kOffC + kNCb * kTile;
    static constexpr int kBytes = kOffVec + 64 + 448;  // red[16], barriers
    static_assert(kBytes * kMinBlocks <= 232448 - 1024 * (kMinBlocks - 1), "shared memory budget");
};

template <bool kBwd, int N, bool kDeep, int kR>
__global__ void __launch_bounds__(kThreads, ScanSmem<kBwd, N, kDeep, kR>::kMinBlocks)
    state_scan_kernel(const __grid_constant__ CUtensorMap mapA,
                      const __grid_constant__ CUtensorMap mapB,
                      const __grid_constant__ CUtensorMap mapS,
                      const __grid_constant__ CUtensorMap mapC,
                      const __grid_constant__ CUtensorMap mapAs, ScanArgs args, int ncl) {
    using SM = ScanSmem<kBwd, N, kDeep, kR>;
    constexpr int kStages = SM::kStages;
    constexpr int kAStage = SM::kAStage;
    constexpr int kAtom = kR * 128;  // one 64-column MN atom of a stage
    constexpr int kNCbM = SM::kNCb > 0 ? SM::kNCb : 1;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* stages = smem;
    uint8_t* staging = smem + SM::kOffStaging;  // [kNSt][kTile]
    uint8_t* cbuf = smem + SM::kOffC;           // [kNCb][kTile] (bwd)
    float* red = reinterpret_cast<float*>(smem + SM::kOffVec);  // [16]
    uint64_t* bars = reinterpret_cast<uint64_t*>(red + 16);
    uint64_t* full = bars;
    uint64_t* tfull = full + kStages;
    uint64_t* empty = tfull + kStages;
    uint64_t* accfull = empty + kStages;   // [kNB]
    uint64_t* accempty = accfull + kNB;    // [kNB]
    uint64_t* cfull = accempty + kNB;      // [kNCbM] (>= 2)
    uint64_t* sready = cfull + 4;          // [kNCbM] (bwd, shared staging) staged state tile written
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sready + 4);

    const Geom& G = args.g;
    const int T = G.T, L = G.L, NC = G.NC, dqk = G.dqk, dhv = G.dhv;
    const int xt = blockIdx.x, pt = blockIdx.y, bh = blockIdx.z;
    const int x0 = xt * N, p0 = pt * 128;
    const int nA = (dqk - p0) >= 128 ? 2 : 1;
    const int nkb = L / kR;
    const int total = NC * nkb;
    const int warp = tc::warp_id();
    const bool tracing = args.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0;
#define TRACE_ST(gi, e) \
    do { if (tracing && (gi) < 256) args.trace[(gi) * 4 + (e)] = clock64(); } while (0)
#define TRACE_CH(it, e) \
    do { if (tracing && (it) < 128) args.trace[1024 + (it) * 8 + (e)] = clock64(); } while (0)

    if (threadIdx.x == 0) {
        if (tc::smem_u32(smem) & 1023) __trap();
        for (int s = 0; s < kStages; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&tfull[s], kTr);
            tc::mbar_init(&empty[s], ncl);  // every cluster CTA's MMAs release the slot
        }
        for (int b = 0; b < kNB; ++b) {
            tc::mbar_init(&accfull[b], 1);
            tc::mbar_init(&accempty[b], kUp);
        }
        for (int b = 0; b < 4; ++b) {
            tc::mbar_init(&cfull[b], 1);
            tc::mbar_init(&sready[b], kUp);
        }
        tc::fence_barrier_init();
    }
    if (nA == 1) {  // d_qk tail: the second MN atom of A is never loaded -> zeros
        for (int i = threadIdx.x; i < kStages * kAtom / 16; i += blockDim.x) {
            const int s = i / (kAtom / 16), u = i % (kAtom / 16);
            reinterpret_cast<uint4*>(stages + s * SM::kStage + kAtom)[u] = make_uint4(0, 0, 0, 0);
        }
        tc::fence_proxy_async_smem();
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, kNB * N);
    tc::tc_fence_before();
    __syncthreads();
    if (ncl > 1) tc::cluster_sync();  // peers' barriers initialised before any multicast
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint16_t mc_mask = static_cast<uint16_t>((1u << ncl) - 1u);

    const bool do_dg = kBwd && args.dg_part != nullptr;
    // (bwd) TMA prefetch of the bf16 C tile of processing step `it` for d_g
    // (bwd) d_g partials are optional: the fused backward can derive d_g from its
    // own per-token partials instead (tfla_bwd.cpp), so the C tiles are not read
    auto issue_c = [&](int it) {
        if (!do_dg || it >= NC) return;
        const int c = NC - 1 - it;
        const int b = it % kNCbM;
        tc::mbar_arrive_expect_tx(&cfull[b], SM::kTile);
        for (int a = 0; a < (N + 63) / 64; ++a)
            tc::tma_load_3d(cbuf + b * SM::kTile + a * 16384, &mapC, &cfull[b], x0 + 64 * a, p0, bh * NC + c);
    };

    if (warp == 0 && SM::kShare && tc::lane_id() == 31) {
        // ------------------------------------------------ (bwd, shared staging) store helper
        // The update warps write the state tile over the C_k tile they just dotted
        // and arrive on sready; this lane stores it, sums the d_g partial and, once
        // the store has read the tile, refills it with C_{k-2} (or just frees it).
        // The update warps never wait for a store or a named barrier.
        for (int i = 0; i < kNCbM; ++i) {
            if (do_dg) issue_c(i);
            else tc::mbar_arrive(&cfull[i]);
        }
        for (int it = 0; it < NC; ++it) {
            const int b = it % kNCbM, c = NC - 1 - it;
            tc::mbar_wait(&sready[b], (it / kNCbM) & 1);
            uint8_t* stg = cbuf + b * SM::kTile;
            for (int a = 0; a < (N + 63) / 64; ++a) tc::tma_store_3d(&mapS, stg + a * 16384, x0 + 64 * a, p0, bh * NC + c);
            tc::tma_store_commit();
            if (do_dg) {
                const float sum = red[4 * b] + red[4 * b + 1] + red[4 * b + 2] + red[4 * b + 3];
                const int ntiles = gridDim.x * gridDim.y;
                args.dg_part[(static_cast<size_t>(bh) * NC + c) * ntiles + pt * gridDim.x + xt] = sum;
            }
            tc::tma_store_wait_read<0>();
            if (it + kNCbM < NC) {
                if (do_dg) issue_c(it + kNCbM);
                else tc::mbar_arrive(&cfull[b]);
            }
        }
        tc::tma_store_wait_all<0>();
    } else if (warp == 0) {
        // ------------------------------------------------ TMA producer
        // (lane 0, not elect.sync: lane 31 may be on the helper path)
        if (tc::lane_id() == 0) {
            const uint32_t bytes = nA * kAtom + N * kR * 2;
            for (int gi = 0; gi < total; ++gi) {
                const int it = gi / nkb, kb = gi % nkb;
                const int c = kBwd ? NC - 1 - it : it;
                const int row = c * L + kb * kR;
                const int s = gi % kStages;
                tc::mbar_wait(&empty[s], ((gi / kStages) & 1) ^ 1);
                TRACE_ST(gi, 0);
                uint8_t* sa = stages + s * SM::kStage;
                uint8_t* sb = sa + kAStage;
                tc::mbar_arrive_expect_tx(&full[s], bytes);
                if (ncl > 1) {  // this CTA's 64/ncl-row slice of A, multicast to the cluster
                    const int rr = kR / ncl, r0 = static_cast<int>(tc::cluster_ctarank()) * rr;
                    for (int a = 0; a < nA; ++a)
                        tc::tma_load_3d_mc(sa + a * kAtom + r0 * 128, &mapAs, &full[s], p0 + 64 * a, row + r0, bh,
                                           mc_mask);
                } else {
                    for (int a = 0; a < nA; ++a)
                        tc::tma_load_3d(sa + a * kAtom, &mapA, &full[s], p0 + 64 * a, row, bh);
                }
                for (int a = 0; a < (N + 63) / 64; ++a)
                    tc::tma_load_3d(sb + a * kAtom, &mapB, &full[s], x0 + 64 * a, row, bh);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ tcgen05 issuer
        const uint32_t idesc = tc::idesc_bf16(128, N, 1, 1);
        for (int it = 0; it < NC; ++it) {
            const int buf = it % kNB;
            tc::mbar_wait(&accempty[buf], ((it / kNB) & 1) ^ 1);
            tc::tc_fence_after();
            for (int kb = 0; kb < nkb; ++kb) {
                const int gi = it * nkb + kb;
                const int s = gi % kStages;
                tc::mbar_wait(&tfull[s], (gi / kStages) & 1);
                TRACE_ST(gi, 3);
                tc::tc_fence_after();
                const uint32_t sa = tc::smem_u32(stages + s * SM::kStage);
                const uint32_t sb = sa + kAStage;
                if (tc::elect_one()) {
#pragma unroll
                    for (int ks = 0; ks < kR / 16; ++ks)
                        tc::mma_bf16(tmem + buf * N, tc::mnmajor_desc(sa, kR, ks),
                                     N == 32 ? tc::mnmajor_desc_sw64(sb, kR, ks) : tc::mnmajor_desc(sb, kR, ks),
                                     idesc, (kb | ks) ? 1u : 0u);
                    if (ncl > 1) tc::mma_commit_mc(&empty[s], mc_mask);
                    else tc::mma_commit(&empty[s]);
                    if (kb == nkb - 1) tc::mma_commit(&accfull[buf]);
                }
                __syncwarp();
            }
        }
    } else if (warp < 6) {
        // ------------------------------------------------ transform warps 2..5
        // Scale the B rows of every landed stage by w (the gate sits on the
        // contraction dim); (fwd, x tile 0) accumulate n partials sum_j w_j k_j[p].
        // Decoupled from the update warps so transforms (and therefore the
        // MMAs) run ahead as far as the stage ring allows.
        const int tt = threadIdx.x - 64;  // 0..127
        // n increments u_k = K_k^T a_bar are split across the x tiles: this CTA
        // sums rows r = xt (mod n_xtiles) of each 64-row k-block
        const bool do_n = !kBwd && args.u_part != nullptr;
        const int nxt = gridDim.x;
        const bool p_ok = tt < dqk - p0;
        const float* wv = args.w + static_cast<size_t>(bh) * T;
        constexpr int kU = SM::kBStage / 16 / kTr;
        constexpr int kCh = N < 64 ? N / 8 : 8;  // 16-B chunks per B-atom row (the row factor ignores the swizzle)
        constexpr int kM = kR / 8;  // n-partial rows per stage for n_xtiles = 8
        float wnext[kU];
        auto load_w = [&](int gi) {
            if (gi >= total) return;
            const int it2 = gi / nkb, kb2 = gi % nkb;
            const int c2 = kBwd ? NC - 1 - it2 : it2;
            const float* wk2 = wv + c2 * L + kb2 * kR;
#pragma unroll
            for (int q = 0; q < kU; ++q) wnext[q] = __ldg(wk2 + (((tt + q * kTr) / kCh) % kR));
        };
        // n-partial gate values for the next stage (rows xt + 8 m: the 7B-shape
        // case n_xtiles = 8, unrolled; other n_xtiles take the generic loop)
        float nwn[kM];
        auto load_nw = [&](int gi) {
            if (!do_n || nxt != 8 || gi >= total) return;
            const int it2 = gi / nkb, kb2 = gi % nkb;
            const int c2 = kBwd ? NC - 1 - it2 : it2;
            const float* wk2 = wv + c2 * L + kb2 * kR + xt;
#pragma unroll
            for (int m = 0; m < kM; ++m) nwn[m] = __ldg(wk2 + 8 * m);
        };
        load_w(0);
        load_nw(0);
        float np = 0.f;
        for (int gi = 0; gi < total; ++gi) {
            const int it = gi / nkb, kb = gi % nkb;
            const int c = kBwd ? NC - 1 - it : it;
            const int s = gi % kStages;
            const float* wk = wv + c * L + kb * kR;
            float wpre[kU];
#pragma unroll
            for (int q = 0; q < kU; ++q) wpre[q] = wnext[q];
            load_w(gi + 1);
            float nw[kM];
#pragma unroll
            for (int m = 0; m < kM; ++m) nw[m] = nwn[m];
            load_nw(gi + 1);
            tc::mbar_wait(&full[s], (gi / kStages) & 1);
            if (tt == 0) TRACE_ST(gi, 1);
            uint8_t* sa = stages + s * SM::kStage;
            uint8_t* sb = sa + kAStage;
            // all loads first, then the math, then the stores (the compiler cannot
            // reorder a load past a possibly aliasing shared store)
            uint4 val[kU];
            uint4* ptr[kU];
#pragma unroll
            for (int q = 0; q < kU; ++q) {
                const int u = tt + q * kTr;
                const int atom = u / (kR * kCh), r = (u / kCh) % kR, ch = u % kCh;
                ptr[q] = reinterpret_cast<uint4*>(sb + atom * kAtom + r * (kCh * 16) + ch * 16);
                val[q] = *ptr[q];
            }
#pragma unroll
            for (int q = 0; q < kU; ++q) {
                const float wr = wpre[q];
                __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&val[q]);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    float2 f = __bfloat1622float2(h2[e]);
                    h2[e] = __floats2bfloat162_rn(f.x * wr, f.y * wr);
                }
            }
#pragma unroll
            for (int q = 0; q < kU; ++q) *ptr[q] = val[q];
            if (do_n && p_ok && nxt == 8) {  // 8 independent loads, then the FMAs
                const int atom = tt >> 6, pc = tt & 63;
                const __nv_bfloat16* a16 = reinterpret_cast<const __nv_bfloat16*>(sa + atom * kAtom);
                float av[kM];
#pragma unroll
                for (int m = 0; m < kM; ++m) {
                    const int r = xt + 8 * m;  // r & 7 == xt
                    av[m] = __bfloat162float(a16[r * 64 + ((((pc >> 3) ^ xt) << 3) | (pc & 7))]);
                }
#pragma unroll
                for (int m = 0; m < kM; ++m) np = fmaf(nw[m], av[m], np);
            } else if (do_n && p_ok) {
                const int atom = tt >> 6, pc = tt & 63;
                const __nv_bfloat16* a16 = reinterpret_cast<const __nv_bfloat16*>(sa + atom * kAtom);
                for (int r = xt; r < kR; r += nxt) {
                    const int off = r * 64 + ((((pc >> 3) ^ (r & 7)) << 3) | (pc & 7));
                    np = fmaf(__ldg(wk + r), __bfloat162float(a16[off]), np);
                }
            }
            tc::fence_proxy_async_smem();
            tc::mbar_arrive(&tfull[s]);
            if (tt == 0) TRACE_ST(gi, 2);
            if (do_n && kb == nkb - 1) {  // partial u_c for this x tile (summed by nscan_kernel)
                if (p_ok) args.u_part[((static_cast<size_t>(bh) * NC + c) * nxt + xt) * dqk + p0 + tt] = np;
                np = 0.f;
            }
        }
    } else {
        // ------------------------------------------------ update / emit warps 6..9
        const int ut = threadIdx.x - 192;                  // 0..127
        const int row = (warp & 3) * 32 + tc::lane_id();   // TMEM lane == p within tile
        const bool row_ok = row < dqk - p0;
        const float* gb = args.gbar + static_cast<size_t>(bh) * NC;
        const uint32_t trow = tc::tmem_row_addr(tmem);

        float st[N];
#pragma unroll
        for (int i = 0; i < N; ++i) st[i] = 0.f;
        if (!kBwd && args.c_init && row_ok) {  // initial state C_0 (fwd)
            const float* src = args.c_init + (static_cast<size_t>(bh) * dqk + p0 + row) * dhv + x0;
#pragma unroll
            for (int i = 0; i < N; i += 4) {
                const float4 v4 = *reinterpret_cast<const float4*>(src + i);
                st[i] = v4.x, st[i + 1] = v4.y, st[i + 2] = v4.z, st[i + 3] = v4.w;
            }
        }

        // Emit the incoming state of chunk c: bf16 operand copy (TMA store),
        // optional fp32 reference-layout states, n, and (bwd) the d_g partial.
        auto emit = [&](int it, int c, bool final_state) {
            if (!kBwd && args.c_states && row_ok) {
                float* dst = args.c_states + ((static_cast<size_t>(bh) * (NC + 1) + c) * dqk + p0 + row) * dhv + x0;
#pragma unroll
                for (int i = 0; i < N; i += 4)
                    *reinterpret_cast<float4*>(dst + i) = make_float4(st[i], st[i + 1], st[i + 2], st[i + 3]);
            }
            if (kBwd && args.dc_states && row_ok) {  // st = dC_{c+1} (c = -1: dC_0)
                float* dst = args.dc_states + ((static_cast<size_t>(bh) * (NC + 1) + c + 1) * dqk + p0 + row) * dhv + x0;
#pragma unroll
                for (int i = 0; i < N; i += 4)
                    *reinterpret_cast<float4*>(dst + i) = make_float4(st[i], st[i + 1], st[i + 2], st[i + 3]);
            }
            if (!kBwd && final_state && args.c_final && row_ok) {
                float* dst = args.c_final + (static_cast<size_t>(bh) * dqk + p0 + row) * dhv + x0;
#pragma unroll
                for (int i = 0; i < N; i += 4)
                    *reinterpret_cast<float4*>(dst + i) = make_float4(st[i], st[i + 1], st[i + 2], st[i + 3]);
            }
            if (final_state) return;
            // shared staging: the tile holds C_k (d_g) or has been freed by the helper
            if (SM::kShare && !do_dg) tc::mbar_wait(&cfull[it % kNCbM], (it / kNCbM) & 1);
            if (do_dg) {
                tc::mbar_wait(&cfull[it % kNCbM], (it / kNCbM) & 1);
                if (ut == 0) TRACE_CH(it, 4);
                const uint8_t* ct = cbuf + (it % kNCbM) * SM::kTile;
                float acc = 0.f;
#pragma unroll
                for (int cc = 0; cc < N / 8; ++cc) {  // 16-B chunk index along the row
                    const int atom = cc >> 3, chunk = (cc & 7) ^ (row & 7);
                    const uint4 raw = *reinterpret_cast<const uint4*>(
                        N == 32 ? ct + tc::sw64_chunk(row, cc) : ct + atom * 16384 + row * 128 + chunk * 16);
                    const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        float2 f = __bfloat1622float2(h2[e]);
                        acc = fmaf(f.x, st[cc * 8 + 2 * e], acc);
                        acc = fmaf(f.y, st[cc * 8 + 2 * e + 1], acc);
                    }
                }
                if (!row_ok) acc = 0.f;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                if (tc::lane_id() == 0) red[(SM::kShare ? 4 * (it % kNCbM) : 0) + warp - 6] = acc;
            }
            if (ut == 0) TRACE_CH(it, 5);
            if (SM::kShare) {  // each thread overwrites only the row it just dotted
                uint8_t* stg = cbuf + (it % kNCbM) * SM::kTile;
#pragma unroll
                for (int c8 = 0; c8 < N / 8; ++c8) {
                    if (N == 32) tc::sw64_store8(stg, row, c8, st + 8 * c8);
                    else tc::sw128_store8(stg, row, c8, 128, st + 8 * c8);
                }
                tc::fence_proxy_async_smem();
                tc::mbar_arrive(&sready[it % kNCbM]);
                if (ut == 0) TRACE_CH(it, 7);
                return;
            }
            uint8_t* stg = staging + (it % (SM::kNSt > 0 ? SM::kNSt : 1)) * SM::kTile;
            if (ut == 0) tc::tma_store_wait_read<(SM::kNSt > 0 ? SM::kNSt - 1 : 0)>();
            tc::named_bar_sync(1, kUp);  // every thread is past its C_c reads
            if (ut == 0) TRACE_CH(it, 6);
            if (do_dg && ut == 0) {
                const float s = red[0] + red[1] + red[2] + red[3];
                const int ntiles = gridDim.x * gridDim.y;
                args.dg_part[(static_cast<size_t>(bh) * NC + c) * ntiles + pt * gridDim.x + xt] = s;
                issue_c(it + SM::kNCb);  // refill this buffer for step it + kNCb
            }
#pragma unroll
            for (int c8 = 0; c8 < N / 8; ++c8) {
                if (N == 32) tc::sw64_store8(stg, row, c8, st + 8 * c8);
                else tc::sw128_store8(stg, row, c8, 128, st + 8 * c8);
            }
            tc::fence_proxy_async_smem();
            tc::named_bar_sync(1, kUp);
            if (ut == 0) TRACE_CH(it, 7);
            if (ut == 0) {
                for (int a = 0; a < (N + 63) / 64; ++a)
                    tc::tma_store_3d(&mapS, stg + a * 16384, x0 + 64 * a, p0, bh * NC + c);
                tc::tma_store_commit();
            }
        };

        if (!SM::kShare && do_dg && ut == 0)
            for (int i = 0; i < SM::kNCb; ++i) issue_c(i);
        for (int it = 0; it < NC; ++it) {
            const int c = kBwd ? NC - 1 - it : it;
            if (ut == 0) TRACE_CH(it, 0);
            emit(it, c, false);
            if (ut == 0) TRACE_CH(it, 1);
            const int buf = it % kNB;
            tc::mbar_wait(&accfull[buf], (it / kNB) & 1);
            if (ut == 0) TRACE_CH(it, 2);
            tc::tc_fence_after();
            const float gbar = __ldg(gb + c);
#pragma unroll
            for (int j = 0; j < N / 16; ++j) {  // 16-column pieces: the state row stays in registers
                float v[16];
                tc::tmem_ld16(trow + buf * N + j * 16, v);
                tc::tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 16; ++i) st[j * 16 + i] = fmaf(gbar, st[j * 16 + i], v[i]);
            }
            tc::tc_fence_before();
            tc::mbar_arrive(&accempty[buf]);
            if (ut == 0) TRACE_CH(it, 3);
        }
        if (!kBwd) emit(NC, NC, true);
        else if (args.dc_states) emit(NC, -1, true);
        if (ut == 0) tc::tma_store_wait_all<0>();
    }
    tc::tc_fence_before();
    __syncthreads();
    if (ncl > 1) tc::cluster_sync();  // no peer multicast / release still in flight
    if (warp == 1) tc::tmem_dealloc(tmem, kNB * N);
#undef TRACE_ST
#undef TRACE_CH
}

template <bool kBwd, int N, bool kDeep, int kR>
int launch_impl(const void* a_src, const void* b_src, void* states_out, const ScanArgs& a,
                cudaStream_t st) {
    using namespace tfla_host;
    const Geom& g = a.g;
    CUtensorMap ma, mb, ms, mc;
    const uint64_t nstate = static_cast<uint64_t>(g.BH) * g.NC;
    // N = 32: B, state and C_k tiles are 32-column boxes in the 64-byte swizzle
    const bool ok = N == 32 ? (make_tmap_bf16_3d(&ma, a_src, g.BH, g.T, g.dqk, 64, kR) &&
                               make_tmap_bf16_3d_sw64(&mb, b_src, g.BH, g.T, g.dhv, kR) &&
                               make_tmap_bf16_3d_sw64(&ms, states_out, nstate, g.dqk, g.dhv, 128))
                            : (make_tmap_bf16_3d(&ma, a_src, g.BH, g.T, g.dqk, 64, kR) &&
                               make_tmap_bf16_3d(&mb, b_src, g.BH, g.T, g.dhv, 64, kR) &&
                               make_tmap_bf16_3d(&ms, states_out, nstate, g.dqk, g.dhv, 64, 128));
    if (!ok) return 4;
    if (kBwd && a.dg_part) {
        if (!(N == 32 ? make_tmap_bf16_3d_sw64(&mc, a.c_saved, nstate, g.dqk, g.dhv, 128)
                      : make_tmap_bf16_3d(&mc, a.c_saved, nstate, g.dqk, g.dhv, 64, 128)))
            return 4;
    } else {
        mc = ms;
    }
    // A (K or Q rows) is the same for every x tile of a (p tile, head): with
    // TFLA_SCAN_MC the x tiles form one cluster and each loads a 64/ncl-row
    // slice of A, multicast to all of them (one L2 read instead of ncl)
    const int nxt = g.dhv / N;
    const int ncl = (nxt == 2 || nxt == 4 || nxt == 8) && env_flag("TFLA_SCAN_MC") ? nxt : 1;
    CUtensorMap mas = ma;
    if (ncl > 1 && !make_tmap_bf16_3d(&mas, a_src, g.BH, g.T, g.dqk, 64, kR / ncl)) return 4;
    const int smem = ScanSmem<kBwd, N, kDeep, kR>::kBytes;
    tfla_host::ensure_smem_attr(reinterpret_cast<const void*>(state_scan_kernel<kBwd, N, kDeep, kR>), smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nxt, (g.dqk + 127) / 128, g.BH);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute cl[1];
    cl[0].id = cudaLaunchAttributeClusterDimension;
    cl[0].val.clusterDim.x = ncl;
    cl[0].val.clusterDim.y = 1;
    cl[0].val.clusterDim.z = 1;
    cfg.attrs = cl;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, state_scan_kernel<kBwd, N, kDeep, kR>, ma, mb, ms, mc, mas, a, ncl) != cudaSuccess)
        return 4;
    return 0;
}

// n_{k+1} = gbar_k n_k + sum_xt u_part[k][xt] (the normaliser recurrence of
// chunkwise.cpp:53-65, with u_k = K_k^T a_bar computed by K1's transform
// warps). The chunk axis is split into kSeg segments per d_qk entry: each
// segment composes its affine maps n -> A n + B (pass 1), one thread per
// entry chains the kSeg segment maps, and pass 2 replays every segment from
// its true start value -- so the sequential depth is NC / kSeg + kSeg instead
// of NC (long sequences: 512 chunks at S = 65536, L = 128).
constexpr int kSeg = 32;

__global__ void nscan_kernel(const float* __restrict__ u_part, const float* __restrict__ gbar,
                             float* __restrict__ n_states, float* __restrict__ n_final, int NC, int dqk,
                             int nxt, const float* __restrict__ n_init) {
    __shared__ float segA[kSeg][32], segB[kSeg][32], start[kSeg][32];
    const int bh = blockIdx.y, pl = threadIdx.x & 31, seg = threadIdx.x >> 5;
    const int p = blockIdx.x * 32 + pl;
    const bool ok = p < dqk;
    const int per = (NC + kSeg - 1) / kSeg;
    const int k0 = seg * per, k1 = min(NC, k0 + per);
    const float* g = gbar + static_cast<size_t>(bh) * NC;
    auto inc = [&](int k) {
        const float* u = u_part + (static_cast<size_t>(bh) * NC + k) * nxt * dqk + p;
        float s = 0.f;
        for (int x = 0; x < nxt; ++x) s += __ldg(u + x * dqk);
        return s;
    };
    // the segment's increments, loaded in blocks of kB with every load in flight
    // before the dependent FMA chain, and kept in registers for pass 2
    constexpr int kB = 16;
    float incs[kB];
    float A = 1.f, B = 0.f;
    const bool fits = k1 - k0 <= kB;
    if (ok)
        for (int kb0 = k0; kb0 < k1; kb0 += kB) {
#pragma unroll
            for (int j = 0; j < kB; ++j) incs[j] = kb0 + j < k1 ? inc(kb0 + j) : 0.f;
#pragma unroll
            for (int j = 0; j < kB; ++j)
                if (kb0 + j < k1) {
                    const float gk = __ldg(g + kb0 + j);
                    A *= gk;
                    B = fmaf(gk, B, incs[j]);
                }
        }
    segA[seg][pl] = A;
    segB[seg][pl] = B;
    __syncthreads();
    if (seg == 0) {
        float n = (ok && n_init) ? n_init[static_cast<size_t>(bh) * dqk + p] : 0.f;
        for (int s2 = 0; s2 < kSeg; ++s2) {
            start[s2][pl] = n;
            n = fmaf(segA[s2][pl], n, segB[s2][pl]);
        }
    }
    __syncthreads();
    if (!ok) return;
    float* out = n_states + static_cast<size_t>(bh) * (NC + 1) * dqk + p;
    if (seg == 0) out[0] = n_init ? n_init[static_cast<size_t>(bh) * dqk + p] : 0.f;
    float n = start[seg][pl];
    for (int kb0 = k0; kb0 < k1; kb0 += kB) {
        if (!fits) {
#pragma unroll
            for (int j = 0; j < kB; ++j) incs[j] = kb0 + j < k1 ? inc(kb0 + j) : 0.f;
        }
#pragma unroll
        for (int j = 0; j < kB; ++j)
            if (kb0 + j < k1) {
                n = fmaf(__ldg(g + kb0 + j), n, incs[j]);
                out[static_cast<size_t>(kb0 + j + 1) * dqk] = n;
            }
    }
    if (n_final && k1 == NC && k0 < k1) n_final[static_cast<size_t>(bh) * dqk + p] = n;
}

}  // namespace

int launch_state_scan_impl(bool bwd, const void* a_src, const void* b_src, void* states_out,
                           const ScanArgs& a, cudaStream_t st);

void launch_nscan(const Geom& g, const float* u_part, const float* gbar, float* n_states, float* n_final,
                  int n_xtiles, cudaStream_t st, const float* n_init) {
    nscan_kernel<<<dim3((g.dqk + 31) / 32, g.BH), 32 * kSeg, 0, st>>>(u_part, gbar, n_states, n_final, g.NC,
                                                                         g.dqk, n_xtiles, n_init);
}

int launch_state_scan(bool bwd, const void* a_src, const void* b_src, void* states_out,
                      const ScanArgs& a0, cudaStream_t st) {
    // debug: TFLA_TRACE_SCAN=<file> (+ TFLA_TRACE_SCAN_DIR=bwd) dumps CTA (0,0,0)'s
    // per-stage (producer / transform in / transform out / MMA) and per-chunk
    // (emit start / emit end / acc ready / folded) clock64 events
    ScanArgs a = a0;
    const char* tf = getenv("TFLA_TRACE_SCAN");
    const char* td = getenv("TFLA_TRACE_SCAN_DIR");
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cap);
    const bool want = tf && *tf && ((td && td[0] == 'b') == bwd) && cap == cudaStreamCaptureStatusNone;
    if (want) {
        cudaMalloc(&a.trace, 2048 * sizeof(long long));
        cudaMemsetAsync(a.trace, 0, 2048 * sizeof(long long), st);
    }
    int rc = launch_state_scan_impl(bwd, a_src, b_src, states_out, a, st);
    if (want) {
        long long h[2048];
        cudaMemcpyAsync(h, a.trace, sizeof(h), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        cudaFree(a.trace);
        if (FILE* f = fopen(tf, "w")) {
            for (int i = 0; i < 256; ++i) fprintf(f, "%lld %lld %lld %lld\n", h[4 * i], h[4 * i + 1], h[4 * i + 2], h[4 * i + 3]);
            for (int i = 0; i < 128; ++i) {
                for (int e = 0; e < 8; ++e) fprintf(f, "%lld%c", h[1024 + 8 * i + e], e == 7 ? '\n' : ' ');
            }
            fclose(f);
        }
    }
    return rc;
}

// 32-column tiles (opt-in, TFLA_SCAN32=1): twice the chains of a grid of at
// most one 64-column CTA per SM, two per SM. Parity-tested, measured slower at
// the long-context shape (fwd 0.50 -> 0.68, bwd 0.64 -> 0.70 ms): the chains
// are TMA-latency bound per chunk and the q / k p-tile (the A operand, 32 KB
// per chunk) is the same size for either width, so two CTAs per SM double the
// L2 -> SM bytes of A while each chain's chunk interval grows (1.9k -> 2.6k
// cycles); the deep 64-column ring stays the default.
int scan_ntile_for(const Geom& g) {
    const long ctas64 = static_cast<long>(g.dhv / 64) * ((g.dqk + 127) / 128) * g.BH;
    if (g.dhv % 64 == 0 && ctas64 <= tfla_host::num_sms() && tfla_host::env_flag("TFLA_SCAN32")) return 32;
    return 64;
}

int launch_state_scan_impl(bool bwd, const void* a_src, const void* b_src, void* states_out,
                           const ScanArgs& a, cudaStream_t st) {
    if (a.ntile == 32) {  // grids of at most one 64-column CTA per SM (long context): two 32-column CTAs per SM
        const bool r128 = a.g.L % 128 == 0 && !bwd && !tfla_host::env_flag("TFLA_SCAN_R64");
        if (r128) return launch_impl<false, 32, false, 128>(a_src, b_src, states_out, a, st);
        return bwd ? launch_impl<true, 32, false, 64>(a_src, b_src, states_out, a, st)
                   : launch_impl<false, 32, false, 64>(a_src, b_src, states_out, a, st);
    }
    if (a.ntile == 128) {
        return bwd ? launch_impl<true, 128, false, 64>(a_src, b_src, states_out, a, st)
                   : launch_impl<false, 128, false, 64>(a_src, b_src, states_out, a, st);
    }
    // 128-row stages (chunk sizes that are multiples of 128) everywhere but the
    // 2-CTA backward, whose C_k tiles leave no room for two 48 KB stages
    // (long context: fwd 0.68 -> 0.49 ms, bwd 0.69 -> 0.63 ms at L = 128,
    // L = 256 fwd / bwd 0.62 -> 0.45 / 0.42 ms; profiles/r02_scan_rows.txt)
    const bool r128 = a.g.L % 128 == 0 && !tfla_host::env_flag("TFLA_SCAN_R64");
    const long ctas = static_cast<long>(a.g.dhv / 64) * ((a.g.dqk + 127) / 128) * a.g.BH;
    if (ctas <= tfla_host::num_sms() && !tfla_host::env_flag("TFLA_NO_DEEP_SCAN")) {
        if (r128)
            return bwd ? launch_impl<true, 64, true, 128>(a_src, b_src, states_out, a, st)
                       : launch_impl<false, 64, true, 128>(a_src, b_src, states_out, a, st);
        return bwd ? launch_impl<true, 64, true, 64>(a_src, b_src, states_out, a, st)
                   : launch_impl<false, 64, true, 64>(a_src, b_src, states_out, a, st);
    }
    if (!bwd && r128) return launch_impl<false, 64, false, 128>(a_src, b_src, states_out, a, st);
    return bwd ? launch_impl<true, 64, false, 64>(a_src, b_src, states_out, a, st)
               : launch_impl<false, 64, false, 64>(a_src, b_src, states_out, a, st);
}

}  // namespace tfla_k
