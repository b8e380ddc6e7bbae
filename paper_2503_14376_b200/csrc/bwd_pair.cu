// bwd_pair.cu -- K4 (dQ / dK / dV) for chunks of L >= 256 as CTA pairs.
//
// Same math and epilogue as the wide (256-column) persistent kernels of
// bwd_parallel.cu (chunkwise.cpp:454-557 / tiled.cpp:391-779), but two CTAs of
// a cluster own two adjacent 128-row tiles of one chunk and issue every MMA
// as ONE cta_group::2 instruction with M = 256: each CTA holds its 128 rows of
// the A operand and of the TMEM accumulators, and HALF of every B operand
// (the other side's K / Q / V / dH rows, the state tile, the intra operand).
// The B tiles -- the bulk of the split backward's operand traffic: every key
// tile is re-streamed for every query tile -- are therefore fetched and read
// from shared memory once per pair instead of once per CTA, halving their L2
// -> SM bytes and the shared-memory bytes per MAC. The even CTA (rank 0) is
// the MMA issuer; both CTAs' TMA loads complete on its ring barriers, its MMA
// commits arrive on both CTAs' barriers (multicast), and both CTAs' epilogue
// threads arrive on its consumer barriers.
//
// Causality: the pair walks the union of its two tiles' "other" ranges; the
// extra tile of the first (dQ) / second (dK, dV) CTA is fully masked by the
// gating (its D' entries are 0), exactly as in the single-CTA kernel.
// Warps: 0 TMA producer (both CTAs), 1 tcgen05 issuer (rank 0) + TMEM owner,
// 2..9 gating / epilogue (lane quarter warp % 4, column half (warp - 2) / 4).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "bwd_parallel.h"
#include "host_util.h"
#include "stab.cuh"
#include "tc.cuh"

namespace tfla_k {
namespace {

constexpr int kStageA = 128 * 64 * 2;  // 16 KB: own rows (A) of one 64-wide k-block
// 48 KB stages: a score stage carries TWO k-blocks (A 2 x 16 KB + this CTA's
// half of B, 2 x 8 KB), an inter stage one (A 16 + B 16 KB), an intra stage
// two (B 2 x 16 KB) -- the ring keeps 144 KB in flight per SM (the kernels
// are bound by TMA latency over the bytes in flight)
constexpr int kStage = 3 * kStageA;
constexpr int kStages = 3;
constexpr int kG = 128 * 128 * 2;      // stationary gated tile
constexpr int kVecs = 2 * 4 * 128 * 4 + 2 * 128 * 4;
constexpr int kSmemBytes = kStages * kStage + 2 * kG + kVecs + 512;
constexpr int kEpi = 256;
constexpr int kThreads = 64 + kEpi;
constexpr int NO = 256;  // output columns per pair tile
constexpr float kLog2e = 1.4426950408889634f;

struct PPlan {
    int own_start;  // first own row of THIS CTA
    int c_first;    // chunk
    int oth_start;  // first row of other tile 0 (the pair's union)
    int n_oth;
};

template <int KIND>
__device__ __forceinline__ PPlan make_pplan(const Geom& G, int rt0, int rank) {
    PPlan p;
    p.own_start = (rt0 + rank) * 128;
    p.c_first = p.own_start / G.L;
    const int cstart = p.c_first * G.L;
    const int r0 = rt0 * 128 - cstart;  // the pair's first row inside the chunk
    if (KIND == kDQ) {                  // key tiles up to the second tile's diagonal
        p.oth_start = cstart;
        p.n_oth = r0 / 128 + 2;
    } else {                            // query tiles from the first tile's diagonal on
        p.oth_start = rt0 * 128;
        p.n_oth = (G.L - r0) / 128;
    }
    return p;
}

struct PMaps {
    CUtensorMap X, Y, X2, Y2, Z, W, St, Out;
};

template <int KIND>
__global__ void __launch_bounds__(kThreads, 1) bwd_pair_kernel(const __grid_constant__ PMaps M, BwdArgs args) {
    constexpr bool kHasDS = KIND != kDV;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* stages = smem;
    uint8_t* gbuf = smem + kStages * kStage;
    float* vec = reinterpret_cast<float*>(gbuf + 2 * kG);
    float* xred = vec + 2 * 4 * 128;
    uint64_t* bars = reinterpret_cast<uint64_t*>(xred + 2 * 128);
    uint64_t* full = bars;              // [kStages] (rank 0): both CTAs' loads landed
    uint64_t* empty = full + kStages;   // [kStages] (both): MMAs consumed the slot
    uint64_t* sfull = empty + kStages;  // (both)
    uint64_t* sempty = sfull + 1;       // (rank 0): both CTAs' gating read S / dS
    uint64_t* gfull = sempty + 1;       // [2] (rank 0): both gated tiles written
    uint64_t* gempty = gfull + 2;       // [2] (both)
    uint64_t* ofull = gempty + 2;       // (both)
    uint64_t* oempty = ofull + 1;       // (rank 0): both drained
    uint64_t* ifull = oempty + 1;       // (both)
    uint64_t* iscaled = ifull + 1;      // (rank 0): both scaled
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(iscaled + 1);

    const Geom& G = args.g;
    const int warp = tc::warp_id();
    const uint32_t rank = tc::cluster_ctarank();
    const bool leader = rank == 0;
    const int nk_qk = G.dqk / 64, nk_hv = G.dhv / 64;
    const int nk_inter = KIND == kDV ? nk_qk : nk_hv;
    const int dim_out = KIND == kDV ? G.dhv : G.dqk;
    const int ncol = dim_out / NO, npr = G.T / 256;  // pairs of row tiles per head
    const int n_pairs = ncol * npr * G.BH;
    const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
    auto decode = [&](int pt, int& ct, int& rt0, int& bh) {
        ct = pt % ncol;
        rt0 = 2 * ((pt / ncol) % npr);
        bh = pt / (ncol * npr);
    };
    const uint32_t colO = 0, colS = 256, colD = 384;
    auto lead = [&](uint64_t* bar) { return tc::mapa_shared(tc::smem_u32(bar), 0); };

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        tc::mbar_init(sfull, 1);
        tc::mbar_init(sempty, 2 * kEpi);
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&gfull[b], 2 * kEpi);
            tc::mbar_init(&gempty[b], 1);
        }
        tc::mbar_init(ofull, 1);
        tc::mbar_init(oempty, 2 * kEpi);
        tc::mbar_init(ifull, 1);
        tc::mbar_init(iscaled, 2 * kEpi);
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc2(tmem_slot, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::cluster_sync();  // both CTAs' barriers initialised, TMEM allocated
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------ TMA producer (both CTAs)
        if (tc::elect_one()) {
            int gi = 0;
            uint32_t fbar = 0;
            auto acquire = [&](uint32_t bytes) -> uint8_t* {
                const int s = gi % kStages;
                tc::mbar_wait(&empty[s], ((gi / kStages) & 1) ^ 1);
                if (leader) tc::mbar_arrive_expect_tx(&full[s], 2 * bytes);  // both CTAs' bytes
                fbar = lead(&full[s]);
                return stages + s * kStage;
            };
            for (int pt = cluster; pt < n_pairs; pt += nclusters) {
                int ct, rt0, bh;
                decode(pt, ct, rt0, bh);
                const int col0 = ct * NO;
                const PPlan P = make_pplan<KIND>(G, rt0, rank);
                // score stage (two k-blocks): A0 | A1 | B0 (8 KB) | B1 (8 KB)
                auto load_scores = [&](int jt) {
                    const int oth = P.oth_start + jt * 128 + 64 * rank;  // this CTA's half of B
                    for (int kb = 0; kb < nk_qk; kb += 2, ++gi) {
                        uint8_t* st = acquire(2 * (16384 + 8192));
                        for (int h = 0; h < 2; ++h) {
                            tc::tma_load_3d_2sm(st + h * kStageA, &M.X, fbar, (kb + h) * 64, P.own_start, bh);
                            tc::tma_load_3d_2sm(st + 2 * kStageA + h * 8192, &M.Y, fbar, (kb + h) * 64, oth, bh);
                        }
                    }
                    if (kHasDS)
                        for (int kb = 0; kb < nk_hv; kb += 2, ++gi) {
                            uint8_t* st = acquire(2 * (16384 + 8192));
                            for (int h = 0; h < 2; ++h) {
                                tc::tma_load_3d_2sm(st + h * kStageA, &M.X2, fbar, (kb + h) * 64, P.own_start, bh);
                                tc::tma_load_3d_2sm(st + 2 * kStageA + h * 8192, &M.Y2, fbar, (kb + h) * 64, oth, bh);
                            }
                        }
                };
                const int cidx = bh * G.NC + P.c_first;
                load_scores(0);
                for (int kb = 0; kb < nk_inter; ++kb, ++gi) {
                    uint8_t* st = acquire(16384 + 16384);
                    tc::tma_load_3d_2sm(st, &M.W, fbar, kb * 64, P.own_start, bh);
                    if (KIND == kDV) {  // dC [p kblk][x half]: MN-major, two 64-column atoms
                        for (int a = 0; a < 2; ++a)
                            tc::tma_load_3d_2sm(st + kStageA + a * 8192, &M.St, fbar, col0 + 128 * rank + 64 * a,
                                                kb * 64, cidx);
                    } else {            // C / dC [p half][x kblk]: K-major, 128 p rows
                        tc::tma_load_3d_2sm(st + kStageA, &M.St, fbar, kb * 64, col0 + 128 * rank, cidx);
                    }
                }
                for (int jt = 0; jt < P.n_oth; ++jt) {
                    if (jt + 1 < P.n_oth) load_scores(jt + 1);
                    const int oth = P.oth_start + jt * 128;
                    uint8_t* st = acquire(2 * 16384);  // intra B, both 64-row k-blocks
                    for (int kb = 0; kb < 2; ++kb)
                        for (int a = 0; a < 2; ++a)
                            tc::tma_load_3d_2sm(st + kStageA + kb * 16384 + a * 8192, &M.Z, fbar,
                                                col0 + 128 * rank + 64 * a, oth + kb * 64, bh);
                    ++gi;
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ tcgen05 issuer (rank 0)
        if (leader) {
            int gi = 0, u = 0, gu = 0, ti = 0;
            const uint32_t id_s = tc::idesc_bf16(256, 128, 0, 0);
            const uint32_t id_o = tc::idesc_bf16(256, NO, 0, 1);
            const uint32_t id_i = tc::idesc_bf16(256, NO, 0, KIND == kDV ? 1 : 0);
            constexpr uint16_t kBoth = 3;
            auto take = [&]() -> uint32_t {
                const int s = gi % kStages;
                tc::mbar_wait(&full[s], (gi / kStages) & 1);
                tc::tc_fence_after();
                return tc::smem_u32(stages + s * kStage);
            };
            auto gemm_kk = [&](uint32_t dcol, int nkb, bool commit_s) {
                for (int kb = 0; kb < nkb; kb += 2) {  // two k-blocks per stage
                    const uint32_t st = take();
                    if (tc::elect_one()) {
#pragma unroll
                        for (int h = 0; h < 2; ++h)
#pragma unroll
                            for (int ks = 0; ks < 4; ++ks)
                                tc::mma_bf16_2sm(tmem + dcol, tc::kmajor_desc(st + h * kStageA, 128, ks),
                                                 tc::kmajor_desc(st + 2 * kStageA + h * 8192, 64, ks), id_s,
                                                 (kb | h | ks) ? 1u : 0u);
                        tc::mma_commit_2sm(&empty[gi % kStages], kBoth);
                        if (commit_s && kb + 2 >= nkb) tc::mma_commit_2sm(sfull, kBoth);
                    }
                    ++gi;
                    __syncwarp();
                }
            };
            auto mma_scores = [&]() {
                if (u > 0) {
                    tc::mbar_wait_cluster(sempty, (u - 1) & 1);
                    tc::tc_fence_after();
                }
                gemm_kk(colS, nk_qk, !kHasDS);
                if (kHasDS) gemm_kk(colD, nk_hv, true);
                ++u;
            };
            for (int pt = cluster; pt < n_pairs; pt += nclusters, ++ti) {
                int ct, rt0, bh;
                decode(pt, ct, rt0, bh);
                const PPlan P = make_pplan<KIND>(G, rt0, 0);
                mma_scores();
                if (ti > 0) {  // the previous pair tile's O has been drained by both CTAs
                    tc::mbar_wait_cluster(oempty, (ti - 1) & 1);
                    tc::tc_fence_after();
                }
                for (int kb = 0; kb < nk_inter; ++kb) {
                    const uint32_t st = take();
                    if (tc::elect_one()) {
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks) {
                            const uint64_t bd = KIND == kDV ? tc::mnmajor_desc(st + kStageA, 64, ks)
                                                            : tc::kmajor_desc(st + kStageA, 128, ks);
                            tc::mma_bf16_2sm(tmem + colO, tc::kmajor_desc(st, 128, ks), bd, id_i, (kb | ks) ? 1u : 0u);
                        }
                        tc::mma_commit_2sm(&empty[gi % kStages], kBoth);
                        if (kb == nk_inter - 1) tc::mma_commit_2sm(ifull, kBoth);
                    }
                    ++gi;
                    __syncwarp();
                }
                for (int jt = 0; jt < P.n_oth; ++jt) {
                    if (jt + 1 < P.n_oth) mma_scores();
                    const int b = gu & 1;
                    tc::mbar_wait_cluster(&gfull[b], (gu >> 1) & 1);
                    if (jt == 0) tc::mbar_wait_cluster(iscaled, ti & 1);  // intra adds onto the scaled inter
                    tc::tc_fence_after();
                    const uint32_t gb = tc::smem_u32(gbuf + b * kG);
                    {
                        const uint32_t st = take();
                        if (tc::elect_one()) {
#pragma unroll
                            for (int kb = 0; kb < 2; ++kb)
#pragma unroll
                                for (int ks = 0; ks < 4; ++ks)
                                    tc::mma_bf16_2sm(tmem + colO, tc::kmajor_desc(gb, 128, kb * 4 + ks),
                                                     tc::mnmajor_desc(st + kStageA + kb * 16384, 64, ks), id_o, 1u);
                            tc::mma_commit_2sm(&empty[gi % kStages], kBoth);
                            tc::mma_commit_2sm(&gempty[b], kBoth);
                        }
                        ++gi;
                        __syncwarp();
                    }
                    ++gu;
                }
                if (tc::elect_one()) tc::mma_commit_2sm(ofull, kBoth);
                __syncwarp();
            }
        }
    } else {
        // ------------------------------------------------ gating + epilogue (both CTAs)
        const int et = threadIdx.x - 64;
        const int row = (warp & 3) * 32 + tc::lane_id();
        const int half = (warp - 2) >> 2;
        const int T = G.T, L = G.L;
        const bool is_exp = args.variant == 0;
        StabLocal sl;
        const bool stab = is_exp && args.gw.stab != nullptr;
        const float rs = rsqrtf(static_cast<float>(G.dqk));
        const uint32_t trow = tc::tmem_row_addr(tmem);
        const uint32_t l_sempty = lead(sempty), l_oempty = lead(oempty), l_iscaled = lead(iscaled);
        const uint32_t l_gfull0 = lead(&gfull[0]), l_gfull1 = lead(&gfull[1]);
        int u = 0, gu = 0, ti = 0;
        for (int pt = cluster; pt < n_pairs; pt += nclusters, ++ti) {
            int ct, rt0, bh;
            decode(pt, ct, rt0, bh);
            const int col0 = ct * NO;
            const PPlan P = make_pplan<KIND>(G, rt0, rank);
            const size_t hb = static_cast<size_t>(bh) * T;
            const int t_own = P.own_start + row;
            const bool own_ok = t_own < T;
            const int c_own = own_ok ? t_own / L : -1;
            float own_term = 0.f, own_dinv = 0.f;
            if (own_ok) {
                if (KIND == kDQ) {
                    own_term = (is_exp ? args.gw.b[hb + t_own] - args.gw.mc[hb + t_own]
                                       : args.gw.b[hb + t_own]) * kLog2e;
                    own_dinv = args.gw.dinv[hb + t_own];
                } else {
                    own_term = (args.gw.ib[hb + t_own] - args.gw.b[hb + t_own]) * kLog2e;
                }
            }
            float acc_dd = 0.f;
            float scale = 0.f;
            if (own_ok) scale = KIND == kDQ ? args.gw.bb[hb + t_own] : args.gw.ab[hb + t_own];
            float dot = 0.f;
            const __nv_bfloat16* xrow = nullptr;
            if (KIND != kDV && own_ok)
                xrow = (KIND == kDQ ? args.q : args.k) + (hb + t_own) * G.dqk + col0;
            // O holds the bare inter term: scale this thread's half of the row in
            // place and take the gate-partial dot from the unscaled values
            auto scale_inter = [&]() {
                tc::mbar_wait(ifull, ti & 1);
                tc::tc_fence_after();
#pragma unroll 1
                for (int g = half * (NO / 64); g < (half + 1) * (NO / 64); ++g) {
                    float iv[32];
                    tc::tmem_ld32(trow + colO + g * 32, iv);
                    tc::tmem_ld_wait();
                    if (KIND != kDV && xrow) {
#pragma unroll
                        for (int e = 0; e < 32; e += 8) {
                            uint4 raw = *reinterpret_cast<const uint4*>(xrow + g * 32 + e);
                            const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
                            for (int z = 0; z < 4; ++z) {
                                float2 f = __bfloat1622float2(h2[z]);
                                dot = fmaf(f.x, iv[e + 2 * z], dot);
                                dot = fmaf(f.y, iv[e + 2 * z + 1], dot);
                            }
                        }
                    }
                    uint32_t w[32];
#pragma unroll
                    for (int e = 0; e < 32; ++e) w[e] = __float_as_uint(scale * iv[e]);
                    tc::tmem_st32(trow + colO + g * 32, w);
                }
                tc::tmem_st_wait();
                tc::tc_fence_before();
                tc::mbar_arrive_cluster(l_iscaled);
            };
            if (et == 0) tc::tma_store_wait_read<0>();  // the previous tile's store still reads gbuf

            for (int jt = 0; jt < P.n_oth; ++jt, ++u, ++gu) {
                const int b = gu & 1;
                float* vt = vec + (u & 1) * 512;  // [term | dinv | chunk | pos]
                if (et < 128) {
                    const int tu = P.oth_start + jt * 128 + et;
                    const bool ok = tu < T;
                    float term = 0.f, dinv = 0.f;
                    if (ok) {
                        if (KIND == kDQ) {
                            term = (args.gw.ib[hb + tu] - args.gw.b[hb + tu]) * kLog2e;
                        } else {
                            term = (is_exp ? args.gw.b[hb + tu] - args.gw.mc[hb + tu] : args.gw.b[hb + tu]) *
                                   kLog2e;
                            dinv = args.gw.dinv[hb + tu];
                        }
                    }
                    vt[et] = term;
                    vt[128 + et] = dinv;
                    reinterpret_cast<int*>(vt)[256 + et] = ok ? tu / L : -2;
                    reinterpret_cast<int*>(vt)[384 + et] = tu;
                }
                tc::named_bar_sync(1, kEpi);
                tc::mbar_wait(sfull, u & 1);
                tc::tc_fence_after();
                tc::mbar_wait(&gempty[b], ((gu >> 1) & 1) ^ 1);
                uint8_t* gt = gbuf + b * kG;
#pragma unroll 1
                for (int g = 2 * half; g < 2 * half + 2; ++g) {
                    float sv[32], dv[32];
                    tc::tmem_ld32(trow + colS + g * 32, sv);
                    if (kHasDS) tc::tmem_ld32(trow + colD + g * 32, dv);
                    tc::tmem_ld_wait();
                    if (stab) {
#pragma unroll 1
                        for (int uu = g * 32; uu < g * 32 + 32; ++uu) {
                            const int tu = reinterpret_cast<const int*>(vt)[384 + uu];
                            const int cu = reinterpret_cast<const int*>(vt)[256 + uu];
                            if ((KIND == kDQ ? (tu <= t_own) : (t_own <= tu)) && cu == c_own)
                                sl.note(own_term + vt[uu]);
                        }
                    }
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        const int uu = g * 32 + e;
                        const int tu = reinterpret_cast<const int*>(vt)[384 + uu];
                        const int cu = reinterpret_cast<const int*>(vt)[256 + uu];
                        const bool ok = (KIND == kDQ ? (tu <= t_own) : (t_own <= tu)) && cu == c_own;
                        const float arg = fminf(own_term + vt[uu], 0.f);
                        const float dprime = ok ? exp2f(arg) : 0.f;
                        const float dinv_i = KIND == kDQ ? own_dinv : vt[128 + uu];
                        float val;
                        if (KIND == kDV) {
                            val = sv[e] * rs * dprime * dinv_i;
                        } else {
                            const float dsb = dv[e] * dinv_i * dprime;
                            acc_dd = fmaf(dsb, sv[e] * rs, acc_dd);
                            val = dsb * rs;
                        }
                        sv[e] = val;
                    }
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) tc::sw128_store8(gt, row, g * 4 + q4, 128, sv + 8 * q4);
                }
                tc::tc_fence_before();
                tc::mbar_arrive_cluster(l_sempty);
                tc::fence_proxy_async_smem();
                tc::mbar_arrive_cluster(b ? l_gfull1 : l_gfull0);
                if (jt == 0) scale_inter();
            }

            // ---- final epilogue: drain O (inter already scaled in), gate partials
            tc::mbar_wait(ofull, ti & 1);
            tc::tc_fence_after();
            uint8_t* stg = gbuf;
#pragma unroll 1
            for (int g = half * (NO / 64); g < (half + 1) * (NO / 64); ++g) {
                float ov[32];
                tc::tmem_ld32(trow + colO + g * 32, ov);
                tc::tmem_ld_wait();
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) tc::sw128_store8(stg, row, g * 4 + q4, 128, ov + 8 * q4);
            }
            tc::tc_fence_before();
            tc::mbar_arrive_cluster(l_oempty);
            if (KIND != kDV) {
                if (half == 1) {
                    xred[row] = acc_dd;
                    xred[128 + row] = dot;
                }
                tc::named_bar_sync(1, kEpi);
                if (half == 0 && own_ok) {
                    acc_dd += xred[row];
                    dot += xred[128 + row];
                    if (KIND == kDQ) args.dbq_part[hb + t_own] = acc_dd + scale * dot;
                    if (KIND == kDK) {
                        args.da_part[hb + t_own] = scale * dot;
                        args.colsum[hb + t_own] = acc_dd;
                    }
                }
            }
            tc::fence_proxy_async_smem();
            tc::named_bar_sync(1, kEpi);
            if (et == 0) {
                for (int a = 0; a < NO / 64; ++a)
                    tc::tma_store_3d(&M.Out, stg + a * 16384, col0 + 64 * a, P.own_start, bh);
                tc::tma_store_commit();
            }
        }
        if (et == 0) tc::tma_store_wait_all<0>();
        if (stab) sl.flush(args.gw.stab);
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::cluster_sync();  // no peer arrives on / MMAs into this CTA any more
    tc::tc_fence_after();
    if (warp == 1) tc::tmem_dealloc2(tmem, 512);
}

template <int KIND>
int launch_pair(const BwdArgs& a, const BwdTensors& t, cudaStream_t st) {
    using namespace tfla_host;
    const Geom& g = a.g;
    const uint64_t BH = g.BH, T = g.T, NCs = static_cast<uint64_t>(g.BH) * g.NC;
    PMaps m;
    bool ok = true;
    auto own = [&](CUtensorMap* mp, const void* p, int d) { ok &= make_tmap_bf16_3d(mp, p, BH, T, d, 64, 128); };
    auto half = [&](CUtensorMap* mp, const void* p, int d) { ok &= make_tmap_bf16_3d(mp, p, BH, T, d, 64, 64); };
    if (KIND == kDQ) {
        own(&m.X, t.q, g.dqk);
        half(&m.Y, t.k, g.dqk);
        own(&m.X2, t.dh, g.dhv);
        half(&m.Y2, t.v, g.dhv);
        half(&m.Z, t.k, g.dqk);
        own(&m.W, t.dh, g.dhv);
        ok &= make_tmap_bf16_3d(&m.St, t.states, NCs, g.dqk, g.dhv, 64, 128);
        own(&m.Out, t.out, g.dqk);
    } else if (KIND == kDK) {
        own(&m.X, t.k, g.dqk);
        half(&m.Y, t.q, g.dqk);
        own(&m.X2, t.v, g.dhv);
        half(&m.Y2, t.dh, g.dhv);
        half(&m.Z, t.q, g.dqk);
        own(&m.W, t.v, g.dhv);
        ok &= make_tmap_bf16_3d(&m.St, t.states, NCs, g.dqk, g.dhv, 64, 128);
        own(&m.Out, t.out, g.dqk);
    } else {
        own(&m.X, t.k, g.dqk);
        half(&m.Y, t.q, g.dqk);
        m.X2 = m.X;
        m.Y2 = m.Y;
        half(&m.Z, t.dh, g.dhv);
        own(&m.W, t.k, g.dqk);
        ok &= make_tmap_bf16_3d(&m.St, t.states, NCs, g.dqk, g.dhv, 64, 64);
        own(&m.Out, t.out, g.dhv);
    }
    if (!ok) return 4;
    ensure_smem_attr(reinterpret_cast<const void*>(bwd_pair_kernel<KIND>), kSmemBytes);
    const int dim_out = KIND == kDV ? g.dhv : g.dqk;
    const long n_pairs = static_cast<long>(dim_out / NO) * (g.T / 256) * g.BH;
    // clusters of 2 on the SM pairs; cluster count coprime to the (column x
    // pair-in-chunk) period for balanced static striding (see bwd_parallel.cu)
    const int period = (dim_out / NO) * (g.L / 256);
    int ncl = coprime_grid(n_pairs, period) / 2;
    if (ncl < 1) ncl = 1;
    while (ncl > 1 && period > 1) {  // keep the cluster count itself coprime to the period
        int x = ncl, y = period;
        while (y) {
            const int r = x % y;
            x = y;
            y = r;
        }
        if (x == 1) break;
        --ncl;
    }
    if (ncl > n_pairs) ncl = static_cast<int>(n_pairs);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * ncl);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmemBytes;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, bwd_pair_kernel<KIND>, m, a) != cudaSuccess) return 4;
    return 0;
}

}  // namespace

// Measured (7B head shape): no faster than the single-CTA wide kernels at
// L = 256 .. 1024 -- the split backward is bound by its gating epilogue, not
// by B-operand traffic -- and the pair's extra (masked) tile costs up to a
// third more work at L = 256, so it is opt-in (TFLA_PAIR_BWD=1).
bool bwd_pair_supported(const Geom& g) {
    return g.L >= 256 && g.L % 256 == 0 && g.dqk == 256 && g.dhv % 256 == 0 && g.T % 256 == 0 &&
           tfla_host::env_flag("TFLA_PAIR_BWD");
}

int launch_bwd_pair(BwdKind kind, const BwdArgs& a, const BwdTensors& t, cudaStream_t st) {
    switch (kind) {
        case kDQ: return launch_pair<kDQ>(a, t, st);
        case kDK: return launch_pair<kDK>(a, t, st);
        default: return launch_pair<kDV>(a, t, st);
    }
}

}  // namespace tfla_k
