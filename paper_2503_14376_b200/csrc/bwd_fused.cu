// bwd_fused.cu -- K4f: fused TFLA parallel backward for chunk size L = 128.
//
// Same math as bwd_parallel.cu (chunkwise.cpp:454-557 / tiled.cpp:391-779),
// but one persistent CTA per 128-row chunk produces dQ, dK AND dV of that
// chunk: the score tiles S = QK^T and dS = dH V^T are computed once (instead
// of once per output kernel and column tile), gated once into the stationary
// bf16 tiles P' = S D' / (sqrt(d) den) and dP' = dS D' / (sqrt(d) den), and
// every output column tile is then one "group" of two TMEM accumulators
// (intra + inter) filled by tcgen05 while the epilogue drains the previous
// group:
//   dQ[:, p] = dP' K[:, p]              + w  o (dH C_k[p, :]^T)
//   dK[:, p] = dP'^T Q[:, p]            + a_bar o (V dC_{k+1}[p, :]^T)
//   dV[:, x] = P'^T dH[:, x]            + a_bar o (K dC_{k+1}[:, x])
// P'^T / dP'^T are the MN-major views of the same smem tiles. L2 streaming per
// chunk drops from ~3.8 MB (three kernels) to ~2.2 MB and the score GEMMs run
// once instead of 8x / 4x.
// Gate partials: row sums of dD (d_b_i +), column sums of dD (warp
// transpose-reduce; d_b_j -, d_ib_j +), w q.(dH C^T) and a_bar k.(V dC^T).
// Warps: 0 TMA producer, 1 tcgen05 issuer, 2..9 epilogue (lane quarter
// warp % 4, the two warps of a quarter split the columns).
#include <cstdlib>

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "bwd_parallel.h"
#include "host_util.h"
#include "stab.cuh"
#include "tc.cuh"

namespace tfla_k {
namespace {

#ifndef TFLA_BWDF_STAGES
#define TFLA_BWDF_STAGES 4  // 5 fits (csum / xred aliased) but measured the same (1.119 vs 1.118 ms)
#endif
constexpr int kStages = TFLA_BWDF_STAGES;
constexpr int kStageA = 128 * 64 * 2;
constexpr int kStage = 2 * kStageA;
constexpr int kTile = 128 * 128 * 2;
constexpr int kEpi = 256;                      // epilogue threads: 4 lane quarters x kParts (512 measured slower: spills)
constexpr int kParts = kEpi / 128;             // column parts of a 128-column tile per row
constexpr int kPCols = 128 / kParts;           // columns per epilogue thread and tile
constexpr int kThreads = 64 + kEpi;
constexpr int kOffG = kStages * kStage;        // gP | gD
constexpr int kOffVec = kOffG + 2 * kTile;     // colterm[128] | csum[512] (xred[kParts-1][3][128] aliases csum)
// per-epilogue-warp 32-row x 64-column bf16 tile (4 KB, SW128): the TMA-loaded
// q / k rows of a dQ / dK group's gate-partial dot, overwritten in place by the
// group's output rows, which leave by TMA store (coalesced; direct per-thread
// 16-B row stores and loads cost one L1 transaction per row)
constexpr int kOffScr = kOffVec + (128 + 512) * 4 + 512;
constexpr int kScr = 32 * 64 * 2;
constexpr int kSmemBytes = kOffScr + (kEpi / 32) * kScr;
static_assert(kOffScr % 1024 == 0, "SW128 scratch alignment");
static_assert(kSmemBytes <= 232448, "shared memory budget");
static_assert((kParts - 1) * 3 * 128 <= 512, "xred must fit in the csum region it aliases");
constexpr float kLog2e = 1.4426950408889634f;

struct FMaps {
    CUtensorMap Q128, K128, V128, dH128;  // K-major row tiles  (box 64 x 128)
    CUtensorMap Q64, K64, dH64;           // MN-major row tiles (box 64 x 64)
    CUtensorMap C128, dC128, dC64;        // states: K-major [p][x] (64 x 128), MN-major (64 x 64)
    CUtensorMap dQo, dKo, dVo;            // outputs (64 x 32: one epilogue warp's rows)
    CUtensorMap Qr, Kr;                   // q / k rows for the gate-partial dots (64 x 32)
};

__global__ void __launch_bounds__(kThreads, 1) bwd_fused_kernel(const __grid_constant__ FMaps M, BwdArgs args) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* stages = smem;
    uint8_t* gP = smem + kOffG;
    uint8_t* gD = gP + kTile;
    float* colterm = reinterpret_cast<float*>(smem + kOffVec);
    float* csum = colterm + 128;  // [4 * kParts warps][kPCols]
    float* xred = csum;           // [kParts - 1][3][128]: the partial sums at the tile end reuse csum
    uint64_t* bars = reinterpret_cast<uint64_t*>(csum + 512);
    uint64_t* full = bars;
    uint64_t* empty = full + kStages;
    uint64_t* sfull = empty + kStages;
    uint64_t* ofull = sfull + 1;   // [2]
    uint64_t* sfree = ofull + 2;   // [2] slot drained by the epilogue
    uint64_t* gfull = sfree + 2;
    uint64_t* gempty = gfull + 1;
    uint64_t* lbar = gempty + 1;   // [kEpi / 32] per-warp scratch loads
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(lbar + kEpi / 32);

    const Geom& G = args.g;
    const int T = G.T, NC = G.NC;
    const int npt = G.dqk / 128, nxt = G.dhv / 128;
    const int nkq = G.dqk / 64, nkv = G.dhv / 64;
    const int ngroups = 2 * npt + nxt;
    const int n_tiles = G.BH * NC;
    const int warp = tc::warp_id();

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        tc::mbar_init(sfull, 1);
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&ofull[b], 1);
            tc::mbar_init(&sfree[b], kEpi);
        }
        tc::mbar_init(gfull, kEpi);
        tc::mbar_init(gempty, 1);
        for (int w = 0; w < kEpi / 32; ++w) tc::mbar_init(&lbar[w], 1);
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // group q of a tile: kind (0 dQ, 1 dK, 2 dV) and column tile; slot = (q + 1) & 1
    auto group_kind = [&](int q, int& kind, int& ct) {
        if (q < npt) {
            kind = 0;
            ct = q;
        } else if (q < 2 * npt) {
            kind = 1;
            ct = q - npt;
        } else {
            kind = 2;
            ct = q - 2 * npt;
        }
    };

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (tc::elect_one()) {
            int gi = 0;
            auto acquire = [&](uint32_t bytes) -> uint8_t* {
                const int s = gi % kStages;
                if (args.trace && blockIdx.x == 0 && gi < 512) args.trace[gi * 4 + 0] = clock64();
                tc::mbar_wait(&empty[s], ((gi / kStages) & 1) ^ 1);
                if (args.trace && blockIdx.x == 0 && gi < 512) args.trace[gi * 4 + 1] = clock64();
                tc::mbar_arrive_expect_tx(&full[s], bytes);
                return stages + s * kStage;
            };
            auto bar = [&]() { return &full[gi % kStages]; };
            // L2 policy: the chunk's q/k/v/dH tiles are re-read by several jobs
            // of this CTA (keep), the state tiles are read once here (stream)
            const uint64_t keep = tc::policy_evict_last(), stream = tc::policy_evict_first();
            for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
                const int bh = tile / NC, c = tile % NC, r0 = c * 128;
                for (int kb = 0; kb < nkq; ++kb, ++gi) {
                    uint8_t* st = acquire(2 * kStageA);
                    tc::tma_load_3d_hint(st, &M.Q128, bar(), kb * 64, r0, bh, keep);
                    tc::tma_load_3d_hint(st + kStageA, &M.K128, bar(), kb * 64, r0, bh, keep);
                }
                for (int kb = 0; kb < nkv; ++kb, ++gi) {
                    uint8_t* st = acquire(2 * kStageA);
                    tc::tma_load_3d_hint(st, &M.dH128, bar(), kb * 64, r0, bh, keep);
                    tc::tma_load_3d_hint(st + kStageA, &M.V128, bar(), kb * 64, r0, bh, keep);
                }
                for (int q = 0; q < ngroups; ++q) {
                    int kind, ct;
                    group_kind(q, kind, ct);
                    const int cidx = bh * NC + c;
                    if (kind == 0 || kind == 1) {  // inter: A = dH | V rows, B = C | dC [p tile][x kblk]
                        for (int kb = 0; kb < nkv; ++kb, ++gi) {
                            uint8_t* st = acquire(2 * kStageA);
                            // last use of V (dK group of the last p tile): stream
                            const uint64_t pa = (kind == 1 && ct == npt - 1 && (args.l2mode & 4)) ? stream : keep;
                            tc::tma_load_3d_hint(st, kind == 0 ? &M.dH128 : &M.V128, bar(), kb * 64, r0, bh, pa);
                            tc::tma_load_3d_hint(st + kStageA, kind == 0 ? &M.C128 : &M.dC128, bar(), kb * 64, ct * 128,
                                                 cidx, kind == 0 ? stream : keep);
                        }
                    } else {  // inter: A = K rows [p kblk], B = dC [p kblk][x tile] MN-major
                        for (int kb = 0; kb < nkq; ++kb, ++gi) {
                            uint8_t* st = acquire(2 * kStageA);
                            // last use of K (dV group of the last x tile): stream
                            tc::tma_load_3d_hint(st, &M.K128, bar(), kb * 64, r0, bh,
                                                 (ct == nxt - 1 && (args.l2mode & 2)) ? stream : keep);
                            for (int a = 0; a < 2; ++a)
                                tc::tma_load_3d_hint(st + kStageA + a * 8192, &M.dC64, bar(), ct * 128 + 64 * a, kb * 64,
                                                     cidx, stream);
                        }
                    }
                    // intra: B = K | Q | dH [row kblk][col tile] MN-major, both 64-row
                    // blocks in one stage (a full 32 KB slot instead of two half-empty ones)
                    const CUtensorMap* z = kind == 0 ? &M.K64 : kind == 1 ? &M.Q64 : &M.dH64;
                    // the dK / dV intra operands (Q, dH column tiles) are their last use
                    const uint64_t pz = ((kind == 1 && (args.l2mode & 1)) || (kind == 2 && (args.l2mode & 8))) ? stream : keep;
                    {
                        uint8_t* st = acquire(2 * kStageA);
                        for (int kb = 0; kb < 2; ++kb)
                            for (int a = 0; a < 2; ++a)
                                tc::tma_load_3d_hint(st + kb * kStageA + a * 8192, z, bar(), ct * 128 + 64 * a,
                                                     r0 + kb * 64, bh, pz);
                        ++gi;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ tcgen05 issuer
        int gi = 0, ti = 0, use0 = 0, use1 = 0;
        const uint32_t id_kk = tc::idesc_bf16(128, 128, 0, 0);
        const uint32_t id_kn = tc::idesc_bf16(128, 128, 0, 1);
        auto take = [&]() -> uint32_t {
            const int s = gi % kStages;
            if (args.trace && blockIdx.x == 0 && gi < 512 && tc::lane_id() == 0) args.trace[gi * 4 + 2] = clock64();
            tc::mbar_wait(&full[s], (gi / kStages) & 1);
            if (args.trace && blockIdx.x == 0 && gi < 512 && tc::lane_id() == 0) args.trace[gi * 4 + 3] = clock64();
            tc::tc_fence_after();
            return tc::smem_u32(stages + s * kStage);
        };
        auto acquire_slot = [&](int slot) {
            int& u = slot ? use1 : use0;
            tc::mbar_wait(&sfree[slot], (u & 1) ^ 1);
            ++u;
            tc::tc_fence_after();
        };
        auto gemm = [&](uint32_t dcol, int nkb, bool b_mn, bool first_acc_zero) {
            for (int kb = 0; kb < nkb; ++kb) {
                const uint32_t st = take();
                if (tc::elect_one()) {
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks) {
                        const uint64_t bd = b_mn ? tc::mnmajor_desc(st + kStageA, 64, ks)
                                                 : tc::kmajor_desc(st + kStageA, 128, ks);
                        tc::mma_bf16(tmem + dcol, tc::kmajor_desc(st, 128, ks), bd, b_mn ? id_kn : id_kk,
                                     (first_acc_zero && (kb | ks) == 0) ? 0u : 1u);
                    }
                    tc::mma_commit(&empty[gi % kStages]);
                }
                ++gi;
                __syncwarp();
            }
        };
        for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++ti) {
            // scores into slot 0: S at [0,128), dS at [128,256)
            acquire_slot(0);
            gemm(0, nkq, false, true);
            gemm(128, nkv, false, true);
            if (tc::elect_one()) tc::mma_commit(sfull);
            __syncwarp();
            for (int q = 0; q < ngroups; ++q) {
                int kind, ct;
                group_kind(q, kind, ct);
                const int slot = (q + 1) & 1;
                const uint32_t base = slot * 256;
                acquire_slot(slot);
                // inter (independent of the gating) -> [base + 128, base + 256)
                gemm(base + 128, kind == 2 ? nkq : nkv, kind == 2, true);
                if (q == 0) {
                    tc::mbar_wait(gfull, ti & 1);
                    tc::tc_fence_after();
                }
                // intra: A = dP' (dQ, K-major) | dP'^T (dK, MN-major) | P'^T (dV, MN-major)
                const uint32_t ga = tc::smem_u32(kind == 2 ? gP : gD);
                {
                    const uint32_t st = take();
                    if (tc::elect_one()) {
                        const uint32_t idesc = tc::idesc_bf16(128, 128, kind == 0 ? 0 : 1, 1);
#pragma unroll
                        for (int kb = 0; kb < 2; ++kb)
#pragma unroll
                            for (int ks = 0; ks < 4; ++ks) {
                                const uint64_t ad = kind == 0 ? tc::kmajor_desc(ga, 128, kb * 4 + ks)
                                                              : tc::mnmajor_desc(ga, 128, kb * 4 + ks);
                                tc::mma_bf16(tmem + base, ad, tc::mnmajor_desc(st + kb * kStageA, 64, ks), idesc,
                                             (kb | ks) ? 1u : 0u);
                            }
                        tc::mma_commit(&empty[gi % kStages]);
                        tc::mma_commit(&ofull[slot]);
                        if (q == ngroups - 1) tc::mma_commit(gempty);
                    }
                    ++gi;
                    __syncwarp();
                }
            }
        }
    } else {
        // ------------------------------------------------ gating + epilogue
        const int et = threadIdx.x - 64;
        const int lane = tc::lane_id();
        const int row = (warp & 3) * 32 + lane;
        const int part = (warp - 2) >> 2;  // columns [part * kPCols, +kPCols) of each tile
        const bool is_exp = args.variant == 0;
        const float rs = rsqrtf(static_cast<float>(G.dqk));
        const uint32_t trow = tc::tmem_row_addr(tmem);
        int ti = 0, use0 = 0, use1 = 0, of0 = 0, of1 = 0, lph = 0;
        uint8_t* scr = smem + kOffScr + (warp - 2) * kScr;
        const uint64_t out_policy = tc::policy_evict_first();
        uint64_t* mylbar = &lbar[warp - 2];
        const int rq = (warp & 3) * 32;  // this warp's rows within the tile
        // lane 0: once the scratch's previous TMA store has read it, load the q / k
        // rows of group q of `tile` (dQ / dK groups only)
        auto issue_rows = [&](int tile_, int q_) {
            if (tile_ >= n_tiles) return;
            int kind_, ct_;
            group_kind(q_, kind_, ct_);
            if (kind_ == 2 || lane != 0) return;
            const int bh_ = tile_ / NC, r0_ = (tile_ % NC) * 128;
            tc::tma_store_wait_read<0>();
            tc::mbar_arrive_expect_tx(mylbar, kScr);
            tc::tma_load_3d(scr, kind_ == 0 ? &M.Qr : &M.Kr, mylbar, ct_ * 128 + part * kPCols, r0_ + rq, bh_);
        };
        issue_rows(blockIdx.x, 0);
        // debug trace (CTA 0, thread et 0, first 64 tiles): [0] tile start, [1] scores
        // ready, [2] gating done, [3 + 3q] group q TMEM ready, [4 + 3q] rows landed,
        // [5 + 3q] group q stored
        const bool etr = args.trace && blockIdx.x == 0 && et == 0;
#define ETRACE(e) \
    do { if (etr && ti < 64) args.trace[2048 + ti * 32 + (e)] = clock64(); } while (0)
        StabLocal sl;
        const bool stab = is_exp && args.gw.stab != nullptr;
        auto release_slot = [&](int slot) {
            tc::tc_fence_before();
            tc::mbar_arrive(&sfree[slot]);
            (slot ? use1 : use0)++;
        };
        for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++ti) {
            const int bh = tile / NC, c = tile % NC, r0 = c * 128;
            const size_t hb = static_cast<size_t>(bh) * T;
            const size_t t = hb + r0 + row;
            const float b_i = args.gw.b[t];
            const float rowterm = (is_exp ? b_i - args.gw.mc[t] : b_i) * kLog2e;
            const float dinv = args.gw.dinv[t];
            const float w_i = args.gw.bb[t];
            const float ab_i = args.gw.ab[t];
            if (et < 128) colterm[et] = (args.gw.ib[hb + r0 + et] - args.gw.b[hb + r0 + et]) * kLog2e;
            ETRACE(0);
            tc::named_bar_sync(1, kEpi);

            // ---- gating: P' and dP' from S and dS; row / column sums of dD
            tc::mbar_wait(sfull, ti & 1);
            tc::tc_fence_after();
            tc::mbar_wait(gempty, (ti & 1) ^ 1);
            ETRACE(1);
            float rowsum = 0.f;
#pragma unroll 1
            for (int g = part * (kPCols / 32); g < (part + 1) * (kPCols / 32); ++g) {
                float sv[32], dv[32];
                tc::tmem_ld32(trow + g * 32, sv);
                tc::tmem_ld32(trow + 128 + g * 32, dv);
                tc::tmem_ld_wait();
                if (stab)
                    for (int j = g * 32; j < g * 32 + 32 && j <= row; ++j) sl.note(rowterm + colterm[j]);
                float dd[32];
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    const int j = g * 32 + e;
                    const float dp = j <= row ? exp2f(fminf(rowterm + colterm[j], 0.f)) * dinv : 0.f;
                    const float s = sv[e] * rs;
                    const float dsb = dv[e] * dp;  // dS_bar * D' (with 1/den)
                    dd[e] = dsb * s;
                    rowsum += dd[e];
                    sv[e] = s * dp;    // P'
                    dv[e] = dsb * rs;  // dP'
                }
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                    tc::sw128_store8(gP, row, g * 4 + q4, 128, sv + 8 * q4);
                    tc::sw128_store8(gD, row, g * 4 + q4, 128, dv + 8 * q4);
                }
                // column sums over this warp's 32 rows: transpose-reduce, lane l <- column g*32 + l
#pragma unroll
                for (int k = 16; k >= 1; k >>= 1) {
                    const bool up = lane & k;
#pragma unroll
                    for (int i = 0; i < k; ++i) {
                        const float send = up ? dd[i] : dd[i + k];
                        const float keep = up ? dd[i + k] : dd[i];
                        dd[i] = keep + __shfl_xor_sync(0xffffffffu, send, k);
                    }
                }
                csum[(warp - 2) * kPCols + (g - part * (kPCols / 32)) * 32 + lane] = dd[0];
            }
            release_slot(0);
            tc::fence_proxy_async_smem();
            tc::mbar_arrive(gfull);
            ETRACE(2);
            tc::named_bar_sync(1, kEpi);
            float colsum = 0.f;
            if (et < 128) {
                const int hj = et / kPCols;
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) colsum += csum[(4 * hj + q4) * kPCols + (et % kPCols)];
            }
            tc::named_bar_sync(1, kEpi);  // csum read: the tile-end partial sums (xred) may reuse it

            // ---- groups: out = intra + scale * inter; gate-partial dots
            float dot_q = 0.f, dot_k = 0.f;
            for (int q = 0; q < ngroups; ++q) {
                int kind, ct;
                group_kind(q, kind, ct);
                const int slot = (q + 1) & 1;
                int& of = slot ? of1 : of0;
                tc::mbar_wait(&ofull[slot], of & 1);
                ++of;
                tc::tc_fence_after();
                ETRACE(3 + 3 * q);
                const float scale = kind == 0 ? w_i : ab_i;
                if (kind != 2) {  // q / k rows landed in the scratch
                    tc::mbar_wait(mylbar, lph & 1);
                    ++lph;
                } else {  // the scratch's previous store must have read it
                    if (lane == 0) tc::tma_store_wait_read<0>();
                    __syncwarp();
                }
                ETRACE(4 + 3 * q);
                uint8_t* my = scr + lane * 128;
#pragma unroll 1
                for (int h2i = 0; h2i < kPCols / 32; ++h2i) {
                    float ov[32], iv[32];
                    tc::tmem_ld32(trow + slot * 256 + part * kPCols + h2i * 32, ov);
                    tc::tmem_ld32(trow + slot * 256 + 128 + part * kPCols + h2i * 32, iv);
                    tc::tmem_ld_wait();
                    if (kind != 2) {  // q.(dH C^T) (dQ) / k.(V dC^T) (dK) over this column chunk
                        float d = 0.f;
#pragma unroll
                        for (int e = 0; e < 32; e += 8) {
                            const int cc = h2i * 4 + e / 8;
                            const uint4 raw = *reinterpret_cast<const uint4*>(my + ((cc ^ (lane & 7)) << 4));
                            const __nv_bfloat162* hh = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
                            for (int z = 0; z < 4; ++z) {
                                const float2 f = __bfloat1622float2(hh[z]);
                                d = fmaf(f.x, iv[e + 2 * z], d);
                                d = fmaf(f.y, iv[e + 2 * z + 1], d);
                            }
                        }
                        if (kind == 0) dot_q += d; else dot_k += d;
                    }
#pragma unroll
                    for (int e = 0; e < 32; ++e) ov[e] = fmaf(scale, iv[e], ov[e]);
                    if (h2i == kPCols / 32 - 1) release_slot(slot);  // all of this thread's TMEM columns read
#pragma unroll
                    for (int q8 = 0; q8 < 4; ++q8) {
                        uint4 w;
                        w.x = tc::pack_bf16(ov[8 * q8], ov[8 * q8 + 1]);
                        w.y = tc::pack_bf16(ov[8 * q8 + 2], ov[8 * q8 + 3]);
                        w.z = tc::pack_bf16(ov[8 * q8 + 4], ov[8 * q8 + 5]);
                        w.w = tc::pack_bf16(ov[8 * q8 + 6], ov[8 * q8 + 7]);
                        *reinterpret_cast<uint4*>(my + (((h2i * 4 + q8) ^ (lane & 7)) << 4)) = w;
                    }
                }
                tc::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    const CUtensorMap* om = kind == 0 ? &M.dQo : kind == 1 ? &M.dKo : &M.dVo;
                    // evict-first: the outputs must not push the tile's kept q/k/v/dH rows
                    // (re-read by the later groups) out of L2
                    tc::tma_store_3d_hint(om, scr, ct * 128 + part * kPCols, r0 + rq, bh, out_policy);
                    tc::tma_store_commit();
                }
                if (q + 1 < ngroups) issue_rows(tile, q + 1);
                else issue_rows(tile + gridDim.x, 0);
                ETRACE(5 + 3 * q);
            }
            // ---- gate partials (one p-tile slot: n_ptile = 1 for the fused path)
            if (part > 0) {
                float* xr3 = xred + (part - 1) * 384;
                xr3[row] = rowsum;
                xr3[128 + row] = dot_q;
                xr3[256 + row] = dot_k;
            }
            tc::named_bar_sync(1, kEpi);
            if (part == 0) {
#pragma unroll
                for (int pp = 0; pp < kParts - 1; ++pp) {
                    rowsum += xred[pp * 384 + row];
                    dot_q += xred[pp * 384 + 128 + row];
                    dot_k += xred[pp * 384 + 256 + row];
                }
                args.dbq_part[t] = rowsum + w_i * dot_q;
                if (args.iq_part) args.iq_part[t] = w_i * dot_q;
                args.da_part[t] = ab_i * dot_k;
            }
            if (et < 128) args.colsum[hb + r0 + et] = colsum;
            tc::named_bar_sync(1, kEpi);
        }
        if (lane == 0) tc::tma_store_wait_all<0>();
        if (stab) sl.flush(args.gw.stab);
#undef ETRACE
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

}  // namespace

bool bwd_fused_supported(const Geom& g) {
    return g.L == 128 && g.dqk % 128 == 0 && g.dhv % 128 == 0 && g.dqk <= 512;
}

int launch_bwd_fused(const BwdArgs& a, const BwdTensors& t, void* dq, void* dk, void* dv,
                     const void* c_states, const void* dc_states, cudaStream_t st) {
    using namespace tfla_host;
    const Geom& g = a.g;
    const uint64_t BH = g.BH, T = g.T, NCs = static_cast<uint64_t>(g.BH) * g.NC;
    FMaps m;
    bool ok = true;
    ok &= make_tmap_bf16_3d(&m.Q128, t.q, BH, T, g.dqk, 64, 128);
    ok &= make_tmap_bf16_3d(&m.K128, t.k, BH, T, g.dqk, 64, 128);
    ok &= make_tmap_bf16_3d(&m.V128, t.v, BH, T, g.dhv, 64, 128);
    ok &= make_tmap_bf16_3d(&m.dH128, t.dh, BH, T, g.dhv, 64, 128);
    ok &= make_tmap_bf16_3d(&m.Q64, t.q, BH, T, g.dqk, 64, 64);
    ok &= make_tmap_bf16_3d(&m.K64, t.k, BH, T, g.dqk, 64, 64);
    ok &= make_tmap_bf16_3d(&m.dH64, t.dh, BH, T, g.dhv, 64, 64);
    ok &= make_tmap_bf16_3d(&m.C128, c_states, NCs, g.dqk, g.dhv, 64, 128);
    ok &= make_tmap_bf16_3d(&m.dC128, dc_states, NCs, g.dqk, g.dhv, 64, 128);
    ok &= make_tmap_bf16_3d(&m.dC64, dc_states, NCs, g.dqk, g.dhv, 64, 64);
    ok &= make_tmap_bf16_3d(&m.dQo, dq, BH, T, g.dqk, 64, 32);
    ok &= make_tmap_bf16_3d(&m.dKo, dk, BH, T, g.dqk, 64, 32);
    ok &= make_tmap_bf16_3d(&m.dVo, dv, BH, T, g.dhv, 64, 32);
    ok &= make_tmap_bf16_3d(&m.Qr, t.q, BH, T, g.dqk, 64, 32);
    ok &= make_tmap_bf16_3d(&m.Kr, t.k, BH, T, g.dqk, 64, 32);
    if (!ok) return 4;
    tfla_host::ensure_smem_attr(reinterpret_cast<const void*>(bwd_fused_kernel), kSmemBytes);
    const int num_sms = tfla_host::num_sms();
    const int n_tiles = g.BH * g.NC;
    BwdArgs aa = a;
    static const int l2mode = [] {
        const char* e = std::getenv("TFLA_BWDF_L2");
        return e ? std::atoi(e) : 15;
    }();
    aa.l2mode = l2mode;
    aa.dq = static_cast<__nv_bfloat16*>(dq);
    aa.dk = static_cast<__nv_bfloat16*>(dk);
    aa.dv = static_cast<__nv_bfloat16*>(dv);
    bwd_fused_kernel<<<n_tiles < num_sms ? n_tiles : num_sms, kThreads, kSmemBytes, st>>>(m, aa);
    return 0;
}

}  // namespace tfla_k
