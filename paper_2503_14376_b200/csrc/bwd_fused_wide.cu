// bwd_fused_wide.cu -- K4f with 256-column output groups (L = 128, d_qk = 256,
// d_hv % 256 == 0).
//
// Same math as bwd_fused.cu (chunkwise.cpp:454-557): one persistent CTA per
// 128-row chunk computes the score tiles S = QK^T and dS = dH V^T once, gates
// them into the stationary bf16 tiles P' / dP' (shared memory), and produces
//   dQ = dP' K + w o (dH C_k^T),   dK = dP'^T Q + a_bar o (V dC_{k+1}^T),
//   dV = P'^T dH + a_bar o (K dC_{k+1}),
// but every output group is 256 columns wide (dQ, dK: all of d_qk; dV: one
// half of d_hv each) instead of 128. The measured bound of the 128-column
// kernel is shared-memory bandwidth (an SS tcgen05 MMA with N = 128 reads 8
// KB of operands per 64 cycles = the whole 128 B/clk port); an
// N = 256 MMA reads 12 KB per 128 cycles, and the state tiles (B of the inter
// terms) are fetched and read once per 256 columns. TMEM then holds one
// 256-column accumulator per group (two slots), so the inter term goes in
// FIRST and the epilogue scales its rows by w / a_bar in place (taking the
// gate-partial dots from the unscaled values), then the intra MMAs accumulate
// on top -- the row scale is applied without a second accumulator.
//
// Order (ngroups = 2 + d_hv / 256; group g lives in TMEM slot (g + 1) & 1,
// slot 0 first holds S | dS):
//   MMA:       S, dS | inter(0) | inter(1) | intra(0) | inter(2) | intra(1) | ... | intra(n-1)
//   epilogue:  gating | scale(0) | scale(1) | drain(0) | scale(2) | drain(1) | ... | drain(n-1)
// so the next group's inter term runs on the tensor core while the epilogue
// scales / drains the previous one.
// Warps: 0 TMA producer, 1 tcgen05 issuer, 2..9 epilogue (lane quarter warp % 4,
// column half (warp - 2) / 4).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "bwd_parallel.h"
#include "host_util.h"
#include "stab.cuh"
#include "tc.cuh"

namespace tfla_k {
namespace {

constexpr int kStages = 3;
constexpr int kStageA = 128 * 64 * 2;          // 16 KB
constexpr int kStage = 3 * kStageA;            // 48 KB: A 16 KB + B up to 32 KB
constexpr int kTile = 128 * 128 * 2;           // gated bf16 tile (P' or dP')
constexpr int kEpi = 256;
constexpr int kThreads = 64 + kEpi;
constexpr int kOffG = kStages * kStage;        // gP | gD
constexpr int kOffVec = kOffG + 2 * kTile;     // colterm[128] | csum[512] | xred[3][128]
constexpr int kSmemBytes = kOffVec + (128 + 512 + 3 * 128) * 4 + 512;
constexpr float kLog2e = 1.4426950408889634f;

struct WMaps {
    CUtensorMap Q128, K128, V128, dH128;  // K-major row tiles (box 64 x 128)
    CUtensorMap K64, Q64, dH64;           // MN-major row tiles (box 64 x 64)
    CUtensorMap C128, dC128, dC64;        // states: K-major [p][x] (64 x 128), MN-major (64 x 64)
};

__global__ void __launch_bounds__(kThreads, 1) bwd_fused_wide_kernel(const __grid_constant__ WMaps M, BwdArgs args) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* stages = smem;
    uint8_t* gP = smem + kOffG;
    uint8_t* gD = gP + kTile;
    float* colterm = reinterpret_cast<float*>(smem + kOffVec);
    float* csum = colterm + 128;  // [8 warps][64]
    float* xred = csum + 512;     // [3][128]
    uint64_t* bars = reinterpret_cast<uint64_t*>(xred + 3 * 128);
    uint64_t* full = bars;
    uint64_t* empty = full + kStages;
    uint64_t* sfull = empty + kStages;  // S, dS accumulated
    uint64_t* ifull = sfull + 1;        // [2] inter term of the slot's group accumulated
    uint64_t* iscaled = ifull + 2;      // [2] ... and row-scaled by the epilogue
    uint64_t* ofull = iscaled + 2;      // [2] group complete
    uint64_t* sfree = ofull + 2;        // [2] slot read out (slot 0 also: S / dS read by the gating)
    uint64_t* gfull = sfree + 2;        // P', dP' written
    uint64_t* gempty = gfull + 1;       // P', dP' consumed by the chunk's last intra MMA
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gempty + 1);

    const Geom& G = args.g;
    const int T = G.T, NC = G.NC;
    const int nkq = G.dqk / 64, nkv = G.dhv / 64;  // nkq == 4
    const int ngroups = 2 + G.dhv / 256;
    const int n_tiles = G.BH * NC;
    const int warp = tc::warp_id();

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        tc::mbar_init(sfull, 1);
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&ifull[b], 1);
            tc::mbar_init(&iscaled[b], kEpi);
            tc::mbar_init(&ofull[b], 1);
            tc::mbar_init(&sfree[b], kEpi);
        }
        tc::mbar_init(gfull, kEpi);
        tc::mbar_init(gempty, 1);
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // group g: kind (0 dQ, 1 dK, 2 dV) and the 256-column tile of its output
    auto group_kind = [&](int g, int& kind, int& ct) {
        kind = g < 2 ? g : 2;
        ct = g < 2 ? 0 : g - 2;
    };

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (tc::elect_one()) {
            int gi = 0;
            auto acquire = [&](uint32_t bytes) -> uint8_t* {
                const int s = gi % kStages;
                tc::mbar_wait(&empty[s], ((gi / kStages) & 1) ^ 1);
                tc::mbar_arrive_expect_tx(&full[s], bytes);
                return stages + s * kStage;
            };
            auto bar = [&]() { return &full[gi % kStages]; };
            const uint64_t keep = tc::policy_evict_last(), stream = tc::policy_evict_first();
            auto load_inter = [&](int g, int bh, int r0, int cidx) {
                int kind, ct;
                group_kind(g, kind, ct);
                if (kind < 2) {  // A = dH | V rows [kblk], B = C | dC [256 p rows][x kblk] (K-major)
                    for (int kb = 0; kb < nkv; ++kb, ++gi) {
                        uint8_t* st = acquire(kStageA + 2 * kStageA);
                        tc::tma_load_3d_hint(st, kind == 0 ? &M.dH128 : &M.V128, bar(), kb * 64, r0, bh, keep);
                        for (int h = 0; h < 2; ++h)
                            tc::tma_load_3d_hint(st + kStageA + h * kStageA, kind == 0 ? &M.C128 : &M.dC128, bar(),
                                                 kb * 64, 128 * h, cidx, kind == 0 ? stream : keep);
                    }
                } else {  // A = K rows [p kblk], B = dC [p kblk][x 256-col half] (MN-major, 4 atoms)
                    for (int kb = 0; kb < nkq; ++kb, ++gi) {
                        uint8_t* st = acquire(kStageA + 4 * 8192);
                        tc::tma_load_3d_hint(st, &M.K128, bar(), kb * 64, r0, bh, keep);
                        for (int a = 0; a < 4; ++a)
                            tc::tma_load_3d_hint(st + kStageA + a * 8192, &M.dC64, bar(), ct * 256 + 64 * a, kb * 64,
                                                 cidx, stream);
                    }
                }
            };
            auto load_intra = [&](int g, int bh, int r0) {  // B = K | Q | dH [row kblk][256 cols], MN-major
                int kind, ct;
                group_kind(g, kind, ct);
                const CUtensorMap* z = kind == 0 ? &M.K64 : kind == 1 ? &M.Q64 : &M.dH64;
                for (int kb = 0; kb < 2; ++kb, ++gi) {
                    uint8_t* st = acquire(4 * 8192);
                    for (int a = 0; a < 4; ++a)
                        tc::tma_load_3d_hint(st + a * 8192, z, bar(), ct * 256 + 64 * a, r0 + kb * 64, bh, keep);
                }
            };
            for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
                const int bh = tile / NC, c = tile % NC, r0 = c * 128;
                const int cidx = bh * NC + c;
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
                // inter(0), inter(1), intra(0), inter(2), intra(1), ..., intra(n-1)
                load_inter(0, bh, r0, cidx);
                for (int g = 0; g < ngroups; ++g) {
                    if (g + 1 < ngroups) load_inter(g + 1, bh, r0, cidx);
                    load_intra(g, bh, r0);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ tcgen05 issuer
        int gi = 0, ti = 0;
        int use[2] = {0, 0}, ifu[2] = {0, 0}, isc[2] = {0, 0};
        const uint32_t id_s = tc::idesc_bf16(128, 128, 0, 0);
        auto take = [&]() -> uint32_t {
            const int s = gi % kStages;
            tc::mbar_wait(&full[s], (gi / kStages) & 1);
            tc::tc_fence_after();
            return tc::smem_u32(stages + s * kStage);
        };
        auto acquire_slot = [&](int slot) {  // the slot's previous user has been read out
            tc::mbar_wait(&sfree[slot], (use[slot] & 1) ^ 1);
            ++use[slot];
            tc::tc_fence_after();
        };
        auto inter = [&](int g) {
            int kind, ct;
            group_kind(g, kind, ct);
            const int slot = (g + 1) & 1;
            acquire_slot(slot);
            const uint32_t idesc = tc::idesc_bf16(128, 256, 0, kind == 2 ? 1 : 0);
            const int nkb = kind == 2 ? nkq : nkv;
            for (int kb = 0; kb < nkb; ++kb) {
                const uint32_t st = take();
                if (tc::elect_one()) {
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks) {
                        const uint64_t bd = kind == 2 ? tc::mnmajor_desc(st + kStageA, 64, ks)
                                                      : tc::kmajor_desc(st + kStageA, 256, ks);
                        tc::mma_bf16(tmem + slot * 256, tc::kmajor_desc(st, 128, ks), bd, idesc, (kb | ks) ? 1u : 0u);
                    }
                    tc::mma_commit(&empty[gi % kStages]);
                    if (kb == nkb - 1) tc::mma_commit(&ifull[slot]);
                }
                ++gi;
                __syncwarp();
            }
        };
        auto intra = [&](int g, bool last) {
            int kind, ct;
            group_kind(g, kind, ct);
            const int slot = (g + 1) & 1;
            tc::mbar_wait(&iscaled[slot], isc[slot] & 1);  // accumulate onto the scaled inter term
            ++isc[slot];
            tc::tc_fence_after();
            const uint32_t ga = tc::smem_u32(kind == 2 ? gP : gD);
            const uint32_t idesc = tc::idesc_bf16(128, 256, kind == 0 ? 0 : 1, 1);
            for (int kb = 0; kb < 2; ++kb) {
                const uint32_t st = take();
                if (tc::elect_one()) {
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks) {
                        const uint64_t ad = kind == 0 ? tc::kmajor_desc(ga, 128, kb * 4 + ks)
                                                      : tc::mnmajor_desc(ga, 128, kb * 4 + ks);
                        tc::mma_bf16(tmem + slot * 256, ad, tc::mnmajor_desc(st, 64, ks), idesc, 1u);
                    }
                    tc::mma_commit(&empty[gi % kStages]);
                    if (kb == 1) {
                        tc::mma_commit(&ofull[slot]);
                        if (last) tc::mma_commit(gempty);
                    }
                }
                ++gi;
                __syncwarp();
            }
        };
        (void)ifu;
        for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++ti) {
            // scores into slot 0: S at [0,128), dS at [128,256)
            acquire_slot(0);
            for (int pass = 0; pass < 2; ++pass) {
                const int nkb = pass == 0 ? nkq : nkv;
                for (int kb = 0; kb < nkb; ++kb) {
                    const uint32_t st = take();
                    if (tc::elect_one()) {
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks)
                            tc::mma_bf16(tmem + pass * 128, tc::kmajor_desc(st, 128, ks),
                                         tc::kmajor_desc(st + kStageA, 128, ks), id_s, (kb | ks) ? 1u : 0u);
                        tc::mma_commit(&empty[gi % kStages]);
                        if (pass == 1 && kb == nkb - 1) tc::mma_commit(sfull);
                    }
                    ++gi;
                    __syncwarp();
                }
            }
            inter(0);
            tc::mbar_wait(gfull, ti & 1);  // P' / dP' written by the gating
            tc::tc_fence_after();
            for (int g = 0; g < ngroups; ++g) {
                if (g + 1 < ngroups) inter(g + 1);
                intra(g, g == ngroups - 1);
            }
        }
    } else {
        // ------------------------------------------------ gating + epilogue
        const int et = threadIdx.x - 64;
        const int lane = tc::lane_id();
        const int row = (warp & 3) * 32 + lane;
        const int part = (warp - 2) >> 2;  // column half of every 128- / 256-wide tile
        const bool is_exp = args.variant == 0;
        const float rs = rsqrtf(static_cast<float>(G.dqk));
        const uint32_t trow = tc::tmem_row_addr(tmem);
        StabLocal sl;
        const bool stab = is_exp && args.gw.stab != nullptr;
        int ti = 0, ifu[2] = {0, 0}, ofu[2] = {0, 0};
        auto release_slot = [&](int slot) {
            tc::tc_fence_before();
            tc::mbar_arrive(&sfree[slot]);
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
            tc::named_bar_sync(1, kEpi);

            // ---- gating: P' and dP' from S and dS; row / column sums of dD
            tc::mbar_wait(sfull, ti & 1);
            tc::tc_fence_after();
            tc::mbar_wait(gempty, (ti & 1) ^ 1);
            float rowsum = 0.f;
#pragma unroll 1
            for (int gq = part * 2; gq < part * 2 + 2; ++gq) {
                float sv[32], dv[32];
                tc::tmem_ld32(trow + gq * 32, sv);
                tc::tmem_ld32(trow + 128 + gq * 32, dv);
                tc::tmem_ld_wait();
                if (stab)
                    for (int j = gq * 32; j < gq * 32 + 32 && j <= row; ++j) sl.note(rowterm + colterm[j]);
                float dd[32];
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    const int j = gq * 32 + e;
                    const float dp = j <= row ? exp2f(fminf(rowterm + colterm[j], 0.f)) * dinv : 0.f;
                    const float s = sv[e] * rs;
                    const float dsb = dv[e] * dp;
                    dd[e] = dsb * s;
                    rowsum += dd[e];
                    sv[e] = s * dp;
                    dv[e] = dsb * rs;
                }
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                    tc::sw128_store8(gP, row, gq * 4 + q4, 128, sv + 8 * q4);
                    tc::sw128_store8(gD, row, gq * 4 + q4, 128, dv + 8 * q4);
                }
#pragma unroll
                for (int k = 16; k >= 1; k >>= 1) {  // column sums over this warp's 32 rows
                    const bool up = lane & k;
#pragma unroll
                    for (int i = 0; i < k; ++i) {
                        const float send = up ? dd[i] : dd[i + k];
                        const float keep = up ? dd[i + k] : dd[i];
                        dd[i] = keep + __shfl_xor_sync(0xffffffffu, send, k);
                    }
                }
                csum[(warp - 2) * 64 + (gq - part * 2) * 32 + lane] = dd[0];
            }
            release_slot(0);  // S / dS read: slot 0 may take group 1's inter term
            tc::fence_proxy_async_smem();
            tc::mbar_arrive(gfull);
            tc::named_bar_sync(1, kEpi);
            float colsum = 0.f;
            if (et < 128) {
                const int hj = et / 64;
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) colsum += csum[(4 * hj + q4) * 64 + (et % 64)];
            }

            float dot_q = 0.f, dot_k = 0.f;
            // scale(g): O_g = scale_i * (inter term), dots for dQ / dK from the unscaled values
            auto scale_group = [&](int g) {
                int kind, ct;
                group_kind(g, kind, ct);
                const int slot = (g + 1) & 1;
                tc::mbar_wait(&ifull[slot], ifu[slot] & 1);
                ++ifu[slot];
                tc::tc_fence_after();
                const float sc = kind == 0 ? w_i : ab_i;
                const __nv_bfloat16* xr = kind == 0 ? args.q + t * G.dqk : kind == 1 ? args.k + t * G.dqk : nullptr;
#pragma unroll 1
                for (int p4 = 0; p4 < 4; ++p4) {
                    const int col = part * 128 + p4 * 32;
                    float iv[32];
                    tc::tmem_ld32(trow + slot * 256 + col, iv);
                    tc::tmem_ld_wait();
                    if (xr) {
                        float d = 0.f;
#pragma unroll
                        for (int e = 0; e < 32; e += 8) {
                            const uint4 raw = *reinterpret_cast<const uint4*>(xr + col + e);
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
                    uint32_t w[32];
#pragma unroll
                    for (int e = 0; e < 32; ++e) w[e] = __float_as_uint(sc * iv[e]);
                    tc::tmem_st32(trow + slot * 256 + col, w);
                }
                tc::tmem_st_wait();
                tc::tc_fence_before();
                tc::mbar_arrive(&iscaled[slot]);
            };
            // drain(g): O_g -> bf16 -> global (one 64-B row segment per thread and piece)
            auto drain_group = [&](int g) {
                int kind, ct;
                group_kind(g, kind, ct);
                const int slot = (g + 1) & 1;
                tc::mbar_wait(&ofull[slot], ofu[slot] & 1);
                ++ofu[slot];
                tc::tc_fence_after();
                __nv_bfloat16* orow = kind == 0   ? args.dq + t * G.dqk
                                      : kind == 1 ? args.dk + t * G.dqk
                                                  : args.dv + t * G.dhv + ct * 256;
#pragma unroll 1
                for (int p4 = 0; p4 < 4; ++p4) {
                    const int col = part * 128 + p4 * 32;
                    float ov[32];
                    tc::tmem_ld32(trow + slot * 256 + col, ov);
                    tc::tmem_ld_wait();
                    if (p4 == 3) release_slot(slot);  // this thread's TMEM columns are read
#pragma unroll
                    for (int q8 = 0; q8 < 4; ++q8) {
                        uint4 w;
                        w.x = tc::pack_bf16(ov[8 * q8], ov[8 * q8 + 1]);
                        w.y = tc::pack_bf16(ov[8 * q8 + 2], ov[8 * q8 + 3]);
                        w.z = tc::pack_bf16(ov[8 * q8 + 4], ov[8 * q8 + 5]);
                        w.w = tc::pack_bf16(ov[8 * q8 + 6], ov[8 * q8 + 7]);
                        __stcs(reinterpret_cast<uint4*>(orow + col) + q8, w);
                    }
                }
            };
            // gating | scale(0) | scale(1) | drain(0) | scale(2) | drain(1) | ... | drain(n-1)
            scale_group(0);
            for (int g = 0; g < ngroups; ++g) {
                if (g + 1 < ngroups) scale_group(g + 1);
                drain_group(g);
            }
            // ---- gate partials (n_ptile = 1)
            if (part == 1) {
                xred[row] = rowsum;
                xred[128 + row] = dot_q;
                xred[256 + row] = dot_k;
            }
            tc::named_bar_sync(1, kEpi);
            if (part == 0) {
                rowsum += xred[row];
                dot_q += xred[128 + row];
                dot_k += xred[256 + row];
                args.dbq_part[t] = rowsum + w_i * dot_q;
                if (args.iq_part) args.iq_part[t] = w_i * dot_q;
                args.da_part[t] = ab_i * dot_k;
            }
            if (et < 128) args.colsum[hb + r0 + et] = colsum;
            tc::named_bar_sync(1, kEpi);
        }
        if (stab) sl.flush(args.gw.stab);
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

}  // namespace

// Measured at the 7B shape: 1.21 vs 1.12 ms for bwd_fused.cu -- the 128-column
// kernel is bound by its epilogue (TMEM drain, gate-partial dots, stores), which
// the extra in-place row-scale pass lengthens -- so this variant is opt-in
// (TFLA_WIDE_FUSED_BWD=1) and kept parity-tested.
bool bwd_fused_wide_supported(const Geom& g) {
    return g.L == 128 && g.dqk == 256 && g.dhv % 256 == 0 && g.dhv <= 1024 &&
           tfla_host::env_flag("TFLA_WIDE_FUSED_BWD");
}

int launch_bwd_fused_wide(const BwdArgs& a, const BwdTensors& t, void* dq, void* dk, void* dv,
                          const void* c_states, const void* dc_states, cudaStream_t st) {
    using namespace tfla_host;
    const Geom& g = a.g;
    const uint64_t BH = g.BH, T = g.T, NCs = static_cast<uint64_t>(g.BH) * g.NC;
    WMaps m;
    bool ok = true;
    ok &= make_tmap_bf16_3d(&m.Q128, t.q, BH, T, g.dqk, 64, 128);
    ok &= make_tmap_bf16_3d(&m.K128, t.k, BH, T, g.dqk, 64, 128);
    ok &= make_tmap_bf16_3d(&m.V128, t.v, BH, T, g.dhv, 64, 128);
    ok &= make_tmap_bf16_3d(&m.dH128, t.dh, BH, T, g.dhv, 64, 128);
    ok &= make_tmap_bf16_3d(&m.K64, t.k, BH, T, g.dqk, 64, 64);
    ok &= make_tmap_bf16_3d(&m.Q64, t.q, BH, T, g.dqk, 64, 64);
    ok &= make_tmap_bf16_3d(&m.dH64, t.dh, BH, T, g.dhv, 64, 64);
    ok &= make_tmap_bf16_3d(&m.C128, c_states, NCs, g.dqk, g.dhv, 64, 128);
    ok &= make_tmap_bf16_3d(&m.dC128, dc_states, NCs, g.dqk, g.dhv, 64, 128);
    ok &= make_tmap_bf16_3d(&m.dC64, dc_states, NCs, g.dqk, g.dhv, 64, 64);
    if (!ok) return 4;
    ensure_smem_attr(reinterpret_cast<const void*>(bwd_fused_wide_kernel), kSmemBytes);
    const int n_tiles = g.BH * g.NC;
    BwdArgs aa = a;
    aa.dq = static_cast<__nv_bfloat16*>(dq);
    aa.dk = static_cast<__nv_bfloat16*>(dk);
    aa.dv = static_cast<__nv_bfloat16*>(dv);
    const int grid = n_tiles < num_sms() ? n_tiles : num_sms();
    bwd_fused_wide_kernel<<<grid, kThreads, kSmemBytes, st>>>(m, aa);
    return 0;
}

}  // namespace tfla_k
