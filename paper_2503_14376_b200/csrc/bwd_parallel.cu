// bwd_parallel.cu -- K4: TFLA parallel backward (dQ, dK, dV) on tcgen05, and
// K7: gate-gradient assembly.
//
// Restates the per-chunk part of chunkwise_backward (chunkwise.cpp:454-557) /
// tfla_backward_dq|dk|dv (tiled.cpp:391-779), normaliser and max states
// detached (the exact gradient of chunkwise_forward_frozen, chunkwise.cpp:304-394):
//   D'_ij  = exp(b_i - b_j + ib_j - m_c,i)  (j <= i, same chunk; exp)  / exp(b_i - b_j + ib_j) (sig)
//   dSb_ij = (dH_i . v_j) / den_i            S_ij = q_i . k_j / sqrt(d)
//   dQ_i = sum_j dSb_ij D'_ij k_j / sqrt(d) + w_i (dH_i C_k^T)          w_i = b_bar_i / (den_i sqrt d)
//   dK_j = sum_i dSb_ij D'_ij q_i / sqrt(d) + a_bar_j (v_j dC_{k+1}^T)
//   dV_j = sum_i S_ij D'_ij dH_i / den_i      + a_bar_j (k_j dC_{k+1})
//   dD_ij = dSb_ij S_ij D'_ij -> row sums (d_b_i +), column sums (d_b_j -, d_ib_j +)
//   d_b_i += w_i q_i . (dH_i C_k^T);  d_a_j = a_bar_j k_j . (v_j dC_{k+1}^T)
//
// One kernel template serves the three gradients (the Table-1 work partition of
// the paper): a CTA owns a 128-row tile ("own" rows = query
// rows for dQ, key rows for dK/dV) and one 128/N-wide output column tile, walks
// the 128-row tiles on the other side of the causal diagonal, recomputes the
// score tiles (S, dS) into TMEM, gates them on CUDA cores into a stationary
// bf16 smem operand, and accumulates the intra term with tcgen05; the
// inter-chunk term (state contraction) goes to its own TMEM accumulator and is
// combined with its row scale in the epilogue. Because one SW128 buffer is a
// K-major operand of shape (M=R, K=C) *and* an MN-major operand of (M=C, K=R),
// no transposes are materialised anywhere.
// Warps: 0 TMA producer, 1 tcgen05 issuer, 2..5 gating / epilogue.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <string>

#include "bwd_parallel.h"
#include "host_util.h"
#include "stab.cuh"
#include "tc.cuh"

namespace tfla_k {
namespace {

constexpr int kStageA = 128 * 64 * 2;
constexpr int kG = 128 * 128 * 2;  // stationary gated tile
constexpr int kVecs = 2 * 4 * 128 * 4 + 2 * 128 * 4 + 64;  // vt[2][4][128] | xred[2][128] | amax[16]
// Ring geometry per output width: N <= 128 -> 4 stages of 32 KB (A 16 + B 16);
// N = 256 ("wide") -> 3 stages of 48 KB (A 16 + B 32: a 256-row state tile or
// the 4 x 64-column intra operand of one 64-row k-block).
template <int N>
struct Ring {
    static constexpr int kStages = N == 256 ? 3 : 4;
    static constexpr int kStage = N == 256 ? 3 * kStageA : 2 * kStageA;
    static constexpr int kSmemBytes = kStages * kStage + 2 * kG + kVecs + 512;
};
constexpr int kEpi = 256;  // gating / epilogue threads (8 warps)
constexpr int kThreads = 64 + kEpi;
constexpr float kLog2e = 1.4426950408889634f;

struct Plan {
    int own_start;   // first own row (position within head)
    int c_first;     // chunk of the own tile's first row
    int R;           // chunks covered by the own tile (2 only for L = 64)
    int oth_start;   // first row of other tile 0
    int n_oth;       // number of other tiles
};

template <int KIND>
__device__ __forceinline__ Plan make_plan(const Geom& G, int tile) {
    Plan p;
    p.own_start = tile * 128;
    p.c_first = p.own_start / G.L;
    if (G.L >= 128) {
        p.R = 1;
        const int cstart = p.c_first * G.L;
        const int r0 = p.own_start - cstart;
        if (KIND == kDQ) {  // kv tiles up to the diagonal
            p.oth_start = cstart;
            p.n_oth = r0 / 128 + 1;
        } else {            // query tiles from the diagonal to the chunk end
            p.oth_start = p.own_start;
            p.n_oth = (G.L - r0) / 128;
        }
    } else {
        p.R = min(128 / G.L, G.NC - p.c_first);
        p.oth_start = p.own_start;
        p.n_oth = 1;
    }
    return p;
}

struct Maps {
    CUtensorMap X, Y, X2, Y2, Z, W, St, Out;
};

// N = 256 ("wide", L >= 128 only): one CTA covers 256 output columns (all of
// d_qk = 256 for dQ / dK, half of d_hv = 512 for dV), so the score tiles are
// recomputed half as often. TMEM then holds O (256) | S (128) | dS (128): there
// is no room for a separate inter accumulator, so the inter term is computed
// FIRST into O, the epilogue scales O's rows by w / a_bar in place (and takes
// the gate-partial dots from the unscaled values on the way), and the intra
// MMAs accumulate on top.
template <int KIND, int N>
__global__ void __launch_bounds__(kThreads, 1)
    bwd_parallel_kernel(const __grid_constant__ Maps M, BwdArgs args) {
    constexpr bool kHasDS = KIND != kDV;
    constexpr bool kWide = N == 256;
    constexpr int NO = (KIND == kDV || kWide) ? N : 128;  // output tile width
    constexpr int kStages = Ring<N>::kStages;
    constexpr int kStage = Ring<N>::kStage;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* stages = smem;
    uint8_t* gbuf = smem + kStages * kStage;  // [2][kG]
    float* vec = reinterpret_cast<float*>(gbuf + 2 * kG);  // [2][4][128]
    float* xred = vec + 2 * 4 * 128;  // [2][128] half-sum exchange
    uint64_t* bars = reinterpret_cast<uint64_t*>(xred + 2 * 128 + 16);
    uint64_t* full = bars;
    uint64_t* empty = full + kStages;
    uint64_t* sfull = empty + kStages;
    uint64_t* sempty = sfull + 1;
    uint64_t* gfull = sempty + 1;   // [2]
    uint64_t* gempty = gfull + 2;   // [2]
    uint64_t* ofull = gempty + 2;
    uint64_t* oempty = ofull + 1;    // O / I drained by the epilogue (next tile may write them)
    uint64_t* ifull = oempty + 1;    // wide: inter term in O
    uint64_t* iscaled = ifull + 1;   // wide: O rows scaled by the epilogue
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(iscaled + 1);

    const Geom& G = args.g;
    const int warp = tc::warp_id();
    const int nk_qk = G.dqk / 64, nk_hv = G.dhv / 64;
    const int nk_inter = KIND == kDV ? nk_qk : nk_hv;
    const int dim_out = KIND == kDV ? G.dhv : G.dqk;
    const int ncol = (dim_out + NO - 1) / NO, nrt = (G.T + 127) / 128;
    const int n_tiles = ncol * nrt * G.BH;
    // Persistent: tile = (column tile fastest, 128-row own tile, head), so the
    // CTAs working on one row tile at a time share its score operands in L2.
    // Barrier phases run on per-CTA counters across tiles: the next tile's
    // operand loads and score MMAs overlap this tile's gating and epilogue.
    auto decode = [&](int tile, int& ct, int& rt, int& bh) {
        ct = tile % ncol;
        rt = (tile / ncol) % nrt;
        bh = tile / (ncol * nrt);
    };
    // TMEM: O | I_0 | (I_1) | S | dS   (wide: O | S | dS, the inter term folded into O)
    const uint32_t colO = 0, colI = kWide ? 0 : NO;
    const uint32_t colS = kWide ? 256 : KIND == kDV ? 3 * NO : 2 * NO;
    const uint32_t colD = colS + 128;
    const bool alias_I1 = KIND != kDV;  // I_1 reuses S (dQ/dK, L = 64 only)
    const uint32_t colI1 = alias_I1 ? colS : colI + NO;
    // L = 64: the second chunk's inter accumulator aliases S (dQ / dK), so a
    // tile's first score MMA must wait until the previous tile is drained
    const bool serial_tiles = G.L < 128;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        tc::mbar_init(sfull, 1);
        tc::mbar_init(sempty, kEpi);
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&gfull[b], kEpi);
            tc::mbar_init(&gempty[b], 1);
        }
        tc::mbar_init(ofull, 1);
        tc::mbar_init(oempty, kEpi);
        tc::mbar_init(ifull, 1);
        tc::mbar_init(iscaled, kEpi);
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

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
            for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
                int ct, rt, bh;
                decode(tile, ct, rt, bh);
                const int col0 = ct * NO;
                const int nZ = min(NO / 64, (dim_out - col0) / 64);
                const Plan P = make_plan<KIND>(G, rt);
                auto load_scores = [&](int jt) {
                    const int oth = P.oth_start + jt * 128;
                    for (int kb = 0; kb < nk_qk; ++kb, ++gi) {
                        uint8_t* st = acquire(2 * 16384);
                        tc::tma_load_3d(st, &M.X, bar(), kb * 64, P.own_start, bh);
                        tc::tma_load_3d(st + kStageA, &M.Y, bar(), kb * 64, oth, bh);
                    }
                    if (kHasDS)
                        for (int kb = 0; kb < nk_hv; ++kb, ++gi) {
                            uint8_t* st = acquire(2 * 16384);
                            tc::tma_load_3d(st, &M.X2, bar(), kb * 64, P.own_start, bh);
                            tc::tma_load_3d(st + kStageA, &M.Y2, bar(), kb * 64, oth, bh);
                        }
                };
                auto load_inter = [&](int r) {
                    const int cidx = bh * G.NC + P.c_first + r;
                    for (int kb = 0; kb < nk_inter; ++kb, ++gi) {
                        if (KIND == kDV) {
                            uint8_t* st = acquire(16384 + NO * 128);
                            tc::tma_load_3d(st, &M.W, bar(), kb * 64, P.own_start, bh);
                            for (int a = 0; a < NO / 64; ++a)
                                tc::tma_load_3d(st + kStageA + a * 8192, &M.St, bar(), col0 + 64 * a,
                                                kb * 64, cidx);
                        } else {
                            uint8_t* st = acquire(16384 + NO * 128);
                            tc::tma_load_3d(st, &M.W, bar(), kb * 64, P.own_start, bh);
                            for (int a = 0; a < NO / 128; ++a)  // 128-row boxes of the [p][x] state tile
                                tc::tma_load_3d(st + kStageA + a * 16384, &M.St, bar(), kb * 64, col0 + 128 * a,
                                                cidx);
                        }
                    }
                };
                load_scores(0);
                load_inter(0);
                for (int jt = 0; jt < P.n_oth; ++jt) {
                    if (jt + 1 < P.n_oth) load_scores(jt + 1);
                    const int oth = P.oth_start + jt * 128;
                    for (int kb = 0; kb < 2; ++kb, ++gi) {
                        uint8_t* st = acquire(nZ * 8192);
                        for (int a = 0; a < nZ; ++a)
                            tc::tma_load_3d(st + kStageA + a * 8192, &M.Z, bar(), col0 + 64 * a,
                                            oth + kb * 64, bh);
                    }
                }
                if (P.R == 2) load_inter(1);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ tcgen05 issuer
        int gi = 0, u = 0, gu = 0, ti = 0;
        const uint32_t id_s = tc::idesc_bf16(128, 128, 0, 0);
        const uint32_t id_o = tc::idesc_bf16(128, NO, 0, 1);
        const uint32_t id_i = tc::idesc_bf16(128, NO, 0, KIND == kDV ? 1 : 0);
        // debug trace (CTA 0): cycles the issuer waits on each barrier kind
        const bool trc = args.trace && blockIdx.x == 0;
        long long w_full = 0, w_s = 0, w_g = 0, w_i = 0, w_o = 0, n_st = 0;
        const long long t_begin = clock64();
        auto timed_wait = [&](uint64_t* bar, uint32_t par, long long& acc) {
            if (trc) {
                const long long t0 = clock64();
                tc::mbar_wait(bar, par);
                acc += clock64() - t0;
            } else {
                tc::mbar_wait(bar, par);
            }
        };
        auto take = [&]() -> uint32_t {
            const int s = gi % kStages;
            timed_wait(&full[s], (gi / kStages) & 1, w_full);
            ++n_st;
            tc::tc_fence_after();
            return tc::smem_u32(stages + s * kStage);
        };
        auto gemm_kk = [&](uint32_t dcol, int nkb, bool last_commit_s) {
            for (int kb = 0; kb < nkb; ++kb) {
                const uint32_t st = take();
                if (tc::elect_one()) {
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks)
                        tc::mma_bf16(tmem + dcol, tc::kmajor_desc(st, 128, ks),
                                     tc::kmajor_desc(st + kStageA, 128, ks), id_s, (kb | ks) ? 1u : 0u);
                    tc::mma_commit(&empty[gi % kStages]);
                    if (last_commit_s && kb == nkb - 1) tc::mma_commit(sfull);
                }
                ++gi;
                __syncwarp();
            }
        };
        // score tile use u: S / dS must have been read by the gating of use u - 1
        auto mma_scores = [&]() {
            if (u > 0) {
                timed_wait(sempty, (u - 1) & 1, w_s);
                tc::tc_fence_after();
            }
            gemm_kk(colS, nk_qk, !kHasDS);
            if (kHasDS) gemm_kk(colD, nk_hv, true);
            ++u;
        };
        auto mma_inter = [&](uint32_t dcol) {
            for (int kb = 0; kb < nk_inter; ++kb) {
                const uint32_t st = take();
                if (tc::elect_one()) {
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks) {
                        const uint64_t bd = KIND == kDV ? tc::mnmajor_desc(st + kStageA, 64, ks)
                                                        : tc::kmajor_desc(st + kStageA, 128, ks);
                        tc::mma_bf16(tmem + dcol, tc::kmajor_desc(st, 128, ks), bd, id_i,
                                     (kb | ks) ? 1u : 0u);
                    }
                    tc::mma_commit(&empty[gi % kStages]);
                }
                ++gi;
                __syncwarp();
            }
        };
        auto wait_drained = [&]() {  // the previous tile's O / I have been read out
            if (ti > 0) {
                timed_wait(oempty, (ti - 1) & 1, w_o);
                tc::tc_fence_after();
            }
        };
        for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++ti) {
            int ct, rt, bh;
            decode(tile, ct, rt, bh);
            const Plan P = make_plan<KIND>(G, rt);
            if (serial_tiles) wait_drained();
            mma_scores();
            if (!serial_tiles) wait_drained();
            mma_inter(colI);
            if (kWide) {
                if (tc::elect_one()) tc::mma_commit(ifull);
                __syncwarp();
            }
            for (int jt = 0; jt < P.n_oth; ++jt) {
                if (jt + 1 < P.n_oth) mma_scores();
                const int b = gu & 1;
                timed_wait(&gfull[b], (gu >> 1) & 1, w_g);
                if (kWide && jt == 0) timed_wait(iscaled, ti & 1, w_i);  // the intra term adds onto the scaled inter
                tc::tc_fence_after();
                const uint32_t gb = tc::smem_u32(gbuf + b * kG);
                for (int kb = 0; kb < 2; ++kb) {
                    const uint32_t st = take();
                    if (tc::elect_one()) {
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks)
                            tc::mma_bf16(tmem + colO, tc::kmajor_desc(gb, 128, kb * 4 + ks),
                                         tc::mnmajor_desc(st + kStageA, 64, ks), id_o,
                                         (kWide || (jt | kb | ks)) ? 1u : 0u);
                        tc::mma_commit(&empty[gi % kStages]);
                        if (kb == 1) tc::mma_commit(&gempty[b]);
                    }
                    ++gi;
                    __syncwarp();
                }
                ++gu;
            }
            if (P.R == 2) {
                if (alias_I1) {
                    tc::mbar_wait(sempty, (u - 1) & 1);
                    tc::tc_fence_after();
                }
                mma_inter(colI1);
            }
            if (tc::elect_one()) tc::mma_commit(ofull);
            __syncwarp();
        }
        if (trc && tc::lane_id() == 0) {
            args.trace[0] = clock64() - t_begin;
            args.trace[1] = w_full;
            args.trace[2] = w_s;
            args.trace[3] = w_g;
            args.trace[4] = w_i;
            args.trace[5] = w_o;
            args.trace[6] = n_st;
            args.trace[7] = ti;
        }
    } else {
        // ------------------------------------------------ gating + epilogue
        // 8 warps: TMEM lane quarter = warp % 4; the two warps of a quarter
        // split the columns (64 of the 128-wide score tile, NO/2 of the output).
        const int et = threadIdx.x - 64;
        const int row = (warp & 3) * 32 + tc::lane_id();
        const int half = (warp - 2) >> 2;
        const int T = G.T, L = G.L;
        const bool is_exp = args.variant == 0;
        StabLocal sl;
        const bool stab = is_exp && args.gw.stab != nullptr;
        const float rs = rsqrtf(static_cast<float>(G.dqk));
        const uint32_t trow = tc::tmem_row_addr(tmem);
        // Strictly-lower tile pairs (every other position j before every own
        // position i, same chunk -- L >= 128) have a rank-1 gate matrix with
        // stable factors: with A = max_{j in tile J} (ib_j - b_j),
        //   D'_ij = exp(b_i - m_c,i + A) * exp(ib_j - b_j - A)
        // and both exponents are <= 0 (m_c,i >= b_i + A since all of J is <= i;
        // A is the max). The gating then costs two multiplies per element
        // instead of an exp2 and three shared loads (the split kernels' gating
        // is their per-tile bound). The diagonal tile keeps the element-wise form.
        float* amax_red = xred + 256;  // [16]: warp maxima for the rank-1 factors
        int u = 0, gu = 0, ti = 0;
        const bool etrc = args.trace && blockIdx.x == 0 && et == 0;
        long long e_sfull = 0, e_gate = 0, e_ofull = 0, e_drain = 0, e_gempty = 0;
        for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++ti) {
            int ct, rt, bh;
            decode(tile, ct, rt, bh);
            const int col0 = ct * NO;
            const int nZ = min(NO / 64, (dim_out - col0) / 64);
            const Plan P = make_plan<KIND>(G, rt);
            const size_t hb = static_cast<size_t>(bh) * T;
            const int t_own = P.own_start + row;
            const bool own_ok = t_own < T;
            const int c_own = own_ok ? t_own / L : -1;
            // own-row gate terms
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
            // dK / dV: A_own = max over this tile's own (key) rows of ib_j - b_j (log2)
            const bool fact_ok = G.L >= 128;
            if (KIND != kDQ && fact_ok && half == 0) {
                float x = own_ok ? own_term : -INFINITY;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
                if (tc::lane_id() == 0) amax_red[8 + (warp & 3)] = x;
            }
            float acc_dd = 0.f;  // dQ: row sums of dD; dK: column sums (this thread's half)
            float scale = 0.f;
            if (own_ok) scale = KIND == kDQ ? args.gw.bb[hb + t_own] : args.gw.ab[hb + t_own];
            float dot = 0.f;  // gate partial: q (dQ) / k (dK) row . unscaled inter term
            const __nv_bfloat16* xrow = nullptr;
            if (KIND != kDV && own_ok)
                xrow = (KIND == kDQ ? args.q : args.k) + (hb + t_own) * G.dqk + col0;
            // wide: O holds the bare inter term; scale this thread's half of the row
            // in place (TMEM ld / st) and take the gate-partial dot on the way
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
                tc::mbar_arrive(iscaled);
            };
            // the previous tile's output store still reads the staging (gbuf)
            if (et == 0) tc::tma_store_wait_read<0>();

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
                // rank-1 gate factors for a strictly-lower tile pair (see above)
                const int oth0 = P.oth_start + jt * 128;
                const bool lower = fact_ok && (KIND == kDQ ? (oth0 + 128 <= P.own_start) : (oth0 >= P.own_start + 128));
                float rowf = 0.f;
                if (lower) {
                    if (KIND == kDQ) {  // A over the other (key) tile's ib_j - b_j
                        if (et < 128) {
                            float x = reinterpret_cast<const int*>(vt)[384 + et] < T ? vt[et] : -INFINITY;
#pragma unroll
                            for (int o = 16; o > 0; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
                            if (tc::lane_id() == 0) amax_red[warp - 2] = x;
                        }
                        tc::named_bar_sync(1, kEpi);
                        const float A = fmaxf(fmaxf(amax_red[0], amax_red[1]), fmaxf(amax_red[2], amax_red[3]));
                        float cf = 0.f;
                        if (et < 128 && reinterpret_cast<const int*>(vt)[384 + et] < T) {
                            if (stab) sl.note(vt[et] - A);
                            cf = exp2f(fminf(vt[et] - A, 0.f));
                        }
                        tc::named_bar_sync(1, kEpi);  // every thread has read A before vt is overwritten
                        if (et < 128) vt[et] = cf;
                        if (stab && own_ok && half == 0) sl.note(own_term + A);
                        rowf = own_ok ? exp2f(fminf(own_term + A, 0.f)) * own_dinv : 0.f;
                    } else {  // A over this tile's own (key) rows; 1/den on the query columns
                        const float A = fmaxf(fmaxf(amax_red[8], amax_red[9]), fmaxf(amax_red[10], amax_red[11]));
                        float cf = 0.f;
                        if (et < 128 && reinterpret_cast<const int*>(vt)[384 + et] < T) {
                            if (stab) sl.note(vt[et] + A);
                            cf = exp2f(fminf(vt[et] + A, 0.f)) * vt[128 + et];
                        }
                        tc::named_bar_sync(1, kEpi);
                        if (et < 128) vt[et] = cf;
                        if (stab && own_ok && half == 0) sl.note(own_term - A);
                        rowf = own_ok ? exp2f(fminf(own_term - A, 0.f)) : 0.f;
                    }
                    tc::named_bar_sync(1, kEpi);
                }
                long long tq0 = etrc ? clock64() : 0;
                tc::mbar_wait(sfull, u & 1);
                if (etrc) { const long long t = clock64(); e_sfull += t - tq0; tq0 = t; }
                tc::tc_fence_after();
                tc::mbar_wait(&gempty[b], ((gu >> 1) & 1) ^ 1);
                if (etrc) { const long long t = clock64(); e_gempty += t - tq0; tq0 = t; }
                uint8_t* gt = gbuf + b * kG;
#pragma unroll 1
                for (int g = 2 * half; g < 2 * half + 2 && lower; ++g) {  // factorised gating
                    float sv[32], dv[32];
                    tc::tmem_ld32(trow + colS + g * 32, sv);
                    if (kHasDS) tc::tmem_ld32(trow + colD + g * 32, dv);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        const float dprime = rowf * vt[g * 32 + e];
                        float val;
                        if (KIND == kDV) {
                            val = sv[e] * rs * dprime;
                        } else {
                            const float dsb = dv[e] * dprime;
                            acc_dd = fmaf(dsb, sv[e] * rs, acc_dd);
                            val = dsb * rs;
                        }
                        sv[e] = val;
                    }
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) tc::sw128_store8(gt, row, g * 4 + q4, 128, sv + 8 * q4);
                }
#pragma unroll 1
                for (int g = 2 * half; g < 2 * half + 2 && !lower; ++g) {
                    float sv[32], dv[32];
                    tc::tmem_ld32(trow + colS + g * 32, sv);
                    if (kHasDS) tc::tmem_ld32(trow + colD + g * 32, dv);
                    tc::tmem_ld_wait();
                    if (stab) {  // audit off the hot loop (one uniform branch)
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
                        // causal: (i, j) = (own, other) for dQ, (other, own) for dK/dV
                        const bool ok = (KIND == kDQ ? (tu <= t_own) : (t_own <= tu)) && cu == c_own;
                        const float arg = fminf(own_term + vt[uu], 0.f);
                        const float dprime = ok ? exp2f(arg) : 0.f;
                        const float dinv_i = KIND == kDQ ? own_dinv : vt[128 + uu];
                        float val;
                        if (KIND == kDV) {
                            val = sv[e] * rs * dprime * dinv_i;
                        } else {
                            const float dsb = dv[e] * dinv_i * dprime;  // dSb * D'
                            acc_dd = fmaf(dsb, sv[e] * rs, acc_dd);
                            val = dsb * rs;
                        }
                        sv[e] = val;
                    }
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) tc::sw128_store8(gt, row, g * 4 + q4, 128, sv + 8 * q4);
                }
                tc::tc_fence_before();
                tc::mbar_arrive(sempty);
                tc::fence_proxy_async_smem();
                tc::mbar_arrive(&gfull[b]);
                if (etrc) e_gate += clock64() - tq0;
                if (kWide && jt == 0) scale_inter();
            }

            // ---- final epilogue: out = O + scale * I_r ; gate partials
            long long to0 = etrc ? clock64() : 0;
            tc::mbar_wait(ofull, ti & 1);
            if (etrc) { const long long t = clock64(); e_ofull += t - to0; to0 = t; }
            tc::tc_fence_after();
            const uint32_t colIr = (P.R == 2 && (warp & 3) >= 2) ? colI1 : colI;
            uint8_t* stg = gbuf;  // every MMA of this tile is done: both gated buffers are free
            const int nvalid = dim_out - col0;
#pragma unroll 1
            for (int g = half * (NO / 64); g < (half + 1) * (NO / 64); ++g) {
                float ov[32], iv[32];
                tc::tmem_ld32(trow + colO + g * 32, ov);
                if (!kWide) tc::tmem_ld32(trow + colIr + g * 32, iv);
                tc::tmem_ld_wait();
                if (!kWide) {
                    if (KIND != kDV && xrow && g * 32 < nvalid) {
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
#pragma unroll
                    for (int e = 0; e < 32; ++e) ov[e] = fmaf(scale, iv[e], ov[e]);
                }
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) tc::sw128_store8(stg, row, g * 4 + q4, 128, ov + 8 * q4);
            }
            tc::tc_fence_before();
            tc::mbar_arrive(oempty);  // O / I may take the next tile's MMAs
            if (KIND != kDV) {  // combine the two halves' partial sums
                if (half == 1) {
                    xred[row] = acc_dd;
                    xred[128 + row] = dot;
                }
                tc::named_bar_sync(1, kEpi);
                if (half == 0 && own_ok) {
                    acc_dd += xred[row];
                    dot += xred[128 + row];
                    const size_t pt_off = static_cast<size_t>(ct) * G.BH * T;
                    if (KIND == kDQ)
                        args.dbq_part[pt_off + hb + t_own] = (ct == 0 ? acc_dd : 0.f) + scale * dot;
                    if (KIND == kDK) {
                        args.da_part[pt_off + hb + t_own] = scale * dot;
                        if (ct == 0) args.colsum[hb + t_own] = acc_dd;
                    }
                }
            }
            tc::fence_proxy_async_smem();
            tc::named_bar_sync(1, kEpi);
            if (et == 0) {
                for (int a = 0; a < nZ; ++a)
                    tc::tma_store_3d(&M.Out, stg + a * 16384, col0 + 64 * a, P.own_start, bh);
                tc::tma_store_commit();
            }
            if (etrc) e_drain += clock64() - to0;
        }
        if (etrc) {
            args.trace[8] = e_sfull;
            args.trace[9] = e_gempty;
            args.trace[10] = e_gate;
            args.trace[11] = e_ofull;
            args.trace[12] = e_drain;
        }
        if (et == 0) tc::tma_store_wait_all<0>();
        if (stab) sl.flush(args.gw.stab);
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------- K7 assembly
// assemble_gate_grads_head (chunkwise.cpp:239-266):
//   d fbar_i = d_g[k] + sum_{j>=i} d_b_j + sum_{j<i} d_a_j ;  d f = d fbar * sigmoid(-f)
//   d i      = d_a + d_ib  (x sigmoid(-i) for sig)
// with d_b = sum_pt dbq_part - colsum, d_a = sum_pt da_part, d_ib = colsum and
// d_g[k] = gbar_k * sum_tiles dg_part. One CTA per (chunk, head), L threads.
__global__ void assemble_kernel(AssembleArgs a) {
    __shared__ double sh[32];
    __shared__ double dgs;
    const int c = blockIdx.x, bh = blockIdx.y, j = threadIdx.x, L = blockDim.x;
    const int T = a.g.T, NC = a.g.NC;
    const size_t BT = static_cast<size_t>(a.g.BH) * T;
    const size_t t = static_cast<size_t>(bh) * T + static_cast<size_t>(c) * L + j;
    if (j == 0) {
        double s = 0.0;
        const float* dp = a.dg_part + (static_cast<size_t>(bh) * NC + c) * a.n_tiles;
        for (int i = 0; i < a.n_tiles; ++i) s += dp[i];
        dgs = a.gbar ? s * a.gbar[static_cast<size_t>(bh) * NC + c] : s;
    }
    double db = a.colsum ? -static_cast<double>(a.colsum[t]) : 0.0;
    double da = 0.0;
    for (int p = 0; p < a.n_ptile; ++p) {
        db += a.dbq_part[p * BT + t];
        da += a.da_part[p * BT + t];
    }
    // suffix sum of d_b (inclusive) and prefix sum of d_a (exclusive)
    const int lane = j & 31, wid = j >> 5, nw = L >> 5;
    auto scan = [&](double v) {  // inclusive block scan
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            double u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += u;
        }
        __syncthreads();
        if (lane == 31) sh[wid] = v;
        __syncthreads();
        if (wid == 0) {
            double x = lane < nw ? sh[lane] : 0.0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                double u = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += u;
            }
            sh[lane] = x;
        }
        __syncthreads();
        if (wid > 0) v += sh[wid - 1];
        return v;
    };
    __shared__ double rev[1024];
    rev[j] = db;
    __syncthreads();
    const double suf_rev = scan(rev[L - 1 - j]);  // sum_{u >= L-1-j} d_b
    __syncthreads();
    rev[L - 1 - j] = suf_rev;
    const double pre = scan(da) - da;  // exclusive prefix
    __syncthreads();
    const double dfbar = dgs + rev[j] + pre;
    const double f = a.f_pre[t], i = a.i_pre[t];
    auto sigm = [](double x) {
        if (x >= 0.0) return 1.0 / (1.0 + exp(-x));
        const double e = exp(x);
        return e / (1.0 + e);
    };
    a.d_fpre[t] = static_cast<float>(dfbar * sigm(-f));
    const double dib = da + static_cast<double>(a.colsum ? a.colsum[t] : a.di_extra[t]);
    a.d_ipre[t] = static_cast<float>(a.variant == 0 ? dib : dib * sigm(-i));
}

__global__ void split_partials_kernel(int kind, size_t BT, int n_ptile, const float* __restrict__ dbq,
                                      const float* __restrict__ da, const float* __restrict__ colsum,
                                      float* out0, float* out1, float* out2) {
    const size_t t = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= BT) return;
    const float* src = kind == kDQ ? dbq : da;
    float s = 0.f;
    for (int p = 0; p < n_ptile; ++p) s += src[p * BT + t];
    out0[t] = s;
    if (kind == kDK) {
        out1[t] = -colsum[t];
        out2[t] = colsum[t];
    }
}

// one CTA per head: chunk sums of iq and da (one warp per chunk), then the
// reverse recurrence d_g[k] = d_g[k+1] + I_{k+1} - A_k in double.
__global__ void dg_from_partials_kernel(int T, int L, int NC, const float* __restrict__ iq,
                                        const float* __restrict__ da, float* __restrict__ d_g) {
    extern __shared__ double sums[];  // [NC] I_j | [NC] A_j
    const int bh = blockIdx.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const float* iqh = iq + static_cast<size_t>(bh) * T;
    const float* dah = da + static_cast<size_t>(bh) * T;
    for (int c = wid; c < NC; c += nw) {
        double si = 0.0, sa = 0.0;
        for (int j = lane; j < L; j += 32) {
            si += iqh[c * L + j];
            sa += dah[c * L + j];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            si += __shfl_xor_sync(0xffffffffu, si, o);
            sa += __shfl_xor_sync(0xffffffffu, sa, o);
        }
        if (lane == 0) {
            sums[c] = si;
            sums[NC + c] = sa;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double acc = 0.0;  // d_g[NC-1] = 0
        d_g[static_cast<size_t>(bh) * NC + NC - 1] = 0.f;
        for (int k = NC - 2; k >= 0; --k) {
            acc += sums[k + 1] - sums[NC + k];
            d_g[static_cast<size_t>(bh) * NC + k] = static_cast<float>(acc);
        }
    }
}

__global__ void dg_reduce_kernel(size_t n, int n_tiles, const float* __restrict__ dg_part,
                                 const float* __restrict__ gbar, float* __restrict__ d_g) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    for (int j = 0; j < n_tiles; ++j) s += dg_part[i * n_tiles + j];
    d_g[i] = static_cast<float>(s * gbar[i]);
}

__global__ void states_to_bf16_kernel(const float* __restrict__ in, __nv_bfloat16* __restrict__ out,
                                      size_t per_state, int NC, size_t total) {
    const size_t i = (static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
    if (i >= total) return;
    const size_t s = i / per_state, e = i % per_state;  // s = bh*NC + c
    const size_t bh = s / NC, c = s % NC;
    const float4 v = *reinterpret_cast<const float4*>(in + (bh * (NC + 1) + c) * per_state + e);
    __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
    *reinterpret_cast<__nv_bfloat162*>(out + i) = lo;
    *reinterpret_cast<__nv_bfloat162*>(out + i + 2) = hi;
}

template <int KIND, int N>
int launch_impl(const BwdArgs& a, const BwdTensors& t, cudaStream_t st) {
    using namespace tfla_host;
    const Geom& g = a.g;
    const uint64_t BH = g.BH, T = g.T, NCs = static_cast<uint64_t>(g.BH) * g.NC;
    Maps m;
    bool ok = true;
    auto rows128 = [&](CUtensorMap* mp, const void* p, int d) {
        ok &= make_tmap_bf16_3d(mp, p, BH, T, d, 64, 128);
    };
    auto rows64 = [&](CUtensorMap* mp, const void* p, int d) {
        ok &= make_tmap_bf16_3d(mp, p, BH, T, d, 64, 64);
    };
    if (KIND == kDQ) {
        rows128(&m.X, t.q, g.dqk);
        rows128(&m.Y, t.k, g.dqk);
        rows128(&m.X2, t.dh, g.dhv);
        rows128(&m.Y2, t.v, g.dhv);
        rows64(&m.Z, t.k, g.dqk);
        rows128(&m.W, t.dh, g.dhv);
        ok &= make_tmap_bf16_3d(&m.St, t.states, NCs, g.dqk, g.dhv, 64, 128);
        rows128(&m.Out, t.out, g.dqk);
    } else if (KIND == kDK) {
        rows128(&m.X, t.k, g.dqk);
        rows128(&m.Y, t.q, g.dqk);
        rows128(&m.X2, t.v, g.dhv);
        rows128(&m.Y2, t.dh, g.dhv);
        rows64(&m.Z, t.q, g.dqk);
        rows128(&m.W, t.v, g.dhv);
        ok &= make_tmap_bf16_3d(&m.St, t.states, NCs, g.dqk, g.dhv, 64, 128);
        rows128(&m.Out, t.out, g.dqk);
    } else {
        rows128(&m.X, t.k, g.dqk);
        rows128(&m.Y, t.q, g.dqk);
        m.X2 = m.X;
        m.Y2 = m.Y;
        rows64(&m.Z, t.dh, g.dhv);
        rows128(&m.W, t.k, g.dqk);
        ok &= make_tmap_bf16_3d(&m.St, t.states, NCs, g.dqk, g.dhv, 64, 64);
        rows128(&m.Out, t.out, g.dhv);
    }
    if (!ok) return 4;
    constexpr int kSmemBytes = Ring<N>::kSmemBytes;
    tfla_host::ensure_smem_attr(reinterpret_cast<const void*>(bwd_parallel_kernel<KIND, N>), kSmemBytes);
    constexpr int NO = (KIND == kDV || N == 256) ? N : 128;
    const int dim_out = KIND == kDV ? g.dhv : g.dqk;
    const long n_tiles = static_cast<long>((dim_out + NO - 1) / NO) * ((g.T + 127) / 128) * g.BH;
    // Static tile striding: tiles of one chunk have unequal work (query tile p
    // of a chunk visits p + 1 key tiles), so the grid size is made coprime to
    // the (column tile x tile-in-chunk) period -- otherwise every CTA would see
    // the same tile-in-chunk position and the heaviest would set the runtime.
    const int period = ((dim_out + NO - 1) / NO) * (g.L >= 128 ? g.L / 128 : 1);
    const int grid = tfla_host::coprime_grid(n_tiles, period);
    bwd_parallel_kernel<KIND, N><<<grid, kThreads, kSmemBytes, st>>>(m, a);
    return 0;
}

}  // namespace

bool bwd_wide_qk(const Geom& g) { return g.L >= 128 && g.dqk == 256 && !tfla_host::env_flag("TFLA_NO_WIDE_BWD"); }
bool bwd_wide_v(const Geom& g) { return g.L >= 128 && g.dhv % 256 == 0 && !tfla_host::env_flag("TFLA_NO_WIDE_BWD"); }
int bwd_n_ptile(const Geom& g) { return bwd_wide_qk(g) ? 1 : (g.dqk + 127) / 128; }

int launch_bwd_parallel_impl(BwdKind kind, const BwdArgs& a, const BwdTensors& t, cudaStream_t st);

// debug: TFLA_TRACE_BWDK=<prefix> dumps CTA 0's barrier-wait cycle totals of
// each split backward kernel (issuer: total, full, sempty, gfull, iscaled,
// oempty, stages, tiles; epilogue thread 0: sfull, gempty, gating, ofull,
// drain) to <prefix>_<kind>.txt (eager launches only)
int launch_bwd_parallel(BwdKind kind, const BwdArgs& a0, const BwdTensors& t, cudaStream_t st) {
    const char* tf = getenv("TFLA_TRACE_BWDK");
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cap);
    if (!tf || !*tf || cap != cudaStreamCaptureStatusNone) return launch_bwd_parallel_impl(kind, a0, t, st);
    BwdArgs a = a0;
    cudaMalloc(&a.trace, 64 * sizeof(long long));
    cudaMemsetAsync(a.trace, 0, 64 * sizeof(long long), st);
    const int rc = launch_bwd_parallel_impl(kind, a, t, st);
    long long h[64];
    cudaMemcpyAsync(h, a.trace, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    cudaFree(a.trace);
    const std::string fn = std::string(tf) + "_" + (kind == kDQ ? "dq" : kind == kDK ? "dk" : "dv") + ".txt";
    if (FILE* f = fopen(fn.c_str(), "w")) {
        for (int i = 0; i < 13; ++i) fprintf(f, "%lld%c", h[i], i == 12 ? '\n' : ' ');
        fclose(f);
    }
    return rc;
}

int launch_bwd_parallel_impl(BwdKind kind, const BwdArgs& a, const BwdTensors& t, cudaStream_t st) {
    const Geom& g = a.g;
    if (bwd_pair_supported(g) && (kind != kDV || a.ntile == 128)) return launch_bwd_pair(kind, a, t, st);
    switch (kind) {
        case kDQ: return bwd_wide_qk(g) ? launch_impl<kDQ, 256>(a, t, st) : launch_impl<kDQ, 128>(a, t, st);
        case kDK: return bwd_wide_qk(g) ? launch_impl<kDK, 256>(a, t, st) : launch_impl<kDK, 128>(a, t, st);
        default:
            if (bwd_wide_v(g) && a.ntile == 128) return launch_impl<kDV, 256>(a, t, st);
            return a.ntile == 128 ? launch_impl<kDV, 128>(a, t, st) : launch_impl<kDV, 64>(a, t, st);
    }
}

void launch_assemble(const AssembleArgs& a, cudaStream_t st) {
    dim3 grid(a.g.NC, a.g.BH);
    assemble_kernel<<<grid, a.g.L, 0, st>>>(a);
}

void launch_split_partials(BwdKind kind, const Geom& g, int n_ptile, const float* dbq_part,
                           const float* da_part, const float* colsum, float* out0, float* out1,
                           float* out2, cudaStream_t st) {
    const size_t BT = static_cast<size_t>(g.BH) * g.T;
    split_partials_kernel<<<static_cast<unsigned>((BT + 255) / 256), 256, 0, st>>>(
        kind, BT, n_ptile, dbq_part, da_part, colsum, out0, out1, out2);
}

void launch_dg_from_partials(const Geom& g, const float* iq, const float* da, float* d_g, cudaStream_t st) {
    dg_from_partials_kernel<<<g.BH, 256, static_cast<size_t>(2 * g.NC) * sizeof(double), st>>>(g.T, g.L, g.NC, iq,
                                                                                             da, d_g);
}

void launch_dg_reduce(const Geom& g, int n_tiles, const float* dg_part, const float* gbar, float* d_g,
                      cudaStream_t st) {
    const size_t n = static_cast<size_t>(g.BH) * g.NC;
    dg_reduce_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(n, n_tiles, dg_part, gbar, d_g);
}

void launch_states_to_bf16(const float* c_states, __nv_bfloat16* out, const Geom& g,
                           cudaStream_t st) {
    const size_t per = static_cast<size_t>(g.dqk) * g.dhv;
    const size_t total = static_cast<size_t>(g.BH) * g.NC * per;
    const int threads = 256;
    const size_t blocks = (total / 4 + threads - 1) / threads;
    states_to_bf16_kernel<<<static_cast<unsigned>(blocks), threads, 0, st>>>(c_states, out, per,
                                                                           g.NC, total);
}

}  // namespace tfla_k
