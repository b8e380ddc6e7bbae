// fwd_parallel.cu -- K2: TFLA parallel forward on tcgen05.
//
// Restates the intra-chunk part + combine of chunkwise_forward_head
// (chunkwise.cpp:99-180) / tfla_forward_head (tiled.cpp:59-240):
//   S_ij  = q_i . k_j / sqrt(d)                                   (QK^T, tcgen05)
//   Sb_ij = S_ij exp(b_i - b_j + ib_j - m_c,i)   (j <= i, same chunk; 0 otherwise)
//   H_i   = [ sum_j Sb_ij v_j  +  b_bar_i (q_i / sqrt(d))^T C_k ] / den_i
//   den_i = max(|sum_j Sb_ij + b_bar_i q_i.n_k / sqrt(d)|, exp(-m_c,i))    (exp)
// Because the in-chunk max is separable (gates.cu), m_c is known before the
// first MMA: there is no online rescaling and mLSTMexp uses the single fused
// accumulation pass the reference only uses for mLSTMsig (tiled.cpp:158-170).
// For mLSTMsig: Sb_ij = S_ij exp(b_i - b_j + ib_j), inter scale exp(b_i), den = 1.
//
// CTA = (x tile of N columns of d_hv, 128-row query tile, head). The query tile
// walks its kv tiles (128 rows each, up to the diagonal, TFLA's L_kv loop); the
// S tiles are double buffered in TMEM so QK^T of tile j+1 overlaps the gating of
// tile j; Q C_k (the inter-chunk term) is issued right after the first QK^T and
// overlaps the gating as well. For L = 64 one 128-row tile spans two chunks and
// gets one inter accumulator per chunk.
// Warps: 0 TMA producer, 1 tcgen05 issuer, 2..5 gating / epilogue.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "fwd_parallel.h"
#include "host_util.h"
#include "stab.cuh"
#include "tc.cuh"

namespace tfla_k {
namespace {

constexpr int kStageA = 128 * 64 * 2;   // 16 KB: 128 rows x 64 K
constexpr int kSbar = 128 * 128 * 2;    // 32 KB stationary gated-score tile
constexpr int kEpi = 256;  // gating / epilogue threads (8 warps)
constexpr int kThreads = 64 + kEpi;
constexpr float kLog2e = 1.4426950408889634f;
// Ring per output width: N <= 128 -> 4 stages of 32 KB (B = 16 KB: 64 K-rows x
// 128 MN); N = 256 ("wide") -> 3 stages of 48 KB (B = 32 KB: 64 K-rows x 256).
template <int N>
struct Ring {
    static constexpr int kStages = N == 256 ? 3 : 4;
    static constexpr int kStage = N == 256 ? 3 * kStageA : 2 * kStageA;
    static constexpr int kSmemBytes = kStages * kStage + 2 * kSbar + 3 * 2 * 128 * 4 + 512;
};

// Job sequence shared by the producer and the MMA issuer.
struct Plan {
    int rows_start, c_first, R, kv_start, n_kv, nkq;
};

__device__ __forceinline__ Plan make_plan(const Geom& G, int rt) {
    Plan p;
    p.rows_start = rt * 128;
    p.c_first = p.rows_start / G.L;
    p.nkq = G.dqk / 64;
    if (G.L >= 128) {
        p.R = 1;
        p.kv_start = p.c_first * G.L;
        p.n_kv = (p.rows_start - p.kv_start) / 128 + 1;
    } else {
        p.R = min(128 / G.L, G.NC - p.c_first);
        p.kv_start = p.rows_start;
        p.n_kv = 1;
    }
    return p;
}

// Persistent: one CTA per SM walks tiles (x tile fastest, so neighbouring
// CTAs share the Q/K tiles in L2). Barrier phases run on global counters, so
// the next tile's loads and QK^T overlap this tile's epilogue.
// N = 256 ("wide", L >= 128): 256 output columns per CTA, so S = QK^T is
// recomputed twice per query tile at d_hv = 512 instead of four times. TMEM
// holds H (256) | S_0 | S_1: the inter term Q C_k goes into H FIRST, the
// epilogue scales H's rows by b_bar / sqrt(d) in place, and the intra S_bar V
// MMAs accumulate on top (one accumulator, no separate inter columns).
template <int N>
__global__ void __launch_bounds__(kThreads, 1)
    fwd_parallel_kernel(const __grid_constant__ CUtensorMap mapQ,
                        const __grid_constant__ CUtensorMap mapK,
                        const __grid_constant__ CUtensorMap mapV,
                        const __grid_constant__ CUtensorMap mapC,
                        const __grid_constant__ CUtensorMap mapH, FwdArgs args) {
    constexpr bool kWide = N == 256;
    constexpr int kStages = Ring<N>::kStages;
    constexpr int kStage = Ring<N>::kStage;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* stages = smem;
    uint8_t* sbar = smem + kStages * kStage;           // [2][32 KB]
    float* colv = reinterpret_cast<float*>(sbar + 2 * kSbar);  // [2][128] column gate term
    int* colc = reinterpret_cast<int*>(colv + 2 * 128);        // [2][128] column chunk id
    float* xred = reinterpret_cast<float*>(colc + 2 * 128);    // [2][128] half-sum exchange
    uint64_t* bars = reinterpret_cast<uint64_t*>(xred + 2 * 128);
    uint64_t* full = bars;
    uint64_t* empty = full + kStages;
    uint64_t* sfull = empty + kStages;   // [2] S accumulator ready
    uint64_t* sempty = sfull + 2;        // [2] S accumulator drained
    uint64_t* bfull = sempty + 2;        // [2] Sbar smem written
    uint64_t* bempty = bfull + 2;        // [2] Sbar smem consumed
    uint64_t* hfull = bempty + 2;        // H + inter accumulators final
    uint64_t* hempty = hfull + 1;        // H + inter accumulators drained
    uint64_t* ifull = hempty + 1;        // wide: inter term in H
    uint64_t* iscaled = ifull + 1;       // wide: H rows scaled
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(iscaled + 1);

    const Geom& G = args.g;
    const int nxt = G.dhv / N, nrt = (G.T + 127) / 128;
    const int n_tiles = nxt * nrt * G.BH;
    const int warp = tc::warp_id();
    // TMEM columns: H | I_0 | I_1 | S_0 | S_1  (S_1 only when R == 1: 2N + 256 <= 512)
    // wide: H | S_0 | S_1 (inter folded into H)
    const uint32_t colH = 0, colI = kWide ? 0 : N;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&sfull[b], 1);
            tc::mbar_init(&sempty[b], kEpi);
            tc::mbar_init(&bfull[b], kEpi);
            tc::mbar_init(&bempty[b], 1);
        }
        tc::mbar_init(hfull, 1);
        tc::mbar_init(hempty, kEpi);
        tc::mbar_init(ifull, 1);
        tc::mbar_init(iscaled, kEpi);
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    auto decode = [&](int tile, int& xt, int& rt, int& bh) {
        xt = tile % nxt;
        rt = (tile / nxt) % nrt;
        bh = tile / (nxt * nrt);
    };
    // S buffers: with two inter accumulators (L = 64) only one S buffer fits
    auto s_col = [&](const Plan& P, int u) -> uint32_t {
        if (kWide) return 256u + (u & 1) * 128u;
        return (P.R == 2 ? 3u * N : 2u * N) + (P.R == 2 ? 0u : (u & 1) * 128u);
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
            for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
                int xt, rt, bh;
                decode(tile, xt, rt, bh);
                const int x0 = xt * N;
                const Plan P = make_plan(G, rt);
                auto load_s = [&](int jt) {
                    for (int kb = 0; kb < P.nkq; ++kb, ++gi) {
                        uint8_t* st = acquire(2 * 16384);
                        const int s = gi % kStages;
                        tc::tma_load_3d(st, &mapQ, &full[s], kb * 64, P.rows_start, bh);
                        tc::tma_load_3d(st + kStageA, &mapK, &full[s], kb * 64, P.kv_start + jt * 128, bh);
                    }
                };
                load_s(0);
                for (int r = 0; r < P.R; ++r)
                    for (int kb = 0; kb < P.nkq; ++kb, ++gi) {
                        uint8_t* st = acquire(16384 + N * 128);
                        const int s = gi % kStages;
                        tc::tma_load_3d(st, &mapQ, &full[s], kb * 64, P.rows_start, bh);
                        for (int a = 0; a < N / 64; ++a)
                            tc::tma_load_3d(st + kStageA + a * 8192, &mapC, &full[s], x0 + 64 * a, kb * 64,
                                            bh * G.NC + P.c_first + r);
                    }
                for (int jt = 0; jt < P.n_kv; ++jt) {
                    if (jt + 1 < P.n_kv) load_s(jt + 1);
                    for (int kb = 0; kb < 2; ++kb, ++gi) {
                        uint8_t* st = acquire(N * 128);
                        const int s = gi % kStages;
                        for (int a = 0; a < N / 64; ++a)
                            tc::tma_load_3d(st + kStageA + a * 8192, &mapV, &full[s], x0 + 64 * a,
                                            P.kv_start + jt * 128 + kb * 64, bh);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ tcgen05 issuer
        int gi = 0, u0 = 0, ti = 0;
        const uint32_t id_s = tc::idesc_bf16(128, 128, 0, 0);
        const uint32_t id_n = tc::idesc_bf16(128, N, 0, 1);
        auto take = [&]() -> uint32_t {
            const int s = gi % kStages;
            tc::mbar_wait(&full[s], (gi / kStages) & 1);
            tc::tc_fence_after();
            return tc::smem_u32(stages + s * kStage);
        };
        for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++ti) {
            int xt, rt, bh;
            decode(tile, xt, rt, bh);
            const Plan P = make_plan(G, rt);
            auto mma_s = [&](int u) {
                const int b = u & 1;
                tc::mbar_wait(&sempty[b], ((u >> 1) & 1) ^ 1);
                tc::tc_fence_after();
                const uint32_t scol = s_col(P, u);
                for (int kb = 0; kb < P.nkq; ++kb) {
                    const uint32_t st = take();
                    if (tc::elect_one()) {
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks)
                            tc::mma_bf16(tmem + scol, tc::kmajor_desc(st, 128, ks),
                                         tc::kmajor_desc(st + kStageA, 128, ks), id_s, (kb | ks) ? 1u : 0u);
                        tc::mma_commit(&empty[gi % kStages]);
                        if (kb == P.nkq - 1) tc::mma_commit(&sfull[b]);
                    }
                    ++gi;
                    __syncwarp();
                }
            };
            mma_s(u0);
            // H / I of the previous tile must be drained by its epilogue
            tc::mbar_wait(hempty, (ti & 1) ^ 1);
            tc::tc_fence_after();
            for (int r = 0; r < P.R; ++r)
                for (int kb = 0; kb < P.nkq; ++kb) {
                    const uint32_t st = take();
                    if (tc::elect_one()) {
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks)
                            tc::mma_bf16(tmem + colI + r * N, tc::kmajor_desc(st, 128, ks),
                                         tc::mnmajor_desc(st + kStageA, 64, ks), id_n, (kb | ks) ? 1u : 0u);
                        tc::mma_commit(&empty[gi % kStages]);
                    }
                    ++gi;
                    __syncwarp();
                }
            if (kWide) {
                if (tc::elect_one()) tc::mma_commit(ifull);
                __syncwarp();
            }
            for (int jt = 0; jt < P.n_kv; ++jt) {
                const int u = u0 + jt;
                if (jt + 1 < P.n_kv) mma_s(u + 1);
                const int b = u & 1;
                tc::mbar_wait(&bfull[b], (u >> 1) & 1);
                if (kWide && jt == 0) tc::mbar_wait(iscaled, ti & 1);  // S_bar V adds onto the scaled inter
                tc::tc_fence_after();
                const uint32_t sb = tc::smem_u32(sbar + b * kSbar);
                for (int kb = 0; kb < 2; ++kb) {
                    const uint32_t st = take();
                    if (tc::elect_one()) {
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks)
                            tc::mma_bf16(tmem + colH, tc::kmajor_desc(sb, 128, kb * 4 + ks),
                                         tc::mnmajor_desc(st + kStageA, 64, ks), id_n,
                                         (kWide || (jt | kb | ks)) ? 1u : 0u);
                        tc::mma_commit(&empty[gi % kStages]);
                        if (kb == 1) tc::mma_commit(&bempty[b]);
                        if (kb == 1 && jt == P.n_kv - 1) tc::mma_commit(hfull);
                    }
                    ++gi;
                    __syncwarp();
                }
            }
            u0 += P.n_kv;
        }
    } else {
        // ------------------------------------------------ gating + epilogue
        // 8 warps: TMEM lane quarter = warp % 4, the two warps of a quarter
        // split the columns (half 0: [0, 64) of S / [0, N/2) of H).
        const int et = threadIdx.x - 64;
        const int row = (warp & 3) * 32 + tc::lane_id();
        const int half = (warp - 2) >> 2;
        const int T = G.T, L = G.L;
        const bool is_exp = args.variant == 0;
        const float rs = rsqrtf(static_cast<float>(G.dqk));
        const uint32_t trow = tc::tmem_row_addr(tmem);
        int u0 = 0, ti = 0;
        StabLocal sl;
        const bool stab = args.gw.stab != nullptr && is_exp;
        // the stabilised exponent is clamped at 0 (rounding can push it to +1e-5);
        // the frozen forward (pinned m_comb) is evaluated off its own stabiliser
        // point by finite differences and, like chunkwise_forward_frozen
        // (chunkwise.cpp:370-372, plain std::exp), must not clamp
        const float arg_max = args.den_fixed ? INFINITY : 0.f;
        for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++ti) {
            int xt, rt, bh;
            decode(tile, xt, rt, bh);
            const int x0 = xt * N;
            const Plan P = make_plan(G, rt);
            const size_t hb = static_cast<size_t>(bh) * T;
            const int t = P.rows_start + row;
            const bool row_ok = t < T;
            float b_i = 0.f, mc_i = 0.f, bb_i = 0.f;
            if (row_ok) {
                b_i = args.gw.b[hb + t];
                mc_i = args.gw.mc[hb + t];
                bb_i = args.gw.bb[hb + t];
            }
            const float rowterm = (is_exp ? (b_i - mc_i) : b_i) * kLog2e;
            const int c_i = row_ok ? t / L : -1;
            float rowsum = 0.f;
            // the previous tile's H store still reads Sbar buffer 0
            if (et == 0) tc::tma_store_wait_read<0>();

            for (int jt = 0; jt < P.n_kv; ++jt) {
                const int u = u0 + jt;
                const int b = u & 1;
                // column gate terms of this kv tile (thread et <-> column et)
                if (et < 128) {
                    const int tj = P.kv_start + jt * 128 + et;
                    const bool ok = tj < T;
                    colv[b * 128 + et] = ok ? (args.gw.ib[hb + tj] - args.gw.b[hb + tj]) * kLog2e : 0.f;
                    colc[b * 128 + et] = ok ? tj / L : -2;
                }
                tc::named_bar_sync(1, kEpi);
                tc::mbar_wait(&sfull[b], (u >> 1) & 1);
                tc::tc_fence_after();
                tc::mbar_wait(&bempty[b], ((u >> 1) & 1) ^ 1);
                uint8_t* sb = sbar + b * kSbar;
                const int kv0 = P.kv_start + jt * 128;
                const uint32_t scol = s_col(P, u);
#pragma unroll 1
                for (int g = 2 * half; g < 2 * half + 2; ++g) {
                    float v[32];
                    tc::tmem_ld32(trow + scol + g * 32, v);
                    tc::tmem_ld_wait();
                    if (stab && xt == 0) {  // audit off the hot loop (one uniform branch)
#pragma unroll 1
                        for (int j = g * 32; j < g * 32 + 32; ++j)
                            if ((kv0 + j <= t) && (colc[b * 128 + j] == c_i)) sl.note(rowterm + colv[b * 128 + j]);
                    }
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        const int j = g * 32 + e;
                        const bool ok = (kv0 + j <= t) && (colc[b * 128 + j] == c_i);
                        const float arg = fminf(rowterm + colv[b * 128 + j], arg_max);
                        const float wgt = ok ? v[e] * rs * exp2f(arg) : 0.f;
                        rowsum += wgt;
                        v[e] = wgt;
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) tc::sw128_store8(sb, row, g * 4 + q, 128, v + 8 * q);
                }
                tc::tc_fence_before();
                tc::mbar_arrive(&sempty[b]);
                tc::fence_proxy_async_smem();
                tc::mbar_arrive(&bfull[b]);
                if (kWide && jt == 0) {  // H = b_bar / sqrt(d) * (Q C_k), in place
                    tc::mbar_wait(ifull, ti & 1);
                    tc::tc_fence_after();
                    const float wi = bb_i * rs;
#pragma unroll 1
                    for (int g = half * (N / 64); g < (half + 1) * (N / 64); ++g) {
                        float iv[32];
                        tc::tmem_ld32(trow + colH + g * 32, iv);
                        tc::tmem_ld_wait();
                        uint32_t w[32];
#pragma unroll
                        for (int e = 0; e < 32; ++e) w[e] = __float_as_uint(wi * iv[e]);
                        tc::tmem_st32(trow + colH + g * 32, w);
                    }
                    tc::tmem_st_wait();
                    tc::tc_fence_before();
                    tc::mbar_arrive(iscaled);
                }
            }

            // denominator (exp): q_i . n_{c_i} comes precomputed (qn_kernel)
            if (half == 1) xred[row] = rowsum;
            tc::named_bar_sync(1, kEpi);
            if (half == 0) xred[row] += rowsum;
            tc::named_bar_sync(1, kEpi);
            rowsum = xred[row];
            const float qn = (is_exp && row_ok && !args.den_fixed) ? args.qn[hb + t] : 0.f;
            float den = 1.f;
            if (is_exp && row_ok) den = fmaxf(fabsf(rowsum + bb_i * rs * qn), exp2f(-mc_i * kLog2e));
            if (is_exp && row_ok && args.den_fixed) den = args.den_fixed[hb + t];
            const float inv_den = 1.f / den;
            const float wint = bb_i * rs;
            if (xt == 0 && row_ok && half == 0 && args.h_denom) args.h_denom[hb + t] = den;

            tc::mbar_wait(hfull, ti & 1);
            tc::tc_fence_after();
            uint8_t* stg = sbar;  // this tile's MMAs are done: Sbar buffer 0 is free
            const uint32_t colIr = colI + (P.R == 2 ? (((warp & 3) >= 2) ? N : 0) : 0);
            if (kWide) {  // H already holds the scaled inter term: drain in 32-column pieces
#pragma unroll 1
                for (int g = half * (N / 64); g < (half + 1) * (N / 64); ++g) {
                    float hv[32];
                    tc::tmem_ld32(trow + colH + g * 32, hv);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int e = 0; e < 32; ++e) hv[e] *= inv_den;
#pragma unroll
                    for (int q = 0; q < 4; ++q) tc::sw128_store8(stg, row, g * 4 + q, 128, hv + 8 * q);
                }
                tc::tc_fence_before();
                tc::mbar_arrive(hempty);
            } else {
            float hv[N / 2], iv[N / 2];
#pragma unroll
            for (int g = 0; g < N / 64; ++g) {
                tc::tmem_ld32(trow + colH + (half * (N / 64) + g) * 32, *reinterpret_cast<float(*)[32]>(hv + 32 * g));
                tc::tmem_ld32(trow + colIr + (half * (N / 64) + g) * 32, *reinterpret_cast<float(*)[32]>(iv + 32 * g));
            }
            tc::tmem_ld_wait();
            tc::tc_fence_before();
            tc::mbar_arrive(hempty);  // H / I may now take the next tile's MMAs
#pragma unroll
            for (int e = 0; e < N / 2; ++e) hv[e] = (hv[e] + wint * iv[e]) * inv_den;
#pragma unroll
            for (int q = 0; q < N / 16; ++q)
                tc::sw128_store8(stg, row, half * (N / 16) + q, 128, hv + 8 * q);
            }
            tc::fence_proxy_async_smem();
            tc::named_bar_sync(1, kEpi);
            if (et == 0) {
                for (int a = 0; a < N / 64; ++a)
                    tc::tma_store_3d(&mapH, stg + a * 16384, x0 + 64 * a, P.rows_start, bh);
                tc::tma_store_commit();
            }
            u0 += P.n_kv;
        }
        if (et == 0) tc::tma_store_wait_all<0>();
        if (stab) sl.flush(args.gw.stab);
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

template <int N>
int launch_impl(const FwdArgs& a, const void* k, const void* v, const void* states, void* h,
                cudaStream_t st) {
    using namespace tfla_host;
    const Geom& g = a.g;
    CUtensorMap mq, mk, mv, mc, mh;
    if (!make_tmap_bf16_3d(&mq, a.q, g.BH, g.T, g.dqk, 64, 128) ||
        !make_tmap_bf16_3d(&mk, k, g.BH, g.T, g.dqk, 64, 128) ||
        !make_tmap_bf16_3d(&mv, v, g.BH, g.T, g.dhv, 64, 64) ||
        !make_tmap_bf16_3d(&mc, states, static_cast<uint64_t>(g.BH) * g.NC, g.dqk, g.dhv, 64, 64) ||
        !make_tmap_bf16_3d(&mh, h, g.BH, g.T, g.dhv, 64, 128))
        return 4;
    constexpr int kSmemBytes = Ring<N>::kSmemBytes;
    tfla_host::ensure_smem_attr(reinterpret_cast<const void*>(fwd_parallel_kernel<N>), kSmemBytes);
    static int num_sms = 0;
    if (!num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int n_tiles = (g.dhv / N) * ((g.T + 127) / 128) * g.BH;
    (void)num_sms;
    // grid coprime to the (x tile x tile-in-chunk) period: balanced static striding
    const int grid = tfla_host::coprime_grid(n_tiles, (g.dhv / N) * (g.L >= 128 ? g.L / 128 : 1));
    fwd_parallel_kernel<N><<<grid, kThreads, kSmemBytes, st>>>(
        mq, mk, mv, mc, mh, a);
    return 0;
}

// qn[t] = q_t . n_{c(t)} (the normaliser's inter-chunk term, chunkwise.cpp:153-159).
// A streaming pass over q: each warp takes 4 rows per step (4 independent
// 16-B loads in flight per lane, then 4 interleaved shuffle reductions), n_k
// staged in shared memory (d_qk <= 512).
__global__ void qn_kernel(const __nv_bfloat16* __restrict__ q, const float* __restrict__ n_states,
                          float* __restrict__ qn, int T, int L, int NC, int dqk) {
    extern __shared__ float nsh[];
    const int c = blockIdx.x, bh = blockIdx.y;
    const float* n = n_states + (static_cast<size_t>(bh) * (NC + 1) + c) * dqk;
    for (int p = threadIdx.x; p < dqk; p += blockDim.x) nsh[p] = n[p];
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const size_t base = static_cast<size_t>(bh) * T + static_cast<size_t>(c) * L;
    for (int r0 = wid * 4; r0 < L; r0 += nw * 4) {
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        for (int p = lane * 8; p < dqk; p += 256) {
            uint4 raw[4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
                raw[i] = r0 + i < L ? __ldcs(reinterpret_cast<const uint4*>(q + (base + r0 + i) * dqk + p))
                                    : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&raw[i]);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 f = __bfloat1622float2(h2[e]);
                    acc[i] = fmaf(f.x, nsh[p + 2 * e], acc[i]);
                    acc[i] = fmaf(f.y, nsh[p + 2 * e + 1], acc[i]);
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
        if (lane < 4 && r0 + lane < L) {
            const float v = lane == 0 ? acc[0] : lane == 1 ? acc[1] : lane == 2 ? acc[2] : acc[3];
            qn[base + r0 + lane] = v;
        }
    }
}

}  // namespace

void launch_qn(const Geom& g, const __nv_bfloat16* q, const float* n_states, float* qn, cudaStream_t st) {
    qn_kernel<<<dim3(g.NC, g.BH), 256, g.dqk * sizeof(float), st>>>(q, n_states, qn, g.T, g.L, g.NC, g.dqk);
}

int launch_fwd_parallel(const FwdArgs& a, const void* k, const void* v, const void* states,
                        void* h, cudaStream_t st) {
    if (a.ntile == 128 && a.g.L >= 128 && a.g.dhv % 256 == 0 && !tfla_host::env_flag("TFLA_NO_WIDE_FWD"))
        return launch_impl<256>(a, k, v, states, h, st);
    return a.ntile == 128 ? launch_impl<128>(a, k, v, states, h, st)
                          : launch_impl<64>(a, k, v, states, h, st);
}

}  // namespace tfla_k
