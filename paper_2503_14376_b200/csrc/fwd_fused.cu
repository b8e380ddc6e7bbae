// fwd_fused.cu -- K12: fused recurrent + parallel TFLA forward for L = 128.
//
// One CTA owns one (head, 128-column d_hv tile) and walks the chunks of its
// head in order, keeping the fp32 inter-chunk state C[:, x tile] resident in
// TMEM for the whole sequence. Per chunk k it computes, on tcgen05:
//   H_k      = Sbar_k V_k + (w o Q_k) C_k          (intra + inter, one accumulator)
//   C_{k+1}  = gbar_k C_k + (a_bar o K_k)^T V_k    (state_recurrence_head, chunkwise.cpp:13-68)
//   S_{k+1}  = Q_{k+1} K_{k+1}^T                   (next chunk's scores)
// with Sbar_ij = S_ij exp(b_i - b_j + ib_j - m_c,i) / sqrt(d) for j <= i and
// w_i = b_bar_i / sqrt(d) (chunkwise.cpp:99-180, tiled.cpp:59-240), so the state
// never makes an HBM round trip inside the forward: C_k is written once, as the
// bf16 operand copy the backward consumes (and as fp32 reference-layout
// states only when the caller asks for them). Compared with K1 + K2 this
// removes the state read (one bf16 state sweep) and the second read of k, v.
//
// The mLSTMexp normaliser runs on the tensor core too: u_k = K_k^T a_bar
// (n_{k+1} = gbar_k n_k + u_k, chunkwise.cpp:53-65) and w o (Q_k n_k) (the
// denominator's inter term, chunkwise.cpp:153-165) are two N = 16 MMAs.
//
// TMEM (512 columns): C halves [0, 128P) | H [128P, +128) | S [128P+128, +128);
// Sbar overwrites S as packed bf16 (A-from-TMEM operand of Sbar V) in the first
// 64 S columns; w q.n uses S columns 64..79 until S_{k+1} is issued, u the
// first 16P H columns between the H_k drain and Sbar V_{k+1}.
// Shared memory: 3-stage ring of 32 KB stages (two 64-column SW128 atoms),
// the bf16 C_k operand tile (MN-major, P*32 KB), V_k (32 KB; scaled by a_bar
// in place for the C update), a 16 KB h staging atom, and the small a_bar / n_k
// operand tiles of the N = 16 MMAs.
//
// Warps: 0 TMA producer, 1 tcgen05 issuer, 2..5 transform (row gate w on the
// streamed Q stages, a_bar on the rows of V_k, bf16x2 math), 6..13 C round trip (the
// recurrence's critical chain: C_{k+1} -> bf16 operand + saved state, TMEM C
// *= gbar, n update, V_{k+1} load), 14..17 one thread per row: gating (Sbar in
// place) and the H drain. MMA order per chunk: Sbar V_k, QC_k (+ q.n), S_{k+1},
// C update_k (+ u): S_{k+1} only waits for q.n to be read out, so the next
// chunk's scores and gating overlap the C update and the C round trip.
#include <cstdlib>

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "fwd_fused.h"
#include "host_util.h"
#include "stab.cuh"
#include "tc.cuh"

namespace tfla_k {
namespace {

constexpr int kR = 3;                 // ring stages
constexpr int kAtom = 128 * 64 * 2;   // one [128 rows][64 cols] SW128 atom (16 KB)
constexpr int kStage = 2 * kAtom;     // 32 KB
constexpr int kTr = 128;              // transform threads (warps 2..5)
constexpr int kCw = 256;              // C round-trip threads (warps 6..13)
constexpr int kHs = 128;              // gating / H-drain threads (warps 14..17)
constexpr int kThreads = 64 + kTr + kCw + kHs;
constexpr float kLog2e = 1.4426950408889634f;
constexpr int kTrEv = 32;             // debug trace events per chunk

template <int P>
struct FSmem {
    static constexpr int kOffCb = kR * kStage;
    static constexpr int kOffV = kOffCb + P * 2 * kAtom;
    static constexpr int kOffHst = kOffV + 2 * kAtom;     // h staging: one 64-column atom
    static constexpr int kOffOnes = kOffHst + kAtom;      // K-major [16][128] ones (2 atoms of 2 KB)
    static constexpr int kOffNb = kOffOnes + 2 * 2048;    // K-major [16][128P] n_k (row 0)
    static constexpr int kOffF = kOffNb + 2 * P * 2048;
    // floats: colv[2][128] | fw[2 buf][2 (w, a_bar)][128][2] (bf16x2 hi | lo split factors)
    static constexpr int kNF = 2 * 128 + 8 * 128;
    // fused output epilogue: the row sums of squares of up to 3 peer x tiles
    static constexpr int kOffX = kOffF + kNF * 4;
    static constexpr int kOffBar = kOffX + 3 * 128 * 4;
    static constexpr int kBytes = kOffBar + 256;
    static_assert(kBytes <= 232448, "shared memory budget");
};

// Stage schedule (shared by producer, transform warps and MMA issuer):
//   pre:      S_0 stages          2P x kind 0 (Q atom a | K atom a), raw
//   chunk k:  QC_k stages          P x kind 1 (Q atoms 2h, 2h+1), rows * w     (transformed)
//             S_{k+1} stages      2P x kind 0 (only when k + 1 < NC)
//             Cupd_k stages        P x kind 2 (K atoms 2h, 2h+1), raw: a_bar is applied
//                                  to the rows of V_k instead (in place, once Sbar V_k
//                                  has read it), off the recurrence's critical chain
// Every waiter observes every phase of the barrier it waits on, in order (a
// parity wait that skips phases can alias): raw stages land on full[s] (MMA
// waits), transformed stages on xfull[s] (transform warps wait), the
// transform signals tfull[s] (MMA waits); parities are tracked per slot.

template <int P>
__global__ void __launch_bounds__(kThreads, 1)
    fwd_fused_kernel(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapK,
                     const __grid_constant__ CUtensorMap mapV, const __grid_constant__ CUtensorMap mapS,
                     const __grid_constant__ CUtensorMap mapH, const __grid_constant__ CUtensorMap mapQs,
                     const __grid_constant__ CUtensorMap mapKs, FusedFwdArgs args) {
    using SM = FSmem<P>;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* ring = smem;
    uint8_t* cb = smem + SM::kOffCb;
    uint8_t* vb = smem + SM::kOffV;
    uint8_t* hst = smem + SM::kOffHst;
    uint8_t* ones = smem + SM::kOffOnes;
    uint8_t* nb = smem + SM::kOffNb;
    float* colv = reinterpret_cast<float*>(smem + SM::kOffF);  // [2][128]
    uint32_t* fw = reinterpret_cast<uint32_t*>(colv + 2 * 128);  // [2][2][128][2]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::kOffBar);
    uint64_t* full = bars;               // [kR] TMA landed (raw stages)
    uint64_t* xfull = full + kR;         // [kR] TMA landed (transformed stages)
    uint64_t* tfull = xfull + kR;        // [kR] transform done
    uint64_t* empty = tfull + kR;        // [kR] MMA consumed
    uint64_t* vfull = empty + kR;
    uint64_t* sfull = vfull + 1;         // S_k accumulated
    uint64_t* bfull = sfull + 1;         // Sbar_k written (TMEM)
    uint64_t* hfull = bfull + 1;         // H_k (and w q.n) accumulated
    uint64_t* hempty = hfull + 1;        // H_k (and w q.n) drained
    uint64_t* cfull = hempty + 1;        // C_{k+1}, u_k accumulated (QC_k done: Cb free)
    uint64_t* cready = cfull + 1;        // Cb_k, n_k operand written, TMEM C scaled by gbar_k
    uint64_t* uread = cready + 1;        // u_k read out of TMEM
    uint64_t* vread = uread + 1;         // Sbar V_k done reading V_k (raw)
    uint64_t* vtr = vread + 1;           // V_k rows scaled by a_bar (and a_bar row written)
    uint64_t* nread = vtr + 1;           // w q.n_k read out of TMEM (S_{k+1} may overwrite it)
    uint64_t* hlo = nread + 1;           // H_k columns 0..63 read (u_k may overwrite them)
    uint64_t* ofull = hlo + 1;           // output epilogue: peers' row sums of chunk k landed
    uint64_t* ofree = ofull + 1;         // output epilogue: peers consumed this CTA's row sums
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ofree + 1);
    float* xbuf = reinterpret_cast<float*>(smem + SM::kOffX);  // [ocl - 1][128] peer row sums

    const Geom& G = args.g;
    const int T = G.T, NC = G.NC, dqk = G.dqk, dhv = G.dhv;
    const int nxt = dhv / 128;
    const int xt = blockIdx.x % nxt, bh = blockIdx.x / nxt;
    const int x0 = xt * 128;
    const bool is_exp = args.variant == 0;
    const int warp = tc::warp_id();
    constexpr uint32_t colC = 0, colH = 128 * P, colS = 128 * P + 128;
    constexpr uint32_t colN = colS + 64, colU = colH;  // w q.n (16) in S | u halves (16 each) in H
    constexpr int kPerChunk = 4 * P;
    const int n_stages = 2 * P + NC * 2 * P + (NC - 1) * 2 * P;
    // Q/K stage sharing: the ncl x-tile CTAs of a head form a cluster; CTA r
    // loads rows [r*128/ncl, (r+1)*128/ncl) of every Q/K atom and multicasts them
    const int ncl = args.cluster > 1 ? args.cluster : 1;
    const uint16_t cl_mask = static_cast<uint16_t>((1u << ncl) - 1);
    const int cl_rank = ncl > 1 ? static_cast<int>(tc::cluster_ctarank()) : 0;
    const int sl_rows = 128 / ncl;
    long long* trace = (args.trace && static_cast<int>(blockIdx.x) == args.trace_cta) ? args.trace : nullptr;
#define TRACE(k, ev)                                      \
    do {                                                  \
        if (trace) trace[(k) * kTrEv + (ev)] = clock64(); \
    } while (0)

    if (threadIdx.x == 0) {
        if (tc::smem_u32(smem) & 1023) __trap();
        for (int s = 0; s < kR; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&xfull[s], 1);
            tc::mbar_init(&tfull[s], kTr);
            tc::mbar_init(&empty[s], ncl);  // every CTA of the cluster frees the slot
        }
        tc::mbar_init(vfull, 1);
        tc::mbar_init(sfull, 1);
        tc::mbar_init(bfull, kHs);
        tc::mbar_init(hfull, 1);
        tc::mbar_init(hempty, kHs);
        tc::mbar_init(cfull, 1);
        tc::mbar_init(cready, kCw);
        tc::mbar_init(uread, kCw);
        tc::mbar_init(vread, 1);
        tc::mbar_init(vtr, kTr);
        tc::mbar_init(nread, kHs);
        tc::mbar_init(hlo, kHs);
        const int npeer = args.ocl > 1 ? args.ocl - 1 : 1;
        tc::mbar_init(ofull, npeer * kHs);
        tc::mbar_init(ofree, npeer * kHs);
        tc::fence_barrier_init();
    }
    // constant operand tiles of the N = 16 MMAs: ones (rows 0..15 all 1) and n_0 = 0
    {
        const uint4 one4 = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
        for (int i = threadIdx.x; i < 2 * 2048 / 16; i += blockDim.x) reinterpret_cast<uint4*>(ones)[i] = one4;
        for (int i = threadIdx.x; i < 2 * P * 2048 / 16; i += blockDim.x)
            reinterpret_cast<uint4*>(nb)[i] = make_uint4(0, 0, 0, 0);
        tc::fence_proxy_async_smem();
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
    tc::tc_fence_before();
    __syncthreads();
    if (ncl > 1 || args.ocl > 1) tc::cluster_sync();  // peers' barriers are initialised before any multicast / arrive
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // stage gi -> (kind, chunk, index within its group)
    auto stage_info = [&](int gi, int& kind, int& c, int& idx) {
        if (gi < 2 * P) {
            kind = 0;
            c = 0;
            idx = gi;
            return;
        }
        const int r = gi - 2 * P;
        const int k = r / kPerChunk, w = r % kPerChunk;  // the last chunk has no S stages
        const int ns = k + 1 < NC ? 2 * P : 0;
        if (w < P) {
            kind = 1;
            c = k;
            idx = w;
        } else if (w < P + ns) {
            kind = 0;
            c = k + 1;
            idx = w - P;
        } else {
            kind = 2;
            c = k;
            idx = w - P - ns;
        }
    };

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (tc::elect_one()) {
            auto load_v = [&](int c) {
                tc::mbar_arrive_expect_tx(vfull, 2 * kAtom);
                for (int a = 0; a < 2; ++a) tc::tma_load_3d(vb + a * kAtom, &mapV, vfull, x0 + 64 * a, c * 128, bh);
            };
            load_v(0);  // V_{k+1} is loaded by the C round trip once C update_k is done
            for (int gi = 0; gi < n_stages; ++gi) {
                int kind, c, idx;
                stage_info(gi, kind, c, idx);
                if (kind == 1 && idx == 0 && c + 1 < NC) {  // warm L2 for the next chunk
                    for (int a = 0; a < 2 * P && cl_rank == 0; ++a) {
                        tc::tma_prefetch_3d(&mapQ, 64 * a, (c + 1) * 128, bh);
                        tc::tma_prefetch_3d(&mapK, 64 * a, (c + 1) * 128, bh);
                    }
                    for (int a = 0; a < 2; ++a) tc::tma_prefetch_3d(&mapV, x0 + 64 * a, (c + 1) * 128, bh);
                }
                const int s = gi % kR;
                // trace: 24/25 QC stage 0, 26/27 Cupd stage 0, 28/29 first and 30/31 last
                // S_{c} stage (recorded under chunk c - 1): before / after the slot wait
                int pev = -1, tk = c;
                if (kind == 1 && idx == 0) pev = 24;
                if (kind == 2 && idx == 0) pev = 26;
                if (kind == 0 && c > 0 && (idx == 0 || idx == 2 * P - 1)) {
                    pev = idx == 0 ? 28 : 30;
                    tk = c - 1;
                }
                if (pev >= 0) TRACE(tk, pev);
                tc::mbar_wait(&empty[s], ((gi / kR) & 1) ^ 1);
                if (pev >= 0) TRACE(tk, pev + 1);
                uint8_t* st = ring + s * kStage;
                uint64_t* fb = kind == 1 ? &xfull[s] : &full[s];
                tc::mbar_arrive_expect_tx(fb, kStage);  // all slices land here, from every CTA
                // (atom 0 | atom 1) = (Q a | K a) for S, (Q|K 2h | Q|K 2h+1) for QC / Cupd
                const CUtensorMap* m0 = kind == 2 ? &mapK : &mapQ;
                const CUtensorMap* m1 = kind == 1 ? &mapQ : &mapK;
                const int col0 = kind == 0 ? 64 * idx : 64 * (2 * idx), col1 = kind == 0 ? 64 * idx : 64 * (2 * idx + 1);
                if (ncl == 1) {
                    tc::tma_load_3d(st, m0, fb, col0, c * 128, bh);
                    tc::tma_load_3d(st + kAtom, m1, fb, col1, c * 128, bh);
                } else {
                    const int r0s = cl_rank * sl_rows;
                    tc::tma_load_3d_mc(st + r0s * 128, m0 == &mapQ ? &mapQs : &mapKs, fb, col0, c * 128 + r0s, bh,
                                       cl_mask);
                    tc::tma_load_3d_mc(st + kAtom + r0s * 128, m1 == &mapQ ? &mapQs : &mapKs, fb, col1,
                                       c * 128 + r0s, bh, cl_mask);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ tcgen05 issuer
        const uint32_t id_kk = tc::idesc_bf16(128, 128, 0, 0);  // both K-major
        const uint32_t id_kn = tc::idesc_bf16(128, 128, 0, 1);  // A K-major, B MN-major
        const uint32_t id_nn = tc::idesc_bf16(128, 128, 1, 1);  // both MN-major
        const uint32_t id_qn = tc::idesc_bf16(128, 16, 0, 0);   // w q.n: A = Qbar, B = n_k rows
        const uint32_t id_un = tc::idesc_bf16(128, 16, 1, 0);   // u: A = Kbar^T, B = ones rows
        uint32_t tpar = 0, rpar = 0;  // per-slot phase parities of tfull / full
        int gi = 0;
        // one fixed issuing lane: tcgen05.commit only tracks the MMAs of the
        // committing thread
        const bool leader = tc::elect_one();
        auto take = [&](bool transformed) -> uint32_t {
            const int s = gi % kR;
            if (transformed) {
                tc::mbar_wait(&tfull[s], (tpar >> s) & 1);
                tpar ^= 1u << s;
            } else {
                tc::mbar_wait(&full[s], (rpar >> s) & 1);
                rpar ^= 1u << s;
            }
            tc::tc_fence_after();
            return tc::smem_u32(ring + s * kStage);
        };
        auto release = [&](uint64_t* extra) {
            if (leader) {
                if (ncl > 1)
                    tc::mma_commit_mc(&empty[gi % kR], cl_mask);
                else
                    tc::mma_commit(&empty[gi % kR]);
                if (extra) tc::mma_commit(extra);
            }
            __syncwarp();
            ++gi;
        };
        auto issue_s = [&]() {  // S = Q K^T over 2P k-blocks of 64
            for (int a = 0; a < 2 * P; ++a) {
                const uint32_t st = take(false);
                if (leader) {
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks)
                        tc::mma_bf16(tmem + colS, tc::kmajor_desc(st, 128, ks), tc::kmajor_desc(st + kAtom, 128, ks),
                                     id_kk, (a | ks) ? 1u : 0u);
                }
                release(a == 2 * P - 1 ? sfull : nullptr);
            }
        };
        const uint32_t cbs = tc::smem_u32(cb), vbs = tc::smem_u32(vb);
        const uint32_t ones_s = tc::smem_u32(ones), nbs = tc::smem_u32(nb);
        const bool has_init = args.c_init != nullptr;  // C_0 != 0: the first C update accumulates
        issue_s();
        for (int k = 0; k < NC; ++k) {
            // Sbar V_k: H = Sbar_k V_k  (first write of H_k; A = Sbar from TMEM).
            // H_{k-1} drained and u_{k-1} (H columns 0..31) read out first.
            if (leader) TRACE(k, 0);
            tc::mbar_wait(bfull, k & 1);
            tc::mbar_wait(vfull, k & 1);
            if (k > 0) {
                tc::mbar_wait(hempty, (k - 1) & 1);
                if (is_exp) tc::mbar_wait(uread, (k - 1) & 1);
            }
            if (leader) TRACE(k, 1);
            tc::tc_fence_after();
            if (leader) {
#pragma unroll
                for (int ks = 0; ks < 8; ++ks)
                    tc::mma_bf16_ts(tmem + colH, tmem + colS + ks * 8, tc::mnmajor_desc(vbs, 128, ks), id_kn,
                                    ks ? 1u : 0u);
                tc::mma_commit(vread);  // V_k may now be scaled in place
            }
            __syncwarp();
            // QC_k: H += (w o Q_k) Cb_k ; w q.n_k into colN (exp)
            tc::mbar_wait(cready, k & 1);
            if (leader) TRACE(k, 2);
            tc::tc_fence_after();
            for (int h = 0; h < P; ++h) {
                const uint32_t st = take(true);
                if (leader) {
#pragma unroll
                    for (int a = 0; a < 2; ++a)
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks) {
                            const uint64_t ad = tc::kmajor_desc(st + a * kAtom, 128, ks);
                            tc::mma_bf16(tmem + colH, ad, tc::mnmajor_desc(cbs, 128 * P, (h * 128 + a * 64) / 16 + ks),
                                         id_kn, 1u);
                            if (is_exp)
                                tc::mma_bf16(tmem + colN, ad, tc::kmajor_desc(nbs, 16, h * 8 + a * 4 + ks), id_qn,
                                             (h | a | ks) ? 1u : 0u);
                        }
                }
                release(h == P - 1 ? hfull : nullptr);
            }
            if (leader) TRACE(k, 3);
            // S_{k+1}: overwrites Sbar_k (consumed by Sbar V_k, issued earlier) and
            // w q.n_k -> only the q.n read-out is waited for
            if (k + 1 < NC) {
                if (is_exp) tc::mbar_wait(nread, k & 1);
                if (leader) TRACE(k, 5);
                tc::tc_fence_after();
                issue_s();
                if (leader) TRACE(k, 6);
            }
            // C update_k: C[h] (+)= K_k[:, h]^T (a_bar o V_k) ; u_k[h] = K_k[:, h]^T a_bar into
            // H columns 0..16P-1, which the H_k drain has read first
            tc::mbar_wait(vtr, k & 1);
            if (is_exp) tc::mbar_wait(hlo, k & 1);
            tc::tc_fence_after();
            for (int h = 0; h < P; ++h) {
                const uint32_t st = take(false);
                if (leader) {
#pragma unroll
                    for (int ks = 0; ks < 8; ++ks) {
                        const uint64_t ad = tc::mnmajor_desc(st, 128, ks);
                        tc::mma_bf16(tmem + colC + h * 128, ad, tc::mnmajor_desc(vbs, 128, ks), id_nn,
                                     (k | ks || has_init) ? 1u : 0u);
                        if (is_exp)
                            tc::mma_bf16(tmem + colU + h * 16, ad, tc::kmajor_desc(ones_s, 16, ks), id_un,
                                         ks ? 1u : 0u);
                    }
                    if (h == P - 1) tc::mma_commit(cfull);  // also: V_k no longer read
                }
                release(nullptr);
            }
            if (leader) TRACE(k, 4);
        }
    } else if (warp < 6) {
        // ------------------------------------------------ transform warps
        // one thread per stage row: the 8 16-B chunks of a row are independent
        // loads (ILP), the row factor is a pre-split bf16x2 (hi, lo) pair
        const int tt = threadIdx.x - 64;  // = row of the stage atoms
        const size_t hb = static_cast<size_t>(bh) * T;
        const float rs = rsqrtf(static_cast<float>(dqk));
        uint32_t xpar = 0;  // per-slot phase parity of xfull
        // row gates (w = b_bar / sqrt(d), a_bar) of chunk c live in fw[c & 1];
        // loads go to registers one chunk ahead, the shared-memory stores happen
        // a chunk later, so the load latency never stalls a transform
        float pf_w = 0.f, pf_a = 0.f;
        auto fetch_fac = [&](int c) {
            const size_t t = hb + static_cast<size_t>(c) * 128 + tt;
            pf_w = __ldg(args.gw.bb + t) * rs;
            pf_a = __ldg(args.gw.ab + t);
        };
        auto put_fac = [&](uint32_t* dst, float f) {
            const tc::Bf16Factor bf = tc::bf16_factor(f);
            dst[0] = *reinterpret_cast<const uint32_t*>(&bf.hi);
            dst[1] = *reinterpret_cast<const uint32_t*>(&bf.lo);
        };
        fetch_fac(0);
        const int swz = tt & 7;
        for (int gi = 0; gi < n_stages; ++gi) {
            int kind, c, idx;
            stage_info(gi, kind, c, idx);
            if (kind != 1) continue;
            if (idx == 0) {
                put_fac(fw + (((c & 1) * 2 + 0) * 128 + tt) * 2, pf_w);
                put_fac(fw + (((c & 1) * 2 + 1) * 128 + tt) * 2, pf_a);
                tc::named_bar_sync(2, kTr);  // fw[c & 1] complete; fw[(c + 1) & 1] no longer read
                if (c + 1 < NC) fetch_fac(c + 1);
            }
            const int s = gi % kR;
            if (tt == 0 && idx == 0) TRACE(c, 16 + (kind - 1) * 2);
            tc::mbar_wait(&xfull[s], (xpar >> s) & 1);
            if (tt == 0 && idx == 0) TRACE(c, 17 + (kind - 1) * 2);
            if (tt == 0 && kind == 1 && idx == 1) TRACE(c, 21);
            xpar ^= 1u << s;
            const uint2 fr = *reinterpret_cast<const uint2*>(fw + (((c & 1) * 2 + (kind == 1 ? 0 : 1)) * 128 + tt) * 2);
            tc::Bf16Factor f;
            f.hi = *reinterpret_cast<const __nv_bfloat162*>(&fr.x);
            f.lo = *reinterpret_cast<const __nv_bfloat162*>(&fr.y);
            uint8_t* rowp = ring + s * kStage + tt * 128;
#pragma unroll
            for (int a = 0; a < 2; ++a) {
                // chunk order rotated by row & 7: each 8-row access phase hits 8
                // distinct 16-B bank groups (conflict-free)
                uint4 v[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) v[q] = *reinterpret_cast<const uint4*>(rowp + a * kAtom + ((q ^ swz) * 16));
#pragma unroll
                for (int q = 0; q < 8; ++q) tc::scale_chunk(v[q], f);
#pragma unroll
                for (int q = 0; q < 8; ++q) *reinterpret_cast<uint4*>(rowp + a * kAtom + ((q ^ swz) * 16)) = v[q];
            }
            if (tt == 0 && kind == 1) TRACE(c, 10 + 2 * idx);  // loop done (q stage idx)
            tc::fence_proxy_async_smem();
            if (tt == 0 && kind == 1) TRACE(c, 11 + 2 * idx);  // fence done
            tc::mbar_arrive(&tfull[s]);
            if (idx == P - 1) {
                // V_k row j *= a_bar_j in place once Sbar V_k has read it (C update_k
                // consumes it with the raw K_k stages); a_bar_j also goes to row 0 of
                // the K-major [16][128] B tile of the u_k = K_k^T a_bar MMA
                if (tt == 0) TRACE(c, 18);
                tc::mbar_wait(vread, c & 1);
                if (tt == 0) TRACE(c, 19);
                const uint2 fa = *reinterpret_cast<const uint2*>(fw + (((c & 1) * 2 + 1) * 128 + tt) * 2);
                tc::Bf16Factor fv;
                fv.hi = *reinterpret_cast<const __nv_bfloat162*>(&fa.x);
                fv.lo = *reinterpret_cast<const __nv_bfloat162*>(&fa.y);
                uint8_t* vrow = vb + tt * 128;
#pragma unroll
                for (int a = 0; a < 2; ++a) {
                    uint4 v[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) v[q] = *reinterpret_cast<const uint4*>(vrow + a * kAtom + ((q ^ swz) * 16));
#pragma unroll
                    for (int q = 0; q < 8; ++q) tc::scale_chunk(v[q], fv);
#pragma unroll
                    for (int q = 0; q < 8; ++q) *reinterpret_cast<uint4*>(vrow + a * kAtom + ((q ^ swz) * 16)) = v[q];
                }
                const float abar = __bfloat162float(fv.hi.x) + __bfloat162float(fv.lo.x);
                reinterpret_cast<__nv_bfloat16*>(ones + (tt >> 6) * 2048)[tt & 63] = __float2bfloat16_rn(abar);
                tc::fence_proxy_async_smem();
                tc::mbar_arrive(vtr);
                if (tt == 0) TRACE(c, 20);
            }
        }
    } else if (warp < 14) {
        // ------------------------------------------------ C round trip (critical chain)
        const int ct = threadIdx.x - 192;
        const int lane = tc::lane_id();
        const int row = (warp & 3) * 32 + lane;
        const uint32_t trow = tc::tmem_row_addr(tmem);
        const int half = (warp - 6) >> 2;
        // ownership: P = 2 -> state row half*128 + row, all 128 columns;
        //            P = 1 -> state row `row`, columns [half*64, +64)
        const int prow = P == 2 ? half * 128 + row : row;
        const int pcol0 = P == 2 ? 0 : half * 64;
        constexpr int kRtG = P == 2 ? 4 : 2;  // 32-column groups per thread
        const uint32_t taC = trow + colC + (P == 2 ? half * 128 : 0) + pcol0;
        const bool n_owner = is_exp && (P == 2 || half == 0);
        const bool write_n = n_owner && xt == 0 && args.n_states != nullptr && prow < dqk;
        const bool write_nf = n_owner && xt == 0 && args.n_final != nullptr && prow < dqk;
        // n_k operand: K-major [16 rows][128P], row 0 = bf16(n_k); element (0, p)
        __nv_bfloat16* nb_elem = reinterpret_cast<__nv_bfloat16*>(
            nb + (prow >> 6) * 2048 + (((prow & 63) >> 3) * 16) + (prow & 7) * 2);
        auto store_cb = [&](int c) {  // TMA store of the bf16 C_c operand tile (saved state)
            if (ct == 0) {
                for (int a = 0; a < 2; ++a)
                    for (int h = 0; h < P; ++h)
                        tc::tma_store_3d(&mapS, cb + a * (128 * P * 128) + h * kAtom, x0 + 64 * a, h * 128,
                                         bh * NC + c);
                tc::tma_store_commit();
            }
        };
        auto write_f32_state = [&](float* dst, const float* v, int g) {
            float* d = dst + static_cast<size_t>(prow) * dhv + x0 + pcol0 + g * 32;
#pragma unroll
            for (int i = 0; i < 32; i += 4)
                *reinterpret_cast<float4*>(d + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
        };
        const float* gbar = args.gw.gbar + static_cast<size_t>(bh) * NC;
        float gb_k = __ldg(gbar);                        // gbar_k (n update)
        float gb_next = NC > 1 ? __ldg(gbar + 1) : 0.f;  // gbar_{k+1} (C scaling)
        // prologue: C_0 (zero, or the caller's initial state) -> operand tile, saved
        // state, optional fp32 states; TMEM C = gbar_0 C_0; n_0 likewise
        if (!args.c_init) {
            for (int i = ct; i < P * 2 * kAtom / 16; i += kCw) reinterpret_cast<uint4*>(cb)[i] = make_uint4(0, 0, 0, 0);
        }
        for (int g = 0; g < kRtG; ++g) {
            float v[32];
            if (args.c_init && prow < dqk) {
                const float* src = args.c_init + (static_cast<size_t>(bh) * dqk + prow) * dhv + x0 + pcol0 + g * 32;
#pragma unroll
                for (int i = 0; i < 32; i += 4) {
                    const float4 f4 = *reinterpret_cast<const float4*>(src + i);
                    v[i] = f4.x, v[i + 1] = f4.y, v[i + 2] = f4.z, v[i + 3] = f4.w;
                }
            } else {
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = 0.f;
            }
            if (args.c_states && prow < dqk)
                write_f32_state(args.c_states + static_cast<size_t>(bh) * (NC + 1) * dqk * dhv, v, g);
            if (args.c_init) {
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    tc::sw128_store8(cb, prow, (pcol0 + g * 32) / 8 + q, 128 * P, v + 8 * q);
                uint32_t sc[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) sc[i] = __float_as_uint(v[i] * gb_k);
                tc::tmem_st32(taC + g * 32, sc);
            }
        }
        float n_reg = (n_owner && args.n_init && prow < dqk) ? args.n_init[static_cast<size_t>(bh) * dqk + prow] : 0.f;
        if (write_n) args.n_states[static_cast<size_t>(bh) * (NC + 1) * dqk + prow] = n_reg;
        if (n_owner && args.n_init) *nb_elem = __float2bfloat16_rn(n_reg);
        if (args.c_init) tc::tmem_st_wait();
        tc::fence_proxy_async_smem();
        tc::tc_fence_before();
        tc::mbar_arrive(cready);
        tc::named_bar_sync(1, kCw);
        store_cb(0);
        for (int k = 0; k < NC; ++k) {
            const bool last = k + 1 == NC;
            const float gb = gb_next;
            const float gbn = gb_k;
            gb_k = gb_next;
            if (k + 2 < NC) gb_next = __ldg(gbar + k + 2);
            if (!last && ct == 0) tc::tma_store_wait_read<0>();  // saved-state store of Cb_k
            if (ct == 0) TRACE(k, 7);
            tc::mbar_wait(cfull, k & 1);
            if (ct == 0) TRACE(k, 8);
            tc::tc_fence_after();
            if (!last && ct == 0) {  // C update_k was V_k's last reader: stream in V_{k+1}
                tc::mbar_arrive_expect_tx(vfull, 2 * kAtom);
                for (int a = 0; a < 2; ++a)
                    tc::tma_load_3d(vb + a * kAtom, &mapV, vfull, x0 + 64 * a, (k + 1) * 128, bh);
            }
            // n_{k+1} = gbar_k n_k + u_k (exp): u read first, S_{k+1} waits for it
            if (is_exp) {
                const float u = tc::tmem_ld1(trow + colU + (P == 2 ? half * 16 : 0));
                tc::tmem_ld_wait();
                if (n_owner) {
                    n_reg = fmaf(gbn, n_reg, u);
                    if (write_n) args.n_states[(static_cast<size_t>(bh) * (NC + 1) + k + 1) * dqk + prow] = n_reg;
                    if (write_nf && last) args.n_final[static_cast<size_t>(bh) * dqk + prow] = n_reg;
                    if (!last) *nb_elem = __float2bfloat16_rn(n_reg);
                }
            }
            tc::tc_fence_before();
            if (is_exp && !last) tc::mbar_arrive(uread);  // exactly the phases Sbar V_{k+1} waits for
            if (!last) tc::named_bar_sync(1, kCw);
            float* cs = args.c_states ? args.c_states + (static_cast<size_t>(bh) * (NC + 1) + k + 1) * dqk * dhv : nullptr;
            float* cf = last && args.c_final ? args.c_final + static_cast<size_t>(bh) * dqk * dhv : nullptr;
#pragma unroll 1
            for (int g = 0; g < kRtG; g += 2) {
                float v[2][32];
                tc::tmem_ld32(taC + g * 32, v[0]);
                tc::tmem_ld32(taC + g * 32 + 32, v[1]);
                tc::tmem_ld_wait();
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    if (prow < dqk) {
                        if (cs) write_f32_state(cs, v[u], g + u);
                        if (cf) write_f32_state(cf, v[u], g + u);
                    }
                    if (!last) {
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            tc::sw128_store8(cb, prow, (pcol0 + (g + u) * 32) / 8 + q, 128 * P, v[u] + 8 * q);
                        uint32_t sc[32];
#pragma unroll
                        for (int i = 0; i < 32; ++i) sc[i] = __float_as_uint(v[u][i] * gb);
                        tc::tmem_st32(taC + (g + u) * 32, sc);
                    }
                }
            }
            if (!last) {
                tc::tmem_st_wait();
                tc::fence_proxy_async_smem();
                tc::tc_fence_before();
                tc::mbar_arrive(cready);
                if (ct == 0) TRACE(k, 9);
                tc::named_bar_sync(1, kCw);
                store_cb(k + 1);
            }
        }
        if (ct == 0) tc::tma_store_wait_all<0>();
    } else {
        // ------------------------------------------------ gating + H drain, one thread per row
        const int ht = threadIdx.x - 448;
        const int lane = tc::lane_id();
        const int row = (warp & 3) * 32 + lane;
        const uint32_t trow = tc::tmem_row_addr(tmem);
        const size_t hb = static_cast<size_t>(bh) * T;
        const float rs = rsqrtf(static_cast<float>(dqk));
        const bool write_den = xt == 0 && args.h_denom != nullptr;
        struct Gv {
            float b, mc, col;
        };
        auto fetch = [&](int c) {  // row gates of chunk c (and this row's column term)
            Gv g;
            const size_t t = hb + static_cast<size_t>(c) * 128 + row;
            g.b = args.gw.b[t];
            g.mc = args.gw.mc[t];
            g.col = (args.gw.ib[t] - g.b) * kLog2e;
            return g;
        };
        // Sbar_c = S_c * gates (packed bf16, written in place over the S columns
        // this thread already read; column groups above the diagonal are zero)
        StabLocal sl;
        const bool stab = is_exp && xt == 0 && args.gw.stab != nullptr;
        auto gating = [&](int c, const Gv& g) -> float {
            const float rowterm = (is_exp ? g.b - g.mc : g.b) * kLog2e;
            float* cv = colv + (c & 1) * 128;
            cv[row] = g.col;
            tc::named_bar_sync(3, kHs);
            tc::mbar_wait(sfull, c & 1);
            tc::tc_fence_after();
            float rsum = 0.f;
#pragma unroll 1
            for (int gq = 0; gq < 4; ++gq) {
                uint32_t pk[16];
                if (gq * 32 > row) {
#pragma unroll
                    for (int e = 0; e < 16; ++e) pk[e] = 0u;
                } else {
                    float v[32];
                    tc::tmem_ld32(trow + colS + gq * 32, v);
                    tc::tmem_ld_wait();
                    if (stab)
                        for (int j = gq * 32; j < gq * 32 + 32 && j <= row; ++j) sl.note(rowterm + cv[j]);
#pragma unroll
                    for (int e = 0; e < 32; e += 2) {
                        const int j = gq * 32 + e;
                        const float w0 = j <= row ? v[e] * rs * exp2f(fminf(rowterm + cv[j], 0.f)) : 0.f;
                        const float w1 = j + 1 <= row ? v[e + 1] * rs * exp2f(fminf(rowterm + cv[j + 1], 0.f)) : 0.f;
                        rsum += w0 + w1;
                        pk[e >> 1] = tc::pack_bf16(w0, w1);
                    }
                }
                tc::tmem_st16(trow + colS + gq * 16, pk);
            }
            tc::tmem_st_wait();
            tc::tc_fence_before();
            tc::mbar_arrive(bfull);
            return rsum;
        };
        // Fused output epilogue (args.o_pre != null): y = sigmoid(o) * h~ / rms * gamma
        // (eq. 5, rms_norm as transfer.cpp:8-18). The drain of H_k sums this
        // row's squares over the CTA's 128 columns (of the bf16 h~ it stores) and
        // sends the partial to the head's other x-tile CTAs (cluster DSMEM); after
        // gating S_{k+1} -- in the row warps' idle time before H_{k+1} is ready --
        // the row's total gives rms and y_k is formed from the stored h~_k row
        // (L2) and o_k (prefetched into L2 at the drain). Partials are summed in
        // x-tile order in every CTA, so all tiles of a row use the same rms.
        const bool fuse_out = args.o_pre != nullptr;
        const int ocl = args.ocl > 1 ? args.ocl : 1;
        const uint32_t orank = ocl > 1 ? tc::cluster_ctarank() : 0u;
        auto out_send = [&](int k, float sq) {
            if (ocl > 1) {
                if (k > 0) tc::mbar_wait_cluster(ofree, (k - 1) & 1);  // peers read chunk k-1's sums
                for (int s = 1; s < ocl; ++s) {
                    const uint32_t peer = (orank + s) % ocl;
                    const int slot = static_cast<int>((orank + ocl - peer - 1) % ocl);
                    tc::st_cluster_f32(tc::mapa_shared(tc::smem_u32(xbuf + slot * 128 + row), peer), sq);
                    tc::mbar_arrive_cluster(tc::mapa_shared(tc::smem_u32(ofull), peer));
                }
            }
            const __nv_bfloat16* orow = args.o_pre + (hb + static_cast<size_t>(k) * 128 + row) * dhv + x0;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(orow));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(orow + 64));
        };
        auto out_finish = [&](int k, float sq) {
            float tot = sq;
            if (ocl > 1) {
                tc::mbar_wait_cluster(ofull, k & 1);
                tot = 0.f;
                for (int r = 0; r < ocl; ++r)
                    tot += r == static_cast<int>(orank) ? sq
                                                        : xbuf[((r - static_cast<int>(orank) - 1 + 2 * ocl) % ocl) * 128 + row];
                for (int s = 1; s < ocl; ++s)
                    tc::mbar_arrive_cluster(tc::mapa_shared(tc::smem_u32(ofree), (orank + s) % ocl));
            }
            const float rms = sqrtf(tot / static_cast<float>(dhv) + args.eps);
            const float irms = rms == 0.f ? 0.f : 1.f / rms;
            // h~_k left by TMA store: complete before the rows are read back
            if (ht == 0) {
                tc::tma_store_wait_all<0>();
                asm volatile("fence.proxy.async.global;" ::: "memory");
            }
            tc::named_bar_sync(3, kHs);
            // y rows of this warp's 32 rows, one row per iteration: the 32 lanes
            // cover the row's 128 columns (8 B each), so every access is one
            // coalesced 256-B segment; the row's 1 / rms comes from its owner lane
            const int lane4 = lane * 4;
            const float4 gv = __ldg(reinterpret_cast<const float4*>(
                args.gamma + static_cast<size_t>(bh % args.n_head) * dhv + x0 + lane4));
            const size_t rbase = (hb + static_cast<size_t>(k) * 128 + (warp & 3) * 32) * dhv + x0 + lane4;
#pragma unroll 8
            for (int r = 0; r < 32; ++r) {
                const float ir = __shfl_sync(0xffffffffu, irms, r);
                const size_t off = rbase + static_cast<size_t>(r) * dhv;
                const uint2 xv = __ldcg(reinterpret_cast<const uint2*>(args.h + off));
                const uint2 ov = __ldcs(reinterpret_cast<const uint2*>(args.o_pre + off));
                const __nv_bfloat162* x2 = reinterpret_cast<const __nv_bfloat162*>(&xv);
                const __nv_bfloat162* o2 = reinterpret_cast<const __nv_bfloat162*>(&ov);
                const float gg[4] = {gv.x, gv.y, gv.z, gv.w};
                uint2 yo;
                uint32_t* w = reinterpret_cast<uint32_t*>(&yo);
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const float2 xf = __bfloat1622float2(x2[e]);
                    const float2 of = __bfloat1622float2(o2[e]);
                    const float s0 = 1.f / (1.f + __expf(-of.x)), s1 = 1.f / (1.f + __expf(-of.y));
                    const __nv_bfloat162 hv = __floats2bfloat162_rn(s0 * xf.x * ir * gg[2 * e],
                                                                    s1 * xf.y * ir * gg[2 * e + 1]);
                    w[e] = *reinterpret_cast<const uint32_t*>(&hv);
                }
                __stcs(reinterpret_cast<uint2*>(args.y + off), yo);
            }
        };
        Gv gcur = fetch(0);
        float rsum = gating(0, gcur);
        Gv gnext = NC > 1 ? fetch(1) : gcur;
        for (int k = 0; k < NC; ++k) {
            const size_t t = hb + static_cast<size_t>(k) * 128 + row;
            // drain H_k (+ w q.n) in two 64-column halves through the 16 KB staging atom
            if (ht == 0) TRACE(k, 14);
            tc::mbar_wait(hfull, k & 1);
            if (ht == 0) TRACE(k, 15);
            tc::tc_fence_after();
            float den = 1.f;
            if (is_exp) {
                const float qnw = tc::tmem_ld1(trow + colN);
                tc::tmem_ld_wait();
                den = fmaxf(fabsf(rsum + qnw), exp2f(-gcur.mc * kLog2e));
            }
            tc::tc_fence_before();
            if (is_exp && k + 1 < NC) tc::mbar_arrive(nread);  // S_{k+1} may overwrite w q.n_k
            if (write_den) args.h_denom[t] = den;
            const float inv = 1.f / den;
            float sq = 0.f;  // fused output epilogue: this row's sum of squares of h~ (as stored, bf16)
#pragma unroll 1
            for (int hh = 0; hh < 2; ++hh) {
                float v[64];
                tc::tmem_ld32(trow + colH + hh * 64, *reinterpret_cast<float(*)[32]>(v));
                tc::tmem_ld32(trow + colH + hh * 64 + 32, *reinterpret_cast<float(*)[32]>(v + 32));
                tc::tmem_ld_wait();
                tc::tc_fence_before();
                // u_k may overwrite columns 0..63 (hlo, exp) / Sbar V_{k+1} all of H (hempty)
                if (hh == 0 ? is_exp : k + 1 < NC) tc::mbar_arrive(hh == 0 ? hlo : hempty);
#pragma unroll
                for (int e = 0; e < 64; ++e) v[e] *= inv;
                if (fuse_out) {
#pragma unroll
                    for (int e = 0; e < 64; ++e) {
                        const float r = __bfloat162float(__float2bfloat16_rn(v[e]));
                        sq = fmaf(r, r, sq);
                    }
                }
                if (ht == 0) tc::tma_store_wait_read<0>();
                tc::named_bar_sync(3, kHs);
#pragma unroll
                for (int q = 0; q < 8; ++q) tc::sw128_store8(hst, row, q, 128, v + 8 * q);
                tc::fence_proxy_async_smem();
                tc::named_bar_sync(3, kHs);
                if (ht == 0) {
                    tc::tma_store_3d(&mapH, hst, x0 + 64 * hh, k * 128, bh);
                    tc::tma_store_commit();
                }
            }
            if (ht == 0) TRACE(k, 22);
            if (fuse_out) out_send(k, sq);
            if (k + 1 < NC) {
                gcur = gnext;
                rsum = gating(k + 1, gcur);
                if (ht == 0) TRACE(k, 23);
                if (k + 2 < NC) gnext = fetch(k + 2);
            }
            if (fuse_out) out_finish(k, sq);
        }
        if (ht == 0) tc::tma_store_wait_all<0>();
        if (stab) sl.flush(args.gw.stab);
    }
#undef TRACE
    tc::tc_fence_before();
    __syncthreads();
    if (ncl > 1 || args.ocl > 1) tc::cluster_sync();  // no peer multicasts into / arrives on this CTA any more
    if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

template <int P>
int launch_impl(const FusedFwdArgs& a, const void* q, const void* k, const void* v, void* saved,
                cudaStream_t st) {
    using namespace tfla_host;
    const Geom& g = a.g;
    // Optional (TFLA_FWD_MULTICAST=1): the x-tile CTAs of a head form a cluster
    // and share the Q/K stages by TMA multicast. Correct, but measured slower
    // at the 7B shape (1.06 vs 0.95 ms: the cluster lockstep on every ring slot
    // costs more than the 4x fewer L2 requests save), so off by default.
    const int nxt = g.dhv / 128;
    const int ncl = (nxt == 2 || nxt == 4 || nxt == 8) && env_flag("TFLA_FWD_MULTICAST") ? nxt : 1;
    CUtensorMap mq, mk, mv, ms, mh, mqs, mks;
    if (!make_tmap_bf16_3d(&mqs, q, g.BH, g.T, g.dqk, 64, 128 / ncl) ||
        !make_tmap_bf16_3d(&mks, k, g.BH, g.T, g.dqk, 64, 128 / ncl) ||
        !make_tmap_bf16_3d(&mh, a.h, g.BH, g.T, g.dhv, 64, 128) ||
        !make_tmap_bf16_3d(&mq, q, g.BH, g.T, g.dqk, 64, 128) ||
        !make_tmap_bf16_3d(&mk, k, g.BH, g.T, g.dqk, 64, 128) ||
        !make_tmap_bf16_3d(&mv, v, g.BH, g.T, g.dhv, 64, 128) ||
        !make_tmap_bf16_3d(&ms, saved, static_cast<uint64_t>(g.BH) * g.NC, g.dqk, g.dhv, 64, 128))
        return 4;
    constexpr int smem = FSmem<P>::kBytes;
    tfla_host::ensure_smem_attr(reinterpret_cast<const void*>(fwd_fused_kernel<P>), smem);
    FusedFwdArgs aa = a;
    aa.cluster = ncl;
    aa.ocl = a.o_pre ? nxt : 1;
    const int cdim = aa.ocl > ncl ? aa.ocl : ncl;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(g.BH * nxt);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute cl[1];
    cl[0].id = cudaLaunchAttributeClusterDimension;
    cl[0].val.clusterDim.x = cdim;
    cl[0].val.clusterDim.y = 1;
    cl[0].val.clusterDim.z = 1;
    cfg.attrs = cl;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, fwd_fused_kernel<P>, mq, mk, mv, ms, mh, mqs, mks, aa) != cudaSuccess) return 4;
    return 0;
}

}  // namespace

bool fwd_fused_supported(const Geom& g) {
    return g.L == 128 && (g.dqk == 128 || g.dqk == 256) && g.dhv % 128 == 0;
}

bool fwd_fused_out_supported(const Geom& g) {
    const int nxt = g.dhv / 128;
    return fwd_fused_supported(g) && (nxt == 1 || nxt == 2 || nxt == 4);
}

int launch_fwd_fused(const FusedFwdArgs& a, const void* q, const void* k, const void* v, void* saved,
                     cudaStream_t st) {
    return a.g.dqk == 256 ? launch_impl<2>(a, q, k, v, saved, st) : launch_impl<1>(a, q, k, v, saved, st);
}

}  // namespace tfla_k
