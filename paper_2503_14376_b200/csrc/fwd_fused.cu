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
// removes the state read (1 bf16 state sweep) and the second read of k and v.
//
// The normaliser (mLSTMexp) n_{k+1} = gbar_k n_k + K_k^T a_bar and q_i . n_k
// are accumulated on CUDA cores by the transform warps while they apply the
// row gates to the streamed Q / K tiles, so the whole forward after K0 is
// this one kernel.
//
// TMEM (512 columns): C halves [0, 128P) | H [128P, +128) | S [128P+128, +128);
// the gated scores Sbar overwrite S as packed bf16 (A-from-TMEM operand of
// Sbar V, tcgen05 "TS" form), so no shared-memory score tile is needed.
// Shared memory: 3-stage ring of 32 KB stages (two 64-column SW128 atoms),
// the bf16 C_k operand tile (MN-major, P*32 KB), the V_k tile (32 KB).
//
// Warps: 0 TMA producer, 1 tcgen05 issuer, 2..5 transform (row gates on the
// streamed Q / K stages, n and q.n), 6..13 epilogue (C round trip, gating,
// H drain). MMA order per chunk: QC_k, Sbar V_k, C update_k, S_{k+1}: the
// C chain (epilogue round trip -> QC_k + C update_k) overlaps S_{k+1} and the
// gating, so the tensor pipe stays busy while the epilogue turns C over.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "fwd_fused.h"
#include "host_util.h"
#include "tc.cuh"

namespace tfla_k {
namespace {

constexpr int kR = 3;                 // ring stages
constexpr int kAtom = 128 * 64 * 2;   // one [128 rows][64 cols] SW128 atom (16 KB)
constexpr int kStage = 2 * kAtom;     // 32 KB
constexpr int kTr = 128;              // transform threads
constexpr int kEpi = 256;             // epilogue threads
constexpr int kThreads = 64 + kTr + kEpi;
constexpr float kLog2e = 1.4426950408889634f;

template <int P>
struct FSmem {
    static constexpr int kOffCb = kR * kStage;
    static constexpr int kOffV = kOffCb + P * 2 * kAtom;
    static constexpr int kOffF = kOffV + 2 * kAtom;
    // floats: nsh[128P] | upart[2][128P] | qnp[2][2][128] | colv[128] | xred[128] | denb[128]
    //         | fw[2 buf][2 (w, a_bar)][128] (row gates of the transform warps)
    static constexpr int kNF = 128 * P + 2 * 128 * P + 4 * 128 + 3 * 128 + 4 * 128;
    static constexpr int kOffBar = kOffF + kNF * 4;
    static constexpr int kBytes = kOffBar + 320;
    static_assert(kBytes <= 232448, "shared memory budget");
};

// Stage schedule (shared by producer, transform warps and MMA issuer):
//   pre:      S_0 stages          2P x kind 0 (Q atom a | K atom a), raw
//   chunk k:  QC_k stages          P x kind 1 (Q atoms 2h, 2h+1), rows * w   (transformed)
//             Cupd_k stages        P x kind 2 (K atoms 2h, 2h+1), rows * a_bar (transformed)
//             S_{k+1} stages      2P x kind 0 (only when k + 1 < NC)

template <int P>
__global__ void __launch_bounds__(kThreads, 1)
    fwd_fused_kernel(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapK,
                     const __grid_constant__ CUtensorMap mapV, const __grid_constant__ CUtensorMap mapS,
                     const __grid_constant__ CUtensorMap mapH, FusedFwdArgs args) {
    using SM = FSmem<P>;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* ring = smem;
    uint8_t* cb = smem + SM::kOffCb;
    uint8_t* vb = smem + SM::kOffV;
    float* nsh = reinterpret_cast<float*>(smem + SM::kOffF);
    float* upart = nsh + 128 * P;        // [2][128P]
    float* qnp = upart + 2 * 128 * P;    // [2 buf][2 atom][128]
    float* colv = qnp + 4 * 128;         // [128]
    float* xred = colv + 128;            // [128]
    float* denb = xred + 128;            // [128]
    float* fw = denb + 128;              // [2][2][128]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::kOffBar);
    // Every waiter observes every phase of the barriers it waits on, in order
    // (a parity wait that skips phases can alias): raw stages land on full[s]
    // (MMA waits), transformed stages on xfull[s] (transform warps wait), the
    // transform signals tfull[s] (MMA waits); parities are tracked per slot.
    uint64_t* full = bars;               // [kR] TMA landed (raw stages)
    uint64_t* xfull = full + kR;         // [kR] TMA landed (transformed stages)
    uint64_t* tfull = xfull + kR;        // [kR] transform done
    uint64_t* empty = tfull + kR;        // [kR] MMA consumed
    uint64_t* vfull = empty + kR;
    uint64_t* vempty = vfull + 1;
    uint64_t* sfull = vempty + 1;        // S_k accumulated
    uint64_t* bfull = sfull + 1;         // Sbar_k written (TMEM)
    uint64_t* hfull = bfull + 1;         // H_k accumulated
    uint64_t* hempty = hfull + 1;        // H_k drained
    uint64_t* cfull = hempty + 1;        // C_{k+1} accumulated (QC_k done: Cb free)
    uint64_t* cready = cfull + 1;        // Cb_k written, TMEM C scaled by gbar_k
    uint64_t* qnfull = cready + 1;       // [2]
    uint64_t* qnempty = qnfull + 2;      // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(qnempty + 2);

    const Geom& G = args.g;
    const int T = G.T, NC = G.NC, dqk = G.dqk, dhv = G.dhv;
    const int nxt = dhv / 128;
    const int xt = blockIdx.x % nxt, bh = blockIdx.x / nxt;
    const int x0 = xt * 128;
    const bool is_exp = args.variant == 0;
    const int warp = tc::warp_id();
    constexpr uint32_t colC = 0, colH = 128 * P, colS = 128 * P + 128;
    constexpr int kPerChunk = 4 * P;
    const int n_stages = 2 * P + NC * 2 * P + (NC - 1) * 2 * P;

    if (threadIdx.x == 0) {
        if (tc::smem_u32(smem) & 1023) __trap();
        for (int s = 0; s < kR; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&xfull[s], 1);
            tc::mbar_init(&tfull[s], kTr);
            tc::mbar_init(&empty[s], 1);
        }
        tc::mbar_init(vfull, 1);
        tc::mbar_init(vempty, 1);
        tc::mbar_init(sfull, 1);
        tc::mbar_init(bfull, kEpi);
        tc::mbar_init(hfull, 1);
        tc::mbar_init(hempty, kEpi);
        tc::mbar_init(cfull, 1);
        tc::mbar_init(cready, kEpi);
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&qnfull[b], kTr);
            tc::mbar_init(&qnempty[b], 1);
        }
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
    tc::tc_fence_before();
    __syncthreads();
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
        const int k = r / kPerChunk, w = r % kPerChunk;
        if (w < P) {
            kind = 1;
            c = k;
            idx = w;
        } else if (w < 2 * P) {
            kind = 2;
            c = k;
            idx = w - P;
        } else {
            kind = 0;
            c = k + 1;
            idx = w - 2 * P;
        }
    };

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (tc::elect_one()) {
            auto load_v = [&](int c) {
                tc::mbar_arrive_expect_tx(vfull, 2 * kAtom);
                for (int a = 0; a < 2; ++a) tc::tma_load_3d(vb + a * kAtom, &mapV, vfull, x0 + 64 * a, c * 128, bh);
            };
            load_v(0);
            int next_v = 1;  // next V chunk to load (after vempty of chunk next_v - 1)
            for (int gi = 0; gi < n_stages; ++gi) {
                int kind, c, idx;
                stage_info(gi, kind, c, idx);
                if (kind == 1 && idx == 0 && c + 1 < NC) {  // warm L2 for the next chunk
                    for (int a = 0; a < 2 * P; ++a) {
                        tc::tma_prefetch_3d(&mapQ, 64 * a, (c + 1) * 128, bh);
                        tc::tma_prefetch_3d(&mapK, 64 * a, (c + 1) * 128, bh);
                    }
                    for (int a = 0; a < 2; ++a) tc::tma_prefetch_3d(&mapV, x0 + 64 * a, (c + 1) * 128, bh);
                }
                const int s = gi % kR;
                tc::mbar_wait(&empty[s], ((gi / kR) & 1) ^ 1);
                uint8_t* st = ring + s * kStage;
                uint64_t* fb = kind == 0 ? &full[s] : &xfull[s];
                tc::mbar_arrive_expect_tx(fb, kStage);
                if (kind == 0) {
                    tc::tma_load_3d(st, &mapQ, fb, 64 * idx, c * 128, bh);
                    tc::tma_load_3d(st + kAtom, &mapK, fb, 64 * idx, c * 128, bh);
                } else {
                    const CUtensorMap* m = kind == 1 ? &mapQ : &mapK;
                    tc::tma_load_3d(st, m, fb, 64 * (2 * idx), c * 128, bh);
                    tc::tma_load_3d(st + kAtom, m, fb, 64 * (2 * idx + 1), c * 128, bh);
                }
                // V_{c} of the chunk whose S stages were just queued: load it once
                // the previous chunk's C update released the V buffer
                if (kind == 0 && idx == 2 * P - 1 && c >= 1 && next_v == c) {
                    tc::mbar_wait(vempty, (c - 1) & 1);
                    load_v(c);
                    ++next_v;
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ tcgen05 issuer
        const uint32_t id_kk = tc::idesc_bf16(128, 128, 0, 0);  // both K-major
        const uint32_t id_kn = tc::idesc_bf16(128, 128, 0, 1);  // A K-major, B MN-major
        const uint32_t id_nn = tc::idesc_bf16(128, 128, 1, 1);  // both MN-major
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
        issue_s();
        for (int k = 0; k < NC; ++k) {
            // QC_k: H = (w o Q_k) Cb_k   (first write of H_k)
            tc::mbar_wait(cready, k & 1);
            if (k > 0) tc::mbar_wait(hempty, (k - 1) & 1);
            tc::tc_fence_after();
            for (int h = 0; h < P; ++h) {
                const uint32_t st = take(true);
                if (leader) {
#pragma unroll
                    for (int a = 0; a < 2; ++a)
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks)
                            tc::mma_bf16(tmem + colH, tc::kmajor_desc(st + a * kAtom, 128, ks),
                                         tc::mnmajor_desc(cbs, 128 * P, (h * 128 + a * 64) / 16 + ks), id_kn,
                                         (h | a | ks) ? 1u : 0u);
                }
                release(nullptr);
            }
            // Sbar V_k: H += Sbar_k V_k  (A = Sbar from TMEM, packed bf16)
            tc::mbar_wait(bfull, k & 1);
            tc::mbar_wait(vfull, k & 1);
            tc::tc_fence_after();
            if (leader) {
#pragma unroll
                for (int ks = 0; ks < 8; ++ks)
                    tc::mma_bf16_ts(tmem + colH, tmem + colS + ks * 8, tc::mnmajor_desc(vbs, 128, ks), id_kn, 1u);
                tc::mma_commit(hfull);
            }
            __syncwarp();
            // C update_k: C[h] (+)= (a_bar o K_k)[:, h]^T V_k
            for (int h = 0; h < P; ++h) {
                const uint32_t st = take(true);
                if (leader) {
#pragma unroll
                    for (int ks = 0; ks < 8; ++ks)
                        tc::mma_bf16(tmem + colC + h * 128, tc::mnmajor_desc(st, 128, ks),
                                     tc::mnmajor_desc(vbs, 128, ks), id_nn, (k | ks) ? 1u : 0u);
                    if (h == P - 1) {
                        tc::mma_commit(cfull);
                        tc::mma_commit(vempty);
                    }
                }
                release(nullptr);
            }
            // S_{k+1}: overwrites the Sbar_k columns -> Sbar V_k must have completed
            if (k + 1 < NC) {
                tc::mbar_wait(hfull, k & 1);
                tc::tc_fence_after();
                issue_s();
            }
        }
    } else if (warp < 6) {
        // ------------------------------------------------ transform warps
        const int tt = threadIdx.x - 64;
        const int atom = tt >> 6, cc = tt & 7, r0 = (tt >> 3) & 7;
        const int swz = (cc ^ r0) * 16;
        const size_t hb = static_cast<size_t>(bh) * T;
        const float rs = rsqrtf(static_cast<float>(dqk));
        const bool write_n = is_exp && xt == 0 && args.n_states != nullptr;
        const bool write_nf = is_exp && xt == 0 && args.n_final != nullptr;
        for (int p = tt; p < 128 * P; p += kTr) nsh[p] = 0.f;
        if (write_n)
            for (int p = tt; p < dqk; p += kTr) args.n_states[static_cast<size_t>(bh) * (NC + 1) * dqk + p] = 0.f;
        tc::named_bar_sync(2, kTr);
        uint32_t xpar = 0;  // per-slot phase parity of xfull
        float qacc[16];
        // row gates (w = b_bar / sqrt(d), a_bar) of chunk c live in fw[c & 1];
        // chunk c + 1's are fetched while chunk c is transformed
        // (loads go to registers one chunk ahead; the shared-memory stores happen
        // a chunk later, so the load latency never stalls a transform)
        float pf_w = 0.f, pf_a = 0.f;
        auto fetch_fac = [&](int c) {
            const size_t t = hb + static_cast<size_t>(c) * 128 + tt;
            pf_w = __ldg(args.gw.bb + t) * rs;
            pf_a = __ldg(args.gw.ab + t);
        };
        fetch_fac(0);
        float gb_next = __ldg(args.gw.gbar + static_cast<size_t>(bh) * NC), gb_cur = 0.f;
        for (int gi = 0; gi < n_stages; ++gi) {
            int kind, c, idx;
            stage_info(gi, kind, c, idx);
            if (kind == 0) continue;
            if (kind == 1 && idx == 0) {
                fw[((c & 1) * 2 + 0) * 128 + tt] = pf_w;
                fw[((c & 1) * 2 + 1) * 128 + tt] = pf_a;
                tc::named_bar_sync(2, kTr);  // fw[c & 1] complete; fw[(c + 1) & 1] no longer read
                if (c + 1 < NC) fetch_fac(c + 1);
            }
            if (kind == 2 && idx == 0) {
                gb_cur = gb_next;
                if (c + 1 < NC) gb_next = __ldg(args.gw.gbar + static_cast<size_t>(bh) * NC + c + 1);
            }
            const int s = gi % kR;
            tc::mbar_wait(&xfull[s], (xpar >> s) & 1);
            xpar ^= 1u << s;
            uint8_t* base = ring + s * kStage + atom * kAtom;
            const float* fac = fw + ((c & 1) * 2 + (kind == 1 ? 0 : 1)) * 128;
            if (kind == 1) {
                if (idx == 0)
#pragma unroll
                    for (int m = 0; m < 16; ++m) qacc[m] = 0.f;
                const float* nrow = nsh + idx * 128 + atom * 64 + cc * 8;
                float nv[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) nv[e] = nrow[e];
#pragma unroll 4
                for (int m = 0; m < 16; ++m) {
                    const int r = r0 + 8 * m;
                    uint4* ptr = reinterpret_cast<uint4*>(base + r * 128 + swz);
                    uint4 val = *ptr;
                    const float f = fac[r];
                    __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&val);
                    float d = 0.f;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 x = __bfloat1622float2(h2[e]);
                        d = fmaf(x.x, nv[2 * e], d);
                        d = fmaf(x.y, nv[2 * e + 1], d);
                        h2[e] = __floats2bfloat162_rn(x.x * f, x.y * f);
                    }
                    qacc[m] += d;
                    *ptr = val;
                }
                tc::fence_proxy_async_smem();
                tc::mbar_arrive(&tfull[s]);
                if (is_exp && idx == P - 1) {  // q . n_c for the rows of chunk c
#pragma unroll
                    for (int m = 0; m < 16; ++m) {
                        float v = qacc[m];
                        v += __shfl_xor_sync(0xffffffffu, v, 1);
                        v += __shfl_xor_sync(0xffffffffu, v, 2);
                        v += __shfl_xor_sync(0xffffffffu, v, 4);
                        qacc[m] = v;
                    }
                    const int b = c & 1;
                    if (c >= 2) tc::mbar_wait(&qnempty[b], ((c - 2) >> 1) & 1);
                    if (cc == 0)
#pragma unroll
                        for (int m = 0; m < 16; ++m) qnp[(b * 2 + atom) * 128 + r0 + 8 * m] = qacc[m];
                    tc::mbar_arrive(&qnfull[b]);
                }
            } else {
                float u[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) u[e] = 0.f;
#pragma unroll 4
                for (int m = 0; m < 16; ++m) {
                    const int r = r0 + 8 * m;
                    uint4* ptr = reinterpret_cast<uint4*>(base + r * 128 + swz);
                    uint4 val = *ptr;
                    const float f = fac[r];
                    __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&val);
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 x = __bfloat1622float2(h2[e]);
                        u[2 * e] = fmaf(f, x.x, u[2 * e]);
                        u[2 * e + 1] = fmaf(f, x.y, u[2 * e + 1]);
                        h2[e] = __floats2bfloat162_rn(x.x * f, x.y * f);
                    }
                    *ptr = val;
                }
                tc::fence_proxy_async_smem();
                tc::mbar_arrive(&tfull[s]);
                if (is_exp) {
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        u[e] += __shfl_xor_sync(0xffffffffu, u[e], 8);
                        u[e] += __shfl_xor_sync(0xffffffffu, u[e], 16);
                    }
                    if ((tc::lane_id() >> 3) == 0) {
                        float* dst = upart + ((tt >> 5) & 1) * 128 * P + idx * 128 + atom * 64 + cc * 8;
#pragma unroll
                        for (int e = 0; e < 8; ++e) dst[e] = u[e];
                    }
                    if (idx == P - 1) {  // n_{c+1} = gbar_c n_c + u_c
                        tc::named_bar_sync(2, kTr);
                        for (int p = tt; p < 128 * P; p += kTr) {
                            const float n = fmaf(gb_cur, nsh[p], upart[p] + upart[128 * P + p]);
                            nsh[p] = n;
                            if (write_n && p < dqk) args.n_states[(static_cast<size_t>(bh) * (NC + 1) + c + 1) * dqk + p] = n;
                            if (write_nf && c + 1 == NC && p < dqk) args.n_final[static_cast<size_t>(bh) * dqk + p] = n;
                        }
                        tc::named_bar_sync(2, kTr);
                    }
                }
            }
        }
    } else {
        // ------------------------------------------------ epilogue warps
        const int et = threadIdx.x - 192;
        const int lane = tc::lane_id();
        const int q4 = warp & 3;
        const int half = (warp - 6) >> 2;
        const int row = q4 * 32 + lane;
        const uint32_t trow = tc::tmem_row_addr(tmem);
        const size_t hb = static_cast<size_t>(bh) * T;
        const float rs = rsqrtf(static_cast<float>(dqk));
        const bool write_den = xt == 0 && args.h_denom != nullptr;
        // round-trip ownership: P = 2 -> state rows half*128 + row, all 128 columns;
        // P = 1 -> state row `row`, columns [half*64, +64)
        const int prow = P == 2 ? half * 128 + row : row;
        const int pcol0 = P == 2 ? 0 : half * 64;
        constexpr int kRtG = P == 2 ? 4 : 2;  // 32-column groups per thread
        const uint32_t taC = trow + colC + (P == 2 ? half * 128 : 0) + pcol0;

        auto store_cb = [&](int c) {  // TMA store of the bf16 C_c operand tile (saved state)
            if (et == 0) {
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
            for (int i = 0; i < 32; i += 4) *reinterpret_cast<float4*>(d + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
        };
        // Per-chunk gate values are fetched one chunk ahead into registers
        // (row t: b, m_c, w = b_bar / sqrt(d); column et: (ib - b) log2e; gbar).
        struct Gv {
            float b, mc, w, col, gb;
        };
        auto fetch = [&](int c) {
            Gv g;
            const size_t t = hb + static_cast<size_t>(c) * 128;
            g.b = args.gw.b[t + row];
            g.mc = args.gw.mc[t + row];
            g.w = args.gw.bb[t + row] * rs;
            g.col = et < 128 ? (args.gw.ib[t + et] - args.gw.b[t + et]) * kLog2e : 0.f;
            g.gb = c + 1 < NC ? __ldg(args.gw.gbar + static_cast<size_t>(bh) * NC + c + 1) : 0.f;
            return g;
        };
        // gating of S_c into packed bf16 Sbar (TMEM), returns this thread's row-sum part
        auto gating = [&](int c, const Gv& g) -> float {
            const float rowterm = (is_exp ? g.b - g.mc : g.b) * kLog2e;
            if (et < 128) colv[et] = g.col;
            tc::named_bar_sync(1, kEpi);
            tc::mbar_wait(sfull, c & 1);
            tc::tc_fence_after();
            float v[64];
            tc::tmem_ld32(trow + colS + half * 64, *reinterpret_cast<float(*)[32]>(v));
            tc::tmem_ld32(trow + colS + half * 64 + 32, *reinterpret_cast<float(*)[32]>(v + 32));
            tc::tmem_ld_wait();
            float rsum = 0.f;
            uint32_t pk[32];
#pragma unroll
            for (int e = 0; e < 64; e += 2) {
                const int j = half * 64 + e;
                const float w0 = j <= row ? v[e] * rs * exp2f(fminf(rowterm + colv[j], 0.f)) : 0.f;
                const float w1 = j + 1 <= row ? v[e + 1] * rs * exp2f(fminf(rowterm + colv[j + 1], 0.f)) : 0.f;
                rsum += w0 + w1;
                pk[e >> 1] = tc::pack_bf16(w0, w1);
            }
            tc::named_bar_sync(1, kEpi);  // every S column read before Sbar overwrites it
            tc::tmem_st32(trow + colS + half * 32, pk);
            tc::tmem_st_wait();
            tc::tc_fence_before();
            tc::mbar_arrive(bfull);
            return rsum;
        };

        // ---- prologue: C_0 = 0 (operand tile, saved state, optional fp32 states)
        Gv gcur = fetch(0);
        for (int i = et; i < P * 2 * kAtom / 16; i += kEpi)
            reinterpret_cast<uint4*>(cb)[i] = make_uint4(0, 0, 0, 0);
        if (args.c_states) {
            float z[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) z[i] = 0.f;
            if (prow < dqk)
                for (int g = 0; g < kRtG; ++g)
                    write_f32_state(args.c_states + static_cast<size_t>(bh) * (NC + 1) * dqk * dhv, z, g);
        }
        tc::fence_proxy_async_smem();
        tc::mbar_arrive(cready);
        tc::named_bar_sync(1, kEpi);
        store_cb(0);
        float rsum = gating(0, gcur);
        Gv gnext = NC > 1 ? fetch(1) : gcur;

        for (int k = 0; k < NC; ++k) {
            const int t = k * 128 + row;
            // ---- a. drain H_k; h is staged in the Cb tile (free between QC_k and the
            //         next round trip) and written with one TMA store
            tc::mbar_wait(hfull, k & 1);
            tc::tc_fence_after();
            float hv[64];
            tc::tmem_ld32(trow + colH + half * 64, *reinterpret_cast<float(*)[32]>(hv));
            tc::tmem_ld32(trow + colH + half * 64 + 32, *reinterpret_cast<float(*)[32]>(hv + 32));
            tc::tmem_ld_wait();
            tc::tc_fence_before();
            tc::mbar_arrive(hempty);
            const int b = k & 1;
            if (is_exp) {
                if (half == 1) xred[row] = rsum;
                tc::mbar_wait(&qnfull[b], (k >> 1) & 1);
            }
            if (et == 0) tc::tma_store_wait_read<0>();  // the saved-state store of Cb_k
            tc::named_bar_sync(1, kEpi);
            float den = 1.f;
            if (is_exp) {
                if (half == 0) {
                    const float qn = qnp[(b * 2) * 128 + row] + qnp[(b * 2 + 1) * 128 + row];
                    den = fmaxf(fabsf(rsum + xred[row] + gcur.w * qn), exp2f(-gcur.mc * kLog2e));
                    denb[row] = den;
                    if (write_den) args.h_denom[hb + t] = den;
                }
                tc::named_bar_sync(1, kEpi);
                if (et == 0) tc::mbar_arrive(&qnempty[b]);
                if (half == 1) den = denb[row];
            } else if (write_den && half == 0) {
                args.h_denom[hb + t] = 1.f;
            }
            {
                const float inv = 1.f / den;
#pragma unroll
                for (int e = 0; e < 64; ++e) hv[e] *= inv;
#pragma unroll
                for (int q = 0; q < 8; ++q) tc::sw128_store8(cb, row, half * 8 + q, 128, hv + 8 * q);
                tc::fence_proxy_async_smem();
                tc::named_bar_sync(1, kEpi);
                if (et == 0) {
                    for (int a = 0; a < 2; ++a) tc::tma_store_3d(&mapH, cb + a * kAtom, x0 + 64 * a, k * 128, bh);
                    tc::tma_store_commit();
                }
            }

            // ---- b. C round trip: C_{k+1} -> Cb (bf16 operand + saved state), TMEM C *= gbar_{k+1}
            tc::mbar_wait(cfull, k & 1);
            tc::tc_fence_after();
            const bool last = k + 1 == NC;
            if (!last) {
                if (et == 0) tc::tma_store_wait_read<0>();  // the h store out of Cb
                tc::named_bar_sync(1, kEpi);
            }
            const float gb = gcur.gb;
            float* cs = args.c_states ? args.c_states + (static_cast<size_t>(bh) * (NC + 1) + k + 1) * dqk * dhv : nullptr;
            float* cf = last && args.c_final ? args.c_final + static_cast<size_t>(bh) * dqk * dhv : nullptr;
#pragma unroll 1
            for (int g = 0; g < kRtG; ++g) {
                float v[32];
                tc::tmem_ld32(taC + g * 32, v);
                tc::tmem_ld_wait();
                if (prow < dqk) {
                    if (cs) write_f32_state(cs, v, g);
                    if (cf) write_f32_state(cf, v, g);
                }
                if (!last) {
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        tc::sw128_store8(cb, prow, (pcol0 + g * 32) / 8 + q, 128 * P, v + 8 * q);
                    uint32_t sc[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i) sc[i] = __float_as_uint(v[i] * gb);
                    tc::tmem_st32(taC + g * 32, sc);
                }
            }
            if (!last) {
                tc::tmem_st_wait();
                tc::fence_proxy_async_smem();
                tc::tc_fence_before();
                tc::mbar_arrive(cready);
                tc::named_bar_sync(1, kEpi);
                store_cb(k + 1);
                // ---- c. gating of S_{k+1}
                gcur = gnext;
                rsum = gating(k + 1, gcur);
                if (k + 2 < NC) gnext = fetch(k + 2);
            }
        }
        if (et == 0) tc::tma_store_wait_all<0>();
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

template <int P>
int launch_impl(const FusedFwdArgs& a, const void* q, const void* k, const void* v, void* saved,
                cudaStream_t st) {
    using namespace tfla_host;
    const Geom& g = a.g;
    CUtensorMap mq, mk, mv, ms, mh;
    if (!make_tmap_bf16_3d(&mh, a.h, g.BH, g.T, g.dhv, 64, 128) ||
        !make_tmap_bf16_3d(&mq, q, g.BH, g.T, g.dqk, 64, 128) ||
        !make_tmap_bf16_3d(&mk, k, g.BH, g.T, g.dqk, 64, 128) ||
        !make_tmap_bf16_3d(&mv, v, g.BH, g.T, g.dhv, 64, 128) ||
        !make_tmap_bf16_3d(&ms, saved, static_cast<uint64_t>(g.BH) * g.NC, g.dqk, g.dhv, 64, 128))
        return 4;
    constexpr int smem = FSmem<P>::kBytes;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(fwd_fused_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    fwd_fused_kernel<P><<<g.BH * (g.dhv / 128), kThreads, smem, st>>>(mq, mk, mv, ms, mh, a);
    return 0;
}

}  // namespace

bool fwd_fused_supported(const Geom& g) {
    return g.L == 128 && (g.dqk == 128 || g.dqk == 256) && g.dhv % 128 == 0;
}

int launch_fwd_fused(const FusedFwdArgs& a, const void* q, const void* k, const void* v, void* saved,
                     cudaStream_t st) {
    return a.g.dqk == 256 ? launch_impl<2>(a, q, k, v, saved, st) : launch_impl<1>(a, q, k, v, saved, st);
}

}  // namespace tfla_k
