// tfla_bwd.cpp -- backward driver behind tfla_chunkwise_backward / tfla_backward.
// Sequence (one stream): K0b gates from the saved stabilisers -> [fp32 -> bf16
// state conversion when only reference-layout states were given] -> K3 reverse
// dC sweep (tcgen05, + d_g partials) -> K4 dQ / dK / dV (tcgen05) -> K7 gate
// assembly. Mirrors chunkwise_backward (chunkwise.cpp:396-566) and
// tfla_backward (tiled.cpp:781-811).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "bwd_parallel.h"
#include "capi_internal.h"
#include "host_util.h"
#include "kernels.h"
#include "workspace.h"

using tfla_host::set_error;

namespace {

// Library-owned side stream (per device) for the split backward's dQ, which
// reads C_k but not dC: it runs beside the reverse state sweep K3 (fork / join
// by events on the caller's stream, so the pattern is CUDA-graph capturable).
struct SideStream {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
SideStream* side_stream() {
    static std::mutex mu;
    static std::vector<SideStream*> per_dev;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    if (static_cast<int>(per_dev.size()) <= dev) per_dev.resize(dev + 1, nullptr);
    if (!per_dev[dev]) {
        auto* ss = new SideStream();
        cudaStreamCreateWithFlags(&ss->s, cudaStreamNonBlocking);
        cudaEventCreateWithFlags(&ss->fork, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&ss->join, cudaEventDisableTiming);
        per_dev[dev] = ss;
    }
    return per_dev[dev];
}

int check_cuda(const char* where) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string(where) + ": " + cudaGetErrorString(e));
        return TFLA_ERR_CUDA;
    }
    return TFLA_OK;
}

// What one call produces: the full gradients (tfla_backward) or one split entry
// point (tiled.hpp:56-84, chunkwise.hpp:73-76).
enum class Part { kFull, kDQ, kDK, kDV, kStatePass };

struct SplitOut {
    void* grad = nullptr;                                   // dq / dk / dv
    float *out0 = nullptr, *out1 = nullptr, *out2 = nullptr;  // gate partials
    float *d_c = nullptr, *d_g = nullptr;                   // state pass
};

int backward_impl(const tfla_dims* dims, const tfla_blocks* blocks, int variant,
                  const tfla_inputs* in, const tfla_bwd_in* sv, const tfla_grads* gr, void* ws,
                  size_t ws_bytes, void* stream, Part part = Part::kFull, const SplitOut& so = {}) {
    set_error("");
    int rc = tfla_host::validate_dims(dims);
    if (rc) return rc;
    if (blocks && (rc = tfla_host::validate_blocks(dims, blocks))) return rc;
    if (variant != TFLA_VARIANT_EXP && variant != TFLA_VARIANT_SIG)
        return set_error("unknown variant"), TFLA_ERR_PARAMETER;
    if (!in || !in->q || !in->k || !in->v || !in->i_pre || !in->f_pre)
        return set_error("backward: missing input tensor"), TFLA_ERR_PARAMETER;
    // chunkwise.cpp:401-403 / tiled.cpp:384-386
    if (!sv || !sv->d_h || !sv->m_states || !sv->m_combine || !sv->h_denom ||
        (!sv->saved_states && !sv->c_states))
        return set_error("chunkwise_backward: missing saved forward tensors"), TFLA_ERR_PARAMETER;
    switch (part) {
        case Part::kFull:
            if (!gr || !gr->dq || !gr->dk || !gr->dv || !gr->d_fpre || !gr->d_ipre)
                return set_error("backward: missing gradient output"), TFLA_ERR_PARAMETER;
            break;
        case Part::kDQ:
            if (!so.grad || !so.out0) return set_error("tfla_backward_dq: missing output"), TFLA_ERR_PARAMETER;
            break;
        case Part::kDK:
            if (!so.grad || !so.out0 || !so.out1 || !so.out2)
                return set_error("tfla_backward_dk: missing output"), TFLA_ERR_PARAMETER;
            break;
        case Part::kDV:
            if (!so.grad) return set_error("tfla_backward_dv: missing output"), TFLA_ERR_PARAMETER;
            break;
        case Part::kStatePass:
            if (!so.d_g) return set_error("backward_state_pass: missing d_g output"), TFLA_ERR_PARAMETER;
            break;
    }
    // TMA-read / -written tensors and the float4-accessed states
    if ((rc = tfla_host::check_aligned({in->q, in->k, in->v, sv->d_h, sv->saved_states, sv->c_states, ws, so.grad,
                                        so.d_c, gr ? gr->dq : nullptr, gr ? gr->dk : nullptr,
                                        gr ? gr->dv : nullptr},
                                       "backward")))
        return rc;
    const int ntile = tfla_host::pick_ntile(*dims, blocks);
    const tfla_host::WsPlan plan = tfla_host::plan_workspace(*dims, 1, ntile);
    if (!ws || ws_bytes < plan.total)
        return set_error("backward: workspace too small (need " + std::to_string(plan.total) +
                         " bytes)"),
               TFLA_ERR_PARAMETER;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const tfla_k::Geom g = tfla_host::geom_of(*dims);
    const tfla_k::GateWS gw = tfla_host::gate_ws(plan, ws);
    uint8_t* w8 = static_cast<uint8_t*>(ws);
    float* dg_part = reinterpret_cast<float*>(w8 + plan.dg_part);
    float* dbq = reinterpret_cast<float*>(w8 + plan.dbq);
    float* da = reinterpret_cast<float*>(w8 + plan.da);
    float* colsum = reinterpret_cast<float*>(w8 + plan.colsum);
    void* dstates = w8 + plan.dstates;

    // K0b: gates from the saved stabilisers
    {
        tfla_host::ProfScope ps(tfla_host::P_GATES_BWD, st, 1);
        tfla_k::launch_gates_bwd(g, variant, in->f_pre, in->i_pre, sv->m_states, sv->m_combine,
                                 sv->h_denom, gw, st);
    }
    if ((rc = check_cuda("gates_bwd"))) return rc;

    const void* saved = sv->saved_states;
    if (!saved && part != Part::kDV) {  // dV never reads C_k
        tfla_host::ProfScope ps(tfla_host::P_STATES_BF16, st, 1);
        tfla_k::launch_states_to_bf16(sv->c_states, reinterpret_cast<__nv_bfloat16*>(w8 + plan.saved),
                                      g, st);
        saved = w8 + plan.saved;
        if ((rc = check_cuda("states_to_bf16"))) return rc;
    }

    // K3: dC_k = gbar dC_{k+1} + (w o Q)^T dH  (+ d_g partials against C_k)
    tfla_k::ScanArgs sa{};
    sa.g = g;
    // K3 column tile: 64 (two CTAs per SM) or 128 (half the L2 re-reads of Q)
    const char* nenv = getenv("TFLA_SCAN_BWD_N");
    sa.ntile = (nenv && atoi(nenv) == 128 && g.dhv % 128 == 0) ? 128 : tfla_k::scan_ntile_for(g);
    const bool scan2 = tfla_k::scan2_use(g, true);
    const int scan_tiles = scan2 ? (g.dqk / 128) * (g.dhv / 256) : plan.n_ptile * (g.dhv / sa.ntile);
    sa.w = gw.bb;
    sa.gbar = gw.gbar;
    sa.c_saved = static_cast<const __nv_bfloat16*>(saved);
    sa.dg_part = dg_part;
    sa.dc_states = so.d_c;
    // Opt-in (TFLA_DG_IDENTITY=1): the fused backward derives d_g from its
    // per-token partials (bwd_parallel.h, launch_dg_from_partials) and the scan
    // skips the C_k reads (a third of its HBM traffic, -0.17 ms at the 7B
    // shape). The identity telescopes differences of O(<U, W>) terms whose bf16
    // rounding does not cancel when gbar is small: d_fpre max_rel rises from
    // 1e-3..5e-3 to 5e-3..2e-2 at the 7B head shape, so the direct
    // <C_k, dC_{k+1}> stays the default.
    const bool fused = part == Part::kFull && tfla_k::bwd_fused_supported(g) &&
                       !tfla_host::env_flag("TFLA_NO_FUSED_BWD");
    const bool dg_identity = fused && tfla_host::env_flag("TFLA_DG_IDENTITY");
    if (dg_identity) sa.dg_part = nullptr;
    // full split path: dQ (C_k, no dC) forks onto the side stream before K3
    // opt-in (TFLA_BWD_OVERLAP=1): measured neutral at L = 256 / 512 -- the
    // persistent dQ grid and K3's CTAs cannot share SMs (shared memory)
    const bool overlap_dq = part == Part::kFull && !fused && tfla_host::env_flag("TFLA_BWD_OVERLAP");
    SideStream* side = overlap_dq ? side_stream() : nullptr;
    tfla_k::BwdArgs ba{};
    ba.g = g;
    ba.ntile = ntile;
    ba.variant = variant;
    ba.gw = gw;
    ba.q = static_cast<const __nv_bfloat16*>(in->q);
    ba.k = static_cast<const __nv_bfloat16*>(in->k);
    ba.dbq_part = dbq;
    ba.da_part = da;
    ba.colsum = colsum;
    if (overlap_dq) {
        tfla_k::BwdTensors bq{in->q, in->k, in->v, sv->d_h, saved, gr->dq};
        cudaEventRecord(side->fork, st);
        cudaStreamWaitEvent(side->s, side->fork, 0);
        {
            tfla_host::ProfScope ps(tfla_host::P_BWD_DQ, side->s, 1);
            if (tfla_k::launch_bwd_parallel(tfla_k::kDQ, ba, bq, side->s)) return TFLA_ERR_CUDA;
        }
        cudaEventRecord(side->join, side->s);
        if ((rc = check_cuda("bwd_dq"))) return rc;
    }
    if (part != Part::kDQ) {  // dQ reads C_k, not dC
        if (part == Part::kDV && !saved) {
            // the d_g partials read C_k; dV alone has no use for them
            saved = w8 + plan.saved;
            cudaMemsetAsync(w8 + plan.saved, 0, static_cast<size_t>(g.BH) * g.NC * g.dqk * g.dhv * 2, st);
            sa.c_saved = static_cast<const __nv_bfloat16*>(saved);
        }
        tfla_host::ProfScope ps(tfla_host::P_SCAN_BWD, st, 1);
        if (scan2 ? tfla_k::launch_state_scan2(true, in->q, sv->d_h, dstates, sa, st)
                  : tfla_k::launch_state_scan(true, in->q, sv->d_h, dstates, sa, st))
            return TFLA_ERR_CUDA;
    }
    if ((rc = check_cuda("state_scan_bwd"))) return rc;
    if (part == Part::kStatePass) {
        tfla_k::launch_dg_reduce(g, scan_tiles, dg_part, gw.gbar, so.d_g, st);
        return check_cuda("dg_reduce");
    }

    // K4: dQ, dK, dV
    if (part != Part::kFull) {  // one gradient kernel of the split path (tiled.cpp:391-779)
        const tfla_k::BwdKind kind =
            part == Part::kDQ ? tfla_k::kDQ : part == Part::kDK ? tfla_k::kDK : tfla_k::kDV;
        tfla_k::BwdTensors bt{in->q, in->k, in->v, sv->d_h, kind == tfla_k::kDQ ? saved : dstates, so.grad};
        {
            tfla_host::ProfScope ps(kind == tfla_k::kDQ   ? tfla_host::P_BWD_DQ
                                    : kind == tfla_k::kDK ? tfla_host::P_BWD_DK
                                                          : tfla_host::P_BWD_DV,
                                    st, 1);
            if (tfla_k::launch_bwd_parallel(kind, ba, bt, st)) return TFLA_ERR_CUDA;
        }
        if ((rc = check_cuda("bwd_split"))) return rc;
        if (kind != tfla_k::kDV)
            tfla_k::launch_split_partials(kind, g, tfla_k::bwd_n_ptile(g), dbq, da, colsum, so.out0, so.out1,
                                          so.out2, st);
        return check_cuda("split_partials");
    }
    tfla_k::BwdTensors bt{in->q, in->k, in->v, sv->d_h, saved, gr->dq};
    float* dg = reinterpret_cast<float*>(w8 + plan.dg);
    if (dg_identity) ba.iq_part = reinterpret_cast<float*>(w8 + plan.iq);
    if (fused) {
        // debug: TFLA_TRACE_BWD=<file> dumps per-stage clock64 events of CTA 0
        const char* trace_file = getenv("TFLA_TRACE_BWD");
        if (trace_file && *trace_file) {
            cudaMalloc(&ba.trace, 4096 * sizeof(long long));
            cudaMemsetAsync(ba.trace, 0, 4096 * sizeof(long long), st);
        }
        {
            tfla_host::ProfScope ps(tfla_host::P_BWD_FUSED, st, 1);
            const bool wide = tfla_k::bwd_fused_wide_supported(g) && !ba.trace;
            if (wide ? tfla_k::launch_bwd_fused_wide(ba, bt, gr->dq, gr->dk, gr->dv, saved, dstates, st)
                     : tfla_k::launch_bwd_fused(ba, bt, gr->dq, gr->dk, gr->dv, saved, dstates, st))
                return TFLA_ERR_CUDA;
        }
        if (ba.trace) {
            std::vector<long long> hbuf(4096);
            cudaMemcpyAsync(hbuf.data(), ba.trace, 4096 * sizeof(long long), cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            cudaFree(ba.trace);
            if (FILE* f = fopen(trace_file, "w")) {  // 512 stage rows, then 64 epilogue rows of 32
                for (int i = 0; i < 512; ++i)
                    fprintf(f, "%lld %lld %lld %lld\n", hbuf[i * 4], hbuf[i * 4 + 1], hbuf[i * 4 + 2], hbuf[i * 4 + 3]);
                for (int i = 0; i < 64; ++i)
                    for (int e = 0; e < 32; ++e) fprintf(f, "%lld%c", hbuf[2048 + 32 * i + e], e == 31 ? '\n' : ' ');
                fclose(f);
            }
        }
        if ((rc = check_cuda("bwd_fused"))) return rc;
        if (dg_identity) {
            tfla_host::ProfScope ps(tfla_host::P_ASSEMBLE, st, 1);
            tfla_k::launch_dg_from_partials(g, ba.iq_part, da, dg, st);
        }
    } else {
        if (!overlap_dq) {
            tfla_host::ProfScope ps(tfla_host::P_BWD_DQ, st, 1);
            if (tfla_k::launch_bwd_parallel(tfla_k::kDQ, ba, bt, st)) return TFLA_ERR_CUDA;
        }
        if ((rc = check_cuda("bwd_dq"))) return rc;
        bt.states = dstates;
        bt.out = gr->dk;
        {
            tfla_host::ProfScope ps(tfla_host::P_BWD_DK, st, 1);
            if (tfla_k::launch_bwd_parallel(tfla_k::kDK, ba, bt, st)) return TFLA_ERR_CUDA;
        }
        if ((rc = check_cuda("bwd_dk"))) return rc;
        bt.out = gr->dv;
        {
            tfla_host::ProfScope ps(tfla_host::P_BWD_DV, st, 1);
            if (tfla_k::launch_bwd_parallel(tfla_k::kDV, ba, bt, st)) return TFLA_ERR_CUDA;
        }
        if ((rc = check_cuda("bwd_dv"))) return rc;
        if (overlap_dq) cudaStreamWaitEvent(st, side->join, 0);  // join before the assembly reads dbq
    }

    // K7: gate gradients
    tfla_k::AssembleArgs aa{};
    aa.g = g;
    aa.variant = variant;
    aa.n_ptile = fused ? 1 : tfla_k::bwd_n_ptile(g);
    aa.f_pre = in->f_pre;
    aa.i_pre = in->i_pre;
    aa.gbar = dg_identity ? nullptr : gw.gbar;  // the identity's d_g carries gbar already
    aa.dg_part = dg_identity ? dg : dg_part;
    aa.n_tiles = dg_identity ? 1 : scan_tiles;
    aa.dbq_part = dbq;
    aa.da_part = da;
    aa.colsum = colsum;
    aa.d_fpre = gr->d_fpre;
    aa.d_ipre = gr->d_ipre;
    {
        tfla_host::ProfScope ps(tfla_host::P_ASSEMBLE, st, 1);
        tfla_k::launch_assemble(aa, st);
    }
    return check_cuda("assemble");
}

}  // namespace

extern "C" {

int tfla_chunkwise_backward(const tfla_dims* dims, int variant, const tfla_inputs* in,
                            const tfla_bwd_in* saved, const tfla_grads* grads, void* workspace,
                            size_t workspace_bytes, void* stream) {
    return backward_impl(dims, nullptr, variant, in, saved, grads, workspace, workspace_bytes,
                         stream);
}

int tfla_backward(const tfla_dims* dims, const tfla_blocks* blocks, int variant,
                  const tfla_inputs* in, const tfla_bwd_in* saved, const tfla_grads* grads,
                  void* workspace, size_t workspace_bytes, void* stream) {
    if (!blocks) {
        set_error("tfla_backward: blocks is NULL");
        return TFLA_ERR_PARAMETER;
    }
    return backward_impl(dims, blocks, variant, in, saved, grads, workspace, workspace_bytes,
                         stream);
}

int tfla_backward_dq(const tfla_dims* dims, const tfla_blocks* blocks, int variant,
                     const tfla_inputs* in, const tfla_bwd_in* saved, void* dq, float* d_b_cum,
                     void* workspace, size_t workspace_bytes, void* stream) {
    if (!blocks) return set_error("tfla_backward_dq: blocks is NULL"), TFLA_ERR_PARAMETER;
    SplitOut so;
    so.grad = dq;
    so.out0 = d_b_cum;
    return backward_impl(dims, blocks, variant, in, saved, nullptr, workspace, workspace_bytes, stream,
                         Part::kDQ, so);
}

int tfla_backward_dk(const tfla_dims* dims, const tfla_blocks* blocks, int variant,
                     const tfla_inputs* in, const tfla_bwd_in* saved, void* dk, float* d_a_tail,
                     float* d_b_cum, float* d_i_log, void* workspace, size_t workspace_bytes,
                     void* stream) {
    if (!blocks) return set_error("tfla_backward_dk: blocks is NULL"), TFLA_ERR_PARAMETER;
    SplitOut so;
    so.grad = dk;
    so.out0 = d_a_tail;
    so.out1 = d_b_cum;
    so.out2 = d_i_log;
    return backward_impl(dims, blocks, variant, in, saved, nullptr, workspace, workspace_bytes, stream,
                         Part::kDK, so);
}

int tfla_backward_dv(const tfla_dims* dims, const tfla_blocks* blocks, int variant,
                     const tfla_inputs* in, const tfla_bwd_in* saved, void* dv, void* workspace,
                     size_t workspace_bytes, void* stream) {
    if (!blocks) return set_error("tfla_backward_dv: blocks is NULL"), TFLA_ERR_PARAMETER;
    SplitOut so;
    so.grad = dv;
    return backward_impl(dims, blocks, variant, in, saved, nullptr, workspace, workspace_bytes, stream,
                         Part::kDV, so);
}

int tfla_backward_state_pass(const tfla_dims* dims, int variant, const tfla_inputs* in,
                             const tfla_bwd_in* saved, float* d_c, float* d_g, void* workspace,
                             size_t workspace_bytes, void* stream) {
    SplitOut so;
    so.d_c = d_c;
    so.d_g = d_g;
    return backward_impl(dims, nullptr, variant, in, saved, nullptr, workspace, workspace_bytes, stream,
                         Part::kStatePass, so);
}

int tfla_assemble_gate_grads(const tfla_dims* dims, int variant, const float* f_pre, const float* i_pre,
                             const float* d_g, const float* d_b_total, const float* d_a,
                             const float* d_i_extra, float* d_fpre, float* d_ipre, void* stream) {
    set_error("");
    int rc = tfla_host::validate_dims(dims);
    if (rc) return rc;
    if (variant != TFLA_VARIANT_EXP && variant != TFLA_VARIANT_SIG)
        return set_error("unknown variant"), TFLA_ERR_PARAMETER;
    if (!f_pre || !i_pre || !d_g || !d_b_total || !d_a || !d_i_extra || !d_fpre || !d_ipre)
        return set_error("assemble_gate_grads: missing tensor"), TFLA_ERR_PARAMETER;

    tfla_k::AssembleArgs aa{};
    aa.g = tfla_host::geom_of(*dims);
    aa.variant = variant;
    aa.n_ptile = 1;
    aa.n_tiles = 1;
    aa.f_pre = f_pre;
    aa.i_pre = i_pre;
    aa.gbar = nullptr;  // d_g already carries gbar (chunkwise.cpp:221)
    aa.dg_part = d_g;
    aa.dbq_part = d_b_total;
    aa.da_part = d_a;
    aa.colsum = nullptr;
    aa.di_extra = d_i_extra;
    aa.d_fpre = d_fpre;
    aa.d_ipre = d_ipre;
    {
        tfla_host::ProfScope ps(tfla_host::P_ASSEMBLE, static_cast<cudaStream_t>(stream), 1);
        tfla_k::launch_assemble(aa, static_cast<cudaStream_t>(stream));
    }
    return check_cuda("assemble_gate_grads");
}

}  // extern "C"
