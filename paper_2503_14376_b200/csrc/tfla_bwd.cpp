// tfla_bwd.cpp -- backward driver behind tfla_chunkwise_backward / tfla_backward.
// Sequence (one stream): K0b gates from the saved stabilisers -> [fp32 -> bf16
// state conversion when only reference-layout states were given] -> K3 reverse
// dC sweep (tcgen05, + d_g partials) -> K4 dQ / dK / dV (tcgen05) -> K7 gate
// assembly. Mirrors chunkwise_backward (chunkwise.cpp:396-566) and
// tfla_backward (tiled.cpp:781-811).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "bwd_parallel.h"
#include "capi_internal.h"
#include "host_util.h"
#include "kernels.h"
#include "workspace.h"

using tfla_host::set_error;

namespace {

int check_cuda(const char* where) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string(where) + ": " + cudaGetErrorString(e));
        return TFLA_ERR_CUDA;
    }
    return TFLA_OK;
}

int backward_impl(const tfla_dims* dims, const tfla_blocks* blocks, int variant,
                  const tfla_inputs* in, const tfla_bwd_in* sv, const tfla_grads* gr, void* ws,
                  size_t ws_bytes, void* stream) {
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
    if (!gr || !gr->dq || !gr->dk || !gr->dv || !gr->d_fpre || !gr->d_ipre)
        return set_error("backward: missing gradient output"), TFLA_ERR_PARAMETER;
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
    if (!saved) {
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
    sa.ntile = (nenv && atoi(nenv) == 128 && g.dhv % 128 == 0) ? 128 : plan.scan_ntile;
    const int scan_tiles = plan.n_ptile * (g.dhv / sa.ntile);
    sa.w = gw.bb;
    sa.gbar = gw.gbar;
    sa.c_saved = static_cast<const __nv_bfloat16*>(saved);
    sa.dg_part = dg_part;
    {
        tfla_host::ProfScope ps(tfla_host::P_SCAN_BWD, st, 1);
        if (tfla_k::launch_state_scan(true, in->q, sv->d_h, dstates, sa, st)) return TFLA_ERR_CUDA;
    }
    if ((rc = check_cuda("state_scan_bwd"))) return rc;

    // K4: dQ, dK, dV
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
    tfla_k::BwdTensors bt{in->q, in->k, in->v, sv->d_h, saved, gr->dq};
    const bool fused = tfla_k::bwd_fused_supported(g) && !tfla_host::env_flag("TFLA_NO_FUSED_BWD");
    if (fused) {
        // debug: TFLA_TRACE_BWD=<file> dumps per-stage clock64 events of CTA 0
        const char* trace_file = getenv("TFLA_TRACE_BWD");
        if (trace_file && *trace_file) {
            cudaMalloc(&ba.trace, 2048 * sizeof(long long));
            cudaMemsetAsync(ba.trace, 0, 2048 * sizeof(long long), st);
        }
        {
            tfla_host::ProfScope ps(tfla_host::P_BWD_FUSED, st, 1);
            if (tfla_k::launch_bwd_fused(ba, bt, gr->dq, gr->dk, gr->dv, saved, dstates, st)) return TFLA_ERR_CUDA;
        }
        if (ba.trace) {
            std::vector<long long> hbuf(2048);
            cudaMemcpyAsync(hbuf.data(), ba.trace, 2048 * sizeof(long long), cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            cudaFree(ba.trace);
            if (FILE* f = fopen(trace_file, "w")) {
                for (int i = 0; i < 512; ++i)
                    fprintf(f, "%lld %lld %lld %lld\n", hbuf[i * 4], hbuf[i * 4 + 1], hbuf[i * 4 + 2], hbuf[i * 4 + 3]);
                fclose(f);
            }
        }
        if ((rc = check_cuda("bwd_fused"))) return rc;
    } else {
        {
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
    }

    // K7: gate gradients
    tfla_k::AssembleArgs aa{};
    aa.g = g;
    aa.variant = variant;
    aa.n_ptile = fused ? 1 : plan.n_ptile;
    aa.n_tiles = scan_tiles;
    aa.f_pre = in->f_pre;
    aa.i_pre = in->i_pre;
    aa.gbar = gw.gbar;
    aa.dg_part = dg_part;
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

}  // extern "C"
