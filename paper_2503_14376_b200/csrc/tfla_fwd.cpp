// tfla_fwd.cpp -- forward driver behind tfla_chunkwise_forward / tfla_forward.
// Sequence (per call, one stream): K0 gates + max-state scan -> K1 recurrent
// state scan (tcgen05) -> K2 TFLA parallel forward (tcgen05). Mirrors
// chunkwise_forward (chunkwise.cpp:270-302) and tfla_forward (tiled.cpp:258-298).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "capi_internal.h"
#include "fwd_fused.h"
#include "bwd_parallel.h"
#include "fwd_parallel.h"
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

// Output epilogue requested with the forward (tfla_chunkwise_forward_gated).
struct OutGate {
    const void* o_pre;
    const float* gamma;
    float eps;
    void* y;
};

// y = sigmoid(o_pre) * rms_norm(h_tilde; gamma, eps) as a separate HBM pass
// (the paths the fused epilogue does not cover).
int output_pass(const tfla_dims* dims, const tfla_fwd_out* out, const OutGate* og, cudaStream_t st) {
    tfla_k::launch_output_norm_gate(static_cast<const __nv_bfloat16*>(out->h),
                                    static_cast<const __nv_bfloat16*>(og->o_pre), og->gamma, og->eps,
                                    static_cast<__nv_bfloat16*>(og->y), dims->n_batch * dims->n_head * dims->T,
                                    static_cast<int>(dims->T), static_cast<int>(dims->n_head),
                                    static_cast<int>(dims->d_hv), st);
    return check_cuda("output");
}

int forward_impl(const tfla_dims* dims, const tfla_blocks* blocks, int variant,
                 const tfla_inputs* in, const tfla_fwd_out* out, void* ws, size_t ws_bytes,
                 void* stream, const tfla_state_in* init = nullptr, bool states_only = false,
                 const OutGate* og = nullptr) {
    set_error("");
    int rc = tfla_host::validate_dims(dims);
    if (rc) return rc;
    if (blocks && (rc = tfla_host::validate_blocks(dims, blocks))) return rc;
    if (variant != TFLA_VARIANT_EXP && variant != TFLA_VARIANT_SIG)
        return set_error("unknown variant"), TFLA_ERR_PARAMETER;
    if (!in || !in->q || !in->k || !in->v || !in->i_pre || !in->f_pre)
        return set_error("forward: missing input tensor"), TFLA_ERR_PARAMETER;
    if (states_only) {  // state_recurrence_head outputs (detail_kernels.hpp:38-44)
        if (!out || !out->m_states || (!out->c_states && !out->saved_states))
            return set_error("state_recurrence: m_states and c_states or saved_states are required"),
                   TFLA_ERR_PARAMETER;
    } else if (!out || !out->h || !out->m_states || !out->m_combine || !out->h_denom) {
        return set_error("forward: h, m_states, m_combine and h_denom are required"),
               TFLA_ERR_PARAMETER;
    }
    if (init && (!init->c || (variant == TFLA_VARIANT_EXP && (!init->n || !init->m))))
        return set_error("forward: initial state needs c (and n, m for mLSTMexp)"), TFLA_ERR_PARAMETER;
    // TMA-read / -written tensors and the float4-accessed states
    if ((rc = tfla_host::check_aligned({in->q, in->k, in->v, out->h, out->c_states, out->c_final,
                                        out->saved_states, ws, init ? init->c : nullptr},
                                       "forward")))
        return rc;
    if (og) {  // output epilogue: the checks of tfla_output_norm_gate
        if (!tfla_k::output_supported(static_cast<int>(dims->d_hv)))
            return set_error("output: B200 kernel needs d_hv a multiple of 8, <= 2048"), TFLA_ERR_GEOMETRY;
        if (!(og->eps >= 0.f)) return set_error("rms_norm: eps must be >= 0"), TFLA_ERR_PARAMETER;  // transfer.cpp:9
        if (!og->o_pre || !og->gamma || !og->y) return set_error("output: missing tensor"), TFLA_ERR_PARAMETER;
        if ((rc = tfla_host::check_aligned({og->o_pre, og->gamma, og->y}, "output"))) return rc;
    }
    const float* c_init = init ? init->c : nullptr;
    const float* n_init = init && variant == TFLA_VARIANT_EXP ? init->n : nullptr;
    const float* m_init = init && variant == TFLA_VARIANT_EXP ? init->m : nullptr;
    const int ntile = tfla_host::pick_ntile(*dims, blocks);
    const tfla_host::WsPlan plan = tfla_host::plan_workspace(*dims, 0, ntile);
    if (!ws || ws_bytes < plan.total)
        return set_error("forward: workspace too small (need " + std::to_string(plan.total) +
                         " bytes)"),
               TFLA_ERR_PARAMETER;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const tfla_k::Geom g = tfla_host::geom_of(*dims);
    const tfla_k::GateWS gw = tfla_host::gate_ws(plan, ws);
    uint8_t* w8 = static_cast<uint8_t*>(ws);
    const bool is_exp = variant == TFLA_VARIANT_EXP;
    float* n_states = out->n_states ? out->n_states : reinterpret_cast<float*>(w8 + plan.n_states);
    void* saved = out->saved_states ? out->saved_states : static_cast<void*>(w8 + plan.saved);
    const size_t BH = g.BH;

    // K0: gates + max-state scan (writes m_states, m_combine, m_final)
    {
    tfla_host::ProfScope ps(tfla_host::P_GATES_FWD, st, 2);
    tfla_k::launch_gates_fwd(g, variant, in->f_pre, in->i_pre, gw, out->m_states, out->m_combine,
                             out->m_final, st, m_init);
    }
    if ((rc = check_cuda("gates"))) return rc;

    // sigmoid variant carries no normaliser state (chunkwise.hpp:8-10)
    if (!is_exp) {
        if (out->n_states)
            cudaMemsetAsync(out->n_states, 0, BH * (g.NC + 1) * g.dqk * sizeof(float), st);
        if (out->n_final) cudaMemsetAsync(out->n_final, 0, BH * g.dqk * sizeof(float), st);
    }

    // K12: fused recurrent + parallel forward (L = 128): C stays in TMEM
    // (one sequential chunk chain per (head, 128-column tile)). Used from about
    // two thirds of a wave of chains on: measured crossover vs K1 + K2 (whose
    // grids also parallelise over chunks) at ~85-100 chains on 148 SMs, for
    // d_qk 128 and 256 alike and independent of the sequence length
    // (profiles/r01e_fused_crossover.txt)
    if (!states_only && tfla_k::fwd_fused_supported(g) && !tfla_host::env_flag("TFLA_NO_FUSED_FWD") &&
        (tfla_host::env_flag("TFLA_FORCE_FUSED_FWD") || 3 * g.BH * (g.dhv / 128) >= 2 * tfla_host::num_sms())) {
        tfla_k::FusedFwdArgs fa{};
        fa.g = g;
        fa.variant = variant;
        fa.gw = gw;
        fa.h = static_cast<__nv_bfloat16*>(out->h);
        fa.h_denom = out->h_denom;
        fa.n_states = is_exp ? out->n_states : nullptr;
        fa.n_final = is_exp ? out->n_final : nullptr;
        fa.c_states = out->c_states;
        fa.c_final = out->c_final;
        fa.c_init = c_init;
        fa.n_init = n_init;
        // The epilogue fused into K12's H drain is correct but slower than the
        // separate pass at the 7B shape (3.74 vs 1.28 ms for forward + output,
        // profiles/r02b_out_epilogue.txt): the y rows are a latency-bound load /
        // store loop in the row warps, which sit on the chunk chain, and the
        // per-chunk row-sum exchange couples the head's 4 CTAs (+0.46 ms alone).
        // Opt-in (TFLA_FUSED_OUT=1); the default runs tfla_output_norm_gate's pass.
        const bool fuse_out = og && tfla_k::fwd_fused_out_supported(g) && tfla_host::env_flag("TFLA_FUSED_OUT");
        if (fuse_out) {
            fa.o_pre = static_cast<const __nv_bfloat16*>(og->o_pre);
            fa.gamma = og->gamma;
            fa.y = static_cast<__nv_bfloat16*>(og->y);
            fa.eps = og->eps;
            fa.n_head = static_cast<int>(dims->n_head);
        }
        // debug: TFLA_TRACE_FWD=<file> dumps per-chunk clock64 events of one CTA
        const char* trace_file = getenv("TFLA_TRACE_FWD");
        long long* trace = nullptr;
        const size_t trace_n = static_cast<size_t>(g.NC) * 32;
        if (trace_file && *trace_file) {
            cudaMalloc(&trace, trace_n * sizeof(long long));
            cudaMemsetAsync(trace, 0, trace_n * sizeof(long long), st);
            fa.trace = trace;
            const char* cta = getenv("TFLA_TRACE_CTA");
            fa.trace_cta = cta ? atoi(cta) : 0;
        }
        {
            tfla_host::ProfScope ps(tfla_host::P_FWD_FUSED, st, 1);
            if (tfla_k::launch_fwd_fused(fa, in->q, in->k, in->v, saved, st)) return TFLA_ERR_CUDA;
        }
        if (trace) {
            std::vector<long long> hbuf(trace_n);
            cudaMemcpyAsync(hbuf.data(), trace, trace_n * sizeof(long long), cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            cudaFree(trace);
            if (FILE* f = fopen(trace_file, "w")) {
                for (int k = 0; k < g.NC; ++k) {
                    for (int e = 0; e < 32; ++e) fprintf(f, "%lld%c", hbuf[k * 32 + e], e == 31 ? '\n' : ' ');
                }
                fclose(f);
            }
        }
        if ((rc = check_cuda("fwd_fused"))) return rc;
        return og && !fuse_out ? output_pass(dims, out, og, st) : TFLA_OK;
    }

    // K1: C_{k+1} = gbar C_k + (a_bar o K)^T V  (+ n for exp)
    tfla_k::ScanArgs sa{};
    sa.g = g;
    sa.ntile = tfla_k::scan_ntile_for(g);
    if (const char* nenv = getenv("TFLA_SCAN_FWD_N"))  // experiment knob: 128-column K1 tiles
        if (atoi(nenv) == 128 && g.dhv % 128 == 0) sa.ntile = 128;
    sa.w = gw.ab;
    sa.gbar = gw.gbar;
    sa.c_states = out->c_states;
    sa.c_final = out->c_final;
    sa.u_part = is_exp ? reinterpret_cast<float*>(w8 + plan.u_part) : nullptr;
    sa.c_init = c_init;
    const bool scan2 = tfla_k::scan2_use(g, false);
    {
        tfla_host::ProfScope ps(tfla_host::P_SCAN_FWD, st, 1);
        if (scan2 ? tfla_k::launch_state_scan2(false, in->k, in->v, saved, sa, st)
                  : tfla_k::launch_state_scan(false, in->k, in->v, saved, sa, st))
            return TFLA_ERR_CUDA;
    }
    if ((rc = check_cuda("state_scan"))) return rc;
    if (is_exp) {
        tfla_host::ProfScope ps(tfla_host::P_QN, st, 1);
        tfla_k::launch_nscan(g, sa.u_part, gw.gbar, n_states, out->n_final, scan2 ? 1 : g.dhv / sa.ntile, st,
                             n_init);
        if ((rc = check_cuda("nscan"))) return rc;
    }
    if (states_only) return TFLA_OK;

    // K2: parallel TFLA forward
    tfla_k::FwdArgs fa{};
    fa.g = g;
    fa.ntile = ntile;
    fa.variant = variant;
    fa.gw = gw;
    fa.q = static_cast<const __nv_bfloat16*>(in->q);
    fa.n_states = n_states;
    fa.qn = gw.dinv;  // the forward does not use dinv: reuse that [BH][T] slot for q.n
    if (is_exp) {
        tfla_host::ProfScope ps(tfla_host::P_QN, st, 1);  // nscan + qn share a profile slot
        tfla_k::launch_qn(g, fa.q, n_states, gw.dinv, st);
        if ((rc = check_cuda("qn"))) return rc;
    }
    fa.h_denom = out->h_denom;
    {
        tfla_host::ProfScope ps(tfla_host::P_FWD_PARALLEL, st, 1);
        if (tfla_k::launch_fwd_parallel(fa, in->k, in->v, saved, out->h, st)) return TFLA_ERR_CUDA;
    }
    if ((rc = check_cuda("fwd_parallel"))) return rc;
    return og ? output_pass(dims, out, og, st) : TFLA_OK;
}

// tfla_forward_head (tiled.hpp:36-44 / tiled.cpp:59-240) over every head:
// the parallel part (K2) from states the caller materialised.
int parallel_impl(const tfla_dims* dims, const tfla_blocks* blocks, int variant, const tfla_inputs* in,
                  const tfla_states_in* sin, void* h, float* m_combine, float* h_denom, void* ws,
                  size_t ws_bytes, void* stream) {
    set_error("");
    int rc = tfla_host::validate_dims(dims);
    if (rc) return rc;
    if (!blocks) return set_error("tfla_forward_parallel: blocks is NULL"), TFLA_ERR_PARAMETER;
    if ((rc = tfla_host::validate_blocks(dims, blocks))) return rc;
    if (variant != TFLA_VARIANT_EXP && variant != TFLA_VARIANT_SIG)
        return set_error("unknown variant"), TFLA_ERR_PARAMETER;
    if (!in || !in->q || !in->k || !in->v || !in->i_pre || !in->f_pre)
        return set_error("forward: missing input tensor"), TFLA_ERR_PARAMETER;
    const bool is_exp = variant == TFLA_VARIANT_EXP;
    if (!sin || (!sin->saved_states && !sin->c_states) || (is_exp && (!sin->n_states || !sin->m_states)))
        return set_error("tfla_forward_parallel: missing states (C, and n, m for mLSTMexp)"), TFLA_ERR_PARAMETER;
    if (!h || !m_combine || !h_denom)
        return set_error("tfla_forward_parallel: h, m_combine and h_denom are required"), TFLA_ERR_PARAMETER;
    if ((rc = tfla_host::check_aligned({in->q, in->k, in->v, sin->saved_states, sin->c_states, h, ws},
                                       "tfla_forward_parallel")))
        return rc;
    const int ntile = tfla_host::pick_ntile(*dims, blocks);
    const tfla_host::WsPlan plan = tfla_host::plan_workspace(*dims, 0, ntile);
    if (!ws || ws_bytes < plan.total)
        return set_error("forward: workspace too small (need " + std::to_string(plan.total) + " bytes)"),
               TFLA_ERR_PARAMETER;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const tfla_k::Geom g = tfla_host::geom_of(*dims);
    const tfla_k::GateWS gw = tfla_host::gate_ws(plan, ws);
    uint8_t* w8 = static_cast<uint8_t*>(ws);
    {
        tfla_host::ProfScope ps(tfla_host::P_GATES_FWD, st, 1);
        tfla_k::launch_gates_fwd_given_m(g, variant, in->f_pre, in->i_pre, gw, sin->m_states, m_combine, st);
    }
    if ((rc = check_cuda("gates"))) return rc;
    const void* saved = sin->saved_states;
    if (!saved) {
        tfla_host::ProfScope ps(tfla_host::P_STATES_BF16, st, 1);
        tfla_k::launch_states_to_bf16(sin->c_states, reinterpret_cast<__nv_bfloat16*>(w8 + plan.saved), g, st);
        saved = w8 + plan.saved;
        if ((rc = check_cuda("states_to_bf16"))) return rc;
    }
    tfla_k::FwdArgs fa{};
    fa.g = g;
    fa.ntile = ntile;
    fa.variant = variant;
    fa.gw = gw;
    fa.q = static_cast<const __nv_bfloat16*>(in->q);
    fa.n_states = sin->n_states;
    fa.qn = gw.dinv;
    if (is_exp) {
        tfla_host::ProfScope ps(tfla_host::P_QN, st, 1);
        tfla_k::launch_qn(g, fa.q, sin->n_states, gw.dinv, st);
        if ((rc = check_cuda("qn"))) return rc;
    }
    fa.h_denom = h_denom;
    {
        tfla_host::ProfScope ps(tfla_host::P_FWD_PARALLEL, st, 1);
        if (tfla_k::launch_fwd_parallel(fa, in->k, in->v, saved, h, st)) return TFLA_ERR_CUDA;
    }
    return check_cuda("fwd_parallel");
}

// chunkwise_forward_frozen (chunkwise.cpp:304-394): the live state recurrence
// under the caller's max-state schedule m_states, the intra + inter combine
// under the caller's m_comb, divided by the caller's h_denom -- the function
// whose exact gradient tfla_chunkwise_backward computes. K0 (m and m_comb
// given) -> K1 state scan -> K2 with fixed denominators; no normaliser state.
int frozen_impl(const tfla_dims* dims, int variant, const tfla_inputs* in, const float* m_states,
                const float* m_combine, const float* h_denom, void* h, void* ws, size_t ws_bytes, void* stream) {
    set_error("");
    int rc = tfla_host::validate_dims(dims);
    if (rc) return rc;
    if (variant != TFLA_VARIANT_EXP && variant != TFLA_VARIANT_SIG)
        return set_error("unknown variant"), TFLA_ERR_PARAMETER;
    if (!in || !in->q || !in->k || !in->v || !in->i_pre || !in->f_pre || !h)
        return set_error("chunkwise_forward_frozen: missing input or output tensor"), TFLA_ERR_PARAMETER;
    const bool is_exp = variant == TFLA_VARIANT_EXP;
    // chunkwise.cpp:308-309: the pinned stats are required (for both variants)
    if (!m_states || !m_combine || !h_denom)
        return set_error("chunkwise_forward_frozen: missing saved stats"), TFLA_ERR_PARAMETER;
    if ((rc = tfla_host::check_aligned({in->q, in->k, in->v, h, ws}, "chunkwise_forward_frozen"))) return rc;
    const int ntile = tfla_host::pick_ntile(*dims, nullptr);
    const tfla_host::WsPlan plan = tfla_host::plan_workspace(*dims, 0, ntile);
    if (!ws || ws_bytes < plan.total)
        return set_error("forward: workspace too small (need " + std::to_string(plan.total) + " bytes)"),
               TFLA_ERR_PARAMETER;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const tfla_k::Geom g = tfla_host::geom_of(*dims);
    const tfla_k::GateWS gw = tfla_host::gate_ws(plan, ws);
    uint8_t* w8 = static_cast<uint8_t*>(ws);
    void* saved = w8 + plan.saved;
    {
        tfla_host::ProfScope ps(tfla_host::P_GATES_FWD, st, 1);
        tfla_k::launch_gates_fwd_given_m(g, variant, in->f_pre, in->i_pre, gw, is_exp ? m_states : nullptr, nullptr,
                                         st, is_exp ? m_combine : nullptr);
    }
    if ((rc = check_cuda("gates"))) return rc;
    tfla_k::ScanArgs sa{};
    sa.g = g;
    sa.ntile = tfla_k::scan_ntile_for(g);
    sa.w = gw.ab;
    sa.gbar = gw.gbar;
    {
        tfla_host::ProfScope ps(tfla_host::P_SCAN_FWD, st, 1);
        if (tfla_k::scan2_use(g, false) ? tfla_k::launch_state_scan2(false, in->k, in->v, saved, sa, st)
                                       : tfla_k::launch_state_scan(false, in->k, in->v, saved, sa, st))
            return TFLA_ERR_CUDA;
    }
    if ((rc = check_cuda("state_scan"))) return rc;
    tfla_k::FwdArgs fa{};
    fa.g = g;
    fa.ntile = ntile;
    fa.variant = variant;
    fa.gw = gw;
    fa.q = static_cast<const __nv_bfloat16*>(in->q);
    fa.den_fixed = is_exp ? h_denom : nullptr;
    {
        tfla_host::ProfScope ps(tfla_host::P_FWD_PARALLEL, st, 1);
        if (tfla_k::launch_fwd_parallel(fa, in->k, in->v, saved, h, st)) return TFLA_ERR_CUDA;
    }
    return check_cuda("fwd_parallel");
}

}  // namespace

extern "C" {

int tfla_chunkwise_forward_frozen(const tfla_dims* dims, int variant, const tfla_inputs* in, const float* m_states,
                                  const float* m_combine, const float* h_denom, void* h, void* workspace,
                                  size_t workspace_bytes, void* stream) {
    return frozen_impl(dims, variant, in, m_states, m_combine, h_denom, h, workspace, workspace_bytes, stream);
}

int tfla_state_recurrence(const tfla_dims* dims, int variant, const tfla_inputs* in, const tfla_fwd_out* out,
                          void* workspace, size_t workspace_bytes, void* stream) {
    return forward_impl(dims, nullptr, variant, in, out, workspace, workspace_bytes, stream, nullptr, true);
}

int tfla_forward_parallel(const tfla_dims* dims, const tfla_blocks* blocks, int variant, const tfla_inputs* in,
                          const tfla_states_in* states, void* h, float* m_combine, float* h_denom,
                          void* workspace, size_t workspace_bytes, void* stream) {
    return parallel_impl(dims, blocks, variant, in, states, h, m_combine, h_denom, workspace, workspace_bytes,
                         stream);
}


size_t tfla_workspace_bytes(const tfla_dims* dims, int variant, int pass) {
    (void)variant;
    if (!dims || tfla_host::validate_dims(dims)) return 0;
    return tfla_host::plan_workspace(*dims, pass ? 1 : 0, tfla_host::pick_ntile(*dims, nullptr))
        .total;
}

size_t tfla_saved_state_bytes(const tfla_dims* dims) {
    if (!dims || tfla_host::validate_dims(dims)) return 0;
    return static_cast<size_t>(dims->n_batch * dims->n_head) * (dims->T / dims->L) * dims->d_qk *
           dims->d_hv * 2;
}

int tfla_chunkwise_forward(const tfla_dims* dims, int variant, const tfla_inputs* in,
                           const tfla_fwd_out* out, void* workspace, size_t workspace_bytes,
                           void* stream) {
    return forward_impl(dims, nullptr, variant, in, out, workspace, workspace_bytes, stream);
}

int tfla_chunkwise_forward_gated(const tfla_dims* dims, int variant, const tfla_inputs* in,
                                 const tfla_fwd_out* out, const void* o_pre, const float* gamma, float eps,
                                 void* y, void* workspace, size_t workspace_bytes, void* stream) {
    const OutGate og{o_pre, gamma, eps, y};
    return forward_impl(dims, nullptr, variant, in, out, workspace, workspace_bytes, stream, nullptr, false, &og);
}

int tfla_chunkwise_forward_f32(const tfla_dims* dims, int variant, const tfla_inputs* in, const tfla_fwd_out* out,
                               void* ws, size_t ws_bytes, void* stream) {
    set_error("");
    int rc = tfla_host::validate_dims(dims);
    if (rc) return rc;
    if (variant != TFLA_VARIANT_EXP && variant != TFLA_VARIANT_SIG)
        return set_error("unknown variant"), TFLA_ERR_PARAMETER;
    if (!in || !in->q || !in->k || !in->v || !in->i_pre || !in->f_pre)
        return set_error("forward_f32: missing input tensor"), TFLA_ERR_PARAMETER;
    if (!out || !out->h || !out->m_states || !out->m_combine || !out->h_denom)
        return set_error("forward_f32: h, m_states, m_combine and h_denom are required"), TFLA_ERR_PARAMETER;
    const tfla_k::Geom g = tfla_host::geom_of(*dims);
    if (!tfla_k::fwd_f32_supported(g))
        return set_error("forward_f32: the fp32 path needs d_hv a multiple of 64, d_qk <= 256 and L * d_qk <= 8192"),
               TFLA_ERR_GEOMETRY;
    const tfla_host::WsPlan plan = tfla_host::plan_workspace(*dims, 0, tfla_host::pick_ntile(*dims, nullptr));
    if (!ws || ws_bytes < plan.total)
        return set_error("forward_f32: workspace too small (need " + std::to_string(plan.total) + " bytes)"),
               TFLA_ERR_PARAMETER;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const tfla_k::GateWS gw = tfla_host::gate_ws(plan, ws);
    {
        tfla_host::ProfScope ps(tfla_host::P_GATES_FWD, st, 2);
        tfla_k::launch_gates_fwd(g, variant, in->f_pre, in->i_pre, gw, out->m_states, out->m_combine, out->m_final,
                                 st);
    }
    if ((rc = check_cuda("gates"))) return rc;
    tfla_k::F32FwdArgs fa{};
    fa.g = g;
    fa.variant = variant;
    fa.gw = gw;
    fa.q = static_cast<const float*>(in->q);
    fa.k = static_cast<const float*>(in->k);
    fa.v = static_cast<const float*>(in->v);
    fa.h = static_cast<float*>(out->h);
    fa.h_denom = out->h_denom;
    fa.c_states = out->c_states;
    fa.n_states = out->n_states;
    fa.c_final = out->c_final;
    fa.n_final = out->n_final;
    if (variant == TFLA_VARIANT_SIG && out->n_states)
        cudaMemsetAsync(out->n_states, 0, static_cast<size_t>(g.BH) * (g.NC + 1) * g.dqk * sizeof(float), st);
    if (tfla_k::launch_fwd_f32(fa, st)) {
        check_cuda("fwd_f32");
        return TFLA_ERR_CUDA;
    }
    return check_cuda("fwd_f32");
}

int tfla_chunkwise_forward_init(const tfla_dims* dims, int variant, const tfla_inputs* in,
                                const tfla_state_in* init, const tfla_fwd_out* out, void* workspace,
                                size_t workspace_bytes, void* stream) {
    return forward_impl(dims, nullptr, variant, in, out, workspace, workspace_bytes, stream, init);
}

int tfla_forward(const tfla_dims* dims, const tfla_blocks* blocks, int variant,
                 const tfla_inputs* in, const tfla_fwd_out* out, void* workspace,
                 size_t workspace_bytes, void* stream) {
    if (!blocks) {
        set_error("tfla_forward: blocks is NULL");
        return TFLA_ERR_PARAMETER;
    }
    return forward_impl(dims, blocks, variant, in, out, workspace, workspace_bytes, stream);
}

}  // extern "C"
