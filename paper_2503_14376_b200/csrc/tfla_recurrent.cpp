// tfla_recurrent.cpp -- C-ABI driver of the recurrent (decode) path
// (run_recurrent, recurrent.cpp:65-115, with an in-place initial / final state).
#include <cuda_runtime.h>

#include <string>

#include "capi_internal.h"
#include "host_util.h"
#include "kernels.h"
#include "workspace.h"

using tfla_host::set_error;

extern "C" int tfla_recurrent_step(const tfla_dims* d, int variant, const tfla_inputs* in, float* c_state,
                                   float* n_state, float* m_state, void* h, void* stream) {
    set_error("");
    if (!d) return set_error("dims is NULL"), TFLA_ERR_PARAMETER;
    // Dims::validate (core.cpp:9-16); L is not used by the step recurrence
    if (d->T < 1 || d->d_qk < 1 || d->d_hv < 1 || d->n_head < 1 || d->n_batch < 1)
        return set_error("recurrent: T, d_qk, d_hv, n_head, n_batch must be >= 1"), TFLA_ERR_GEOMETRY;
    if (d->n_batch > 65535 || d->n_head > 65535 || d->n_batch * d->n_head > 65535)
        return set_error("recurrent: B*NH must stay <= 65535 per call"), TFLA_ERR_GEOMETRY;
    if (!tfla_k::recurrent_supported(static_cast<int>(d->d_qk), static_cast<int>(d->d_hv)))
        return set_error("recurrent: B200 kernel needs d_qk in {64,128,256} and d_hv a multiple of 64"),
               TFLA_ERR_GEOMETRY;
    if (variant != TFLA_VARIANT_EXP && variant != TFLA_VARIANT_SIG)
        return set_error("unknown variant"), TFLA_ERR_PARAMETER;
    if (!in || !in->q || !in->k || !in->v || !in->i_pre || !in->f_pre || !c_state || !h)
        return set_error("recurrent: missing input, state or output tensor"), TFLA_ERR_PARAMETER;
    if (variant == TFLA_VARIANT_EXP && (!n_state || !m_state))
        return set_error("recurrent: mLSTMexp needs n_state and m_state"), TFLA_ERR_PARAMETER;

    tfla_k::RecurrentArgs a{};
    a.T = static_cast<int>(d->T);
    a.dhv = static_cast<int>(d->d_hv);
    a.variant = variant;
    a.q = static_cast<const __nv_bfloat16*>(in->q);
    a.k = static_cast<const __nv_bfloat16*>(in->k);
    a.v = static_cast<const __nv_bfloat16*>(in->v);
    a.i_pre = static_cast<const float*>(in->i_pre);
    a.f_pre = static_cast<const float*>(in->f_pre);
    a.c_state = c_state;
    a.n_state = n_state;
    a.m_state = m_state;
    a.h = static_cast<__nv_bfloat16*>(h);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    a.stab = tfla_host::stab_counters();
    // Every column-slice CTA of a head reads the initial n / m while slice 0
    // writes the final ones in place. With d_hv <= 512 the slices of a head are
    // one cluster and slice 0 writes after a cluster barrier; otherwise the
    // kernel reads a stream-ordered copy, so no CTA can observe another's update.
    float* nm_in = nullptr;
    const size_t BH = static_cast<size_t>(d->n_batch * d->n_head);
    if (variant == TFLA_VARIANT_EXP && !tfla_k::recurrent_cluster(static_cast<int>(d->d_hv))) {
        const size_t n_bytes = BH * d->d_qk * sizeof(float);
        if (cudaMallocAsync(reinterpret_cast<void**>(&nm_in), n_bytes + BH * sizeof(float), st) != cudaSuccess)
            return set_error("recurrent: cudaMallocAsync of the n/m copy failed"), TFLA_ERR_CUDA;
        cudaMemcpyAsync(nm_in, n_state, n_bytes, cudaMemcpyDeviceToDevice, st);
        cudaMemcpyAsync(nm_in + BH * d->d_qk, m_state, BH * sizeof(float), cudaMemcpyDeviceToDevice, st);
        a.n_in = nm_in;
        a.m_in = nm_in + BH * d->d_qk;
    }
    tfla_k::launch_recurrent(a, static_cast<int>(BH), static_cast<int>(d->d_qk), st);
    if (nm_in) cudaFreeAsync(nm_in, st);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(std::string("recurrent: ") + cudaGetErrorString(e)), TFLA_ERR_CUDA;
    return TFLA_OK;
}

extern "C" int tfla_output_norm_gate(const tfla_dims* d, const void* h_tilde, const void* o_pre, const float* gamma,
                                     float eps, void* h, void* stream) {
    set_error("");
    if (!d) return set_error("dims is NULL"), TFLA_ERR_PARAMETER;
    if (d->T < 1 || d->d_hv < 1 || d->n_head < 1 || d->n_batch < 1)
        return set_error("output: T, d_hv, n_head, n_batch must be >= 1"), TFLA_ERR_GEOMETRY;
    if (!tfla_k::output_supported(static_cast<int>(d->d_hv)))
        return set_error("output: B200 kernel needs d_hv a multiple of 8, <= 2048"), TFLA_ERR_GEOMETRY;
    if (!(eps >= 0.f)) return set_error("rms_norm: eps must be >= 0"), TFLA_ERR_PARAMETER;  // transfer.cpp:9
    if (!h_tilde || !o_pre || !gamma || !h) return set_error("output: missing tensor"), TFLA_ERR_PARAMETER;
    if (int rc = tfla_host::check_aligned({h_tilde, o_pre, h}, "output"))  // 16-byte vector accesses
        return rc;
    tfla_k::launch_output_norm_gate(static_cast<const __nv_bfloat16*>(h_tilde), static_cast<const __nv_bfloat16*>(o_pre),
                                    gamma, eps, static_cast<__nv_bfloat16*>(h), d->n_batch * d->n_head * d->T,
                                    static_cast<int>(d->T), static_cast<int>(d->n_head), static_cast<int>(d->d_hv),
                                    static_cast<cudaStream_t>(stream));
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(std::string("output: ") + cudaGetErrorString(e)), TFLA_ERR_CUDA;
    return TFLA_OK;
}

extern "C" int tfla_apply_gate_softcap(const tfla_dims* d, const float* i_pre, const float* f_pre, double cap,
                                       float* i_out, float* f_out, void* stream) {
    set_error("");
    if (!d) return set_error("dims is NULL"), TFLA_ERR_PARAMETER;
    if (d->T < 1 || d->n_head < 1 || d->n_batch < 1)
        return set_error("softcap: T, n_head, n_batch must be >= 1"), TFLA_ERR_GEOMETRY;
    if (!(cap > 0.0)) return set_error("softcap: cap must be > 0"), TFLA_ERR_PARAMETER;  // gates.cpp:16
    if (!i_pre || !f_pre || !i_out || !f_out) return set_error("softcap: missing tensor"), TFLA_ERR_PARAMETER;
    tfla_k::launch_gate_softcap(i_pre, f_pre, i_out, f_out, d->n_batch * d->n_head * d->T, cap,
                                static_cast<cudaStream_t>(stream));
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(std::string("softcap: ") + cudaGetErrorString(e)), TFLA_ERR_CUDA;
    return TFLA_OK;
}

// SequenceInputs::validate's all_finite (core.cpp:106-117) as an opt-in device
// pass: TFLA_ERR_NUMERIC when q, k, v, i_pre or f_pre holds a NaN / Inf.
// Synchronises `stream` (the verdict is read back to the host).
extern "C" int tfla_check_finite(const tfla_dims* d, const tfla_inputs* in, void* stream) {
    set_error("");
    if (!d) return set_error("dims is NULL"), TFLA_ERR_PARAMETER;
    if (d->T < 1 || d->d_qk < 1 || d->d_hv < 1 || d->n_head < 1 || d->n_batch < 1)
        return set_error("check_finite: T, d_qk, d_hv, n_head, n_batch must be >= 1"), TFLA_ERR_GEOMETRY;
    if (!in || !in->q || !in->k || !in->v || !in->i_pre || !in->f_pre)
        return set_error("check_finite: missing input tensor"), TFLA_ERR_PARAMETER;
    if (int rc = tfla_host::check_aligned({in->q, in->k, in->v, in->i_pre, in->f_pre}, "check_finite")) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    unsigned* flag = nullptr;
    if (cudaMallocAsync(reinterpret_cast<void**>(&flag), sizeof(unsigned), st) != cudaSuccess)
        return set_error("check_finite: cudaMallocAsync failed"), TFLA_ERR_CUDA;
    cudaMemsetAsync(flag, 0, sizeof(unsigned), st);
    const size_t rows = static_cast<size_t>(d->n_batch) * d->n_head * d->T;
    const int n_sm = tfla_host::num_sms();
    tfla_k::launch_nonfinite(in->q, rows * d->d_qk * 2, true, flag, n_sm, st);
    tfla_k::launch_nonfinite(in->k, rows * d->d_qk * 2, true, flag, n_sm, st);
    tfla_k::launch_nonfinite(in->v, rows * d->d_hv * 2, true, flag, n_sm, st);
    tfla_k::launch_nonfinite(in->i_pre, rows * 4, false, flag, n_sm, st);
    tfla_k::launch_nonfinite(in->f_pre, rows * 4, false, flag, n_sm, st);
    unsigned host = 0;
    cudaMemcpyAsync(&host, flag, sizeof(unsigned), cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(flag, st);
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return set_error(std::string("check_finite: ") + cudaGetErrorString(e)), TFLA_ERR_CUDA;
    if (host) return set_error("non-finite entries in sequence inputs"), TFLA_ERR_NUMERIC;
    return TFLA_OK;
}

// chunkwise_gates (gates.hpp:21-35 / gates.cpp:20-59) over every head, in f64:
// g_sum [B,NH,NC], b_cum [B,NH,T], a_tail [B,NH,T] (each nullable).
extern "C" int tfla_chunkwise_gates(const tfla_dims* d, int variant, const float* f_pre, const float* i_pre,
                                    double* g_sum, double* b_cum, double* a_tail, void* stream) {
    set_error("");
    int rc = tfla_host::validate_dims(d);
    if (rc) return rc;
    if (variant != TFLA_VARIANT_EXP && variant != TFLA_VARIANT_SIG)
        return set_error("unknown variant"), TFLA_ERR_PARAMETER;
    if (!f_pre || !i_pre) return set_error("chunkwise_gates: missing gate pre-activations"), TFLA_ERR_PARAMETER;
    const tfla_k::Geom g = tfla_host::geom_of(*d);
    tfla_k::launch_gates_export(g, variant, f_pre, i_pre, g_sum, b_cum, a_tail, static_cast<cudaStream_t>(stream));
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(std::string("chunkwise_gates: ") + cudaGetErrorString(e)), TFLA_ERR_CUDA;
    return TFLA_OK;
}
