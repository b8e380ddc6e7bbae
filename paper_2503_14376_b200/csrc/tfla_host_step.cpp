// tfla_host_step.cpp -- the reference-facing call with HOST buffers.
//
// The reference API (chunkwise_forward / chunkwise_backward, chunkwise.hpp:39-54)
// takes host tensors and returns host tensors. tfla_train_step_host is that
// boundary for one training step: q, k, v, i, f and dH come from host memory,
// h and every gradient go back to host memory, and the saved forward tensors
// (states, stabilisers, normaliser) stay on the device between the two passes.
// The batch is streamed in batch-row slices through device slots on
// three streams: slice b's H2D (copy engine), forward + backward (SMs) and D2H
// (the other copy engine) overlap the neighbouring slices', so the step runs at
// the PCIe rate when the host buffers are pinned. Stream-ordered on `stream`
// for the device work and the host outputs (complete once `stream` reaches the
// point of the call); the host inputs are read from the time of the call on.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "capi_internal.h"
#include "host_util.h"

using tfla_host::set_error;

namespace {

// device slots: one per batch row up to this budget (every row's H2D can then be
// issued back to back; fewer slots make a row's H2D wait for an older row's D2H)
constexpr size_t kSlotBudget = size_t(16) << 30;
constexpr int kMaxSlots = 64;

struct Slot {
    void *q = nullptr, *k = nullptr, *v = nullptr, *ip = nullptr, *fp = nullptr, *dh = nullptr;
    void *h = nullptr, *dq = nullptr, *dk = nullptr, *dv = nullptr, *dfp = nullptr, *dip = nullptr;
    void *m = nullptr, *mc = nullptr, *hd = nullptr, *saved = nullptr, *wsf = nullptr, *wsb = nullptr;
    size_t wsf_bytes = 0, wsb_bytes = 0;
    cudaEvent_t in_done = nullptr, cmp_done = nullptr, out_done = nullptr;
};

struct Pipeline {
    int device = -1;
    size_t bytes = 0;  // per-slot stride of the current carve
    size_t alloc = 0;  // bytes of the device allocation
    size_t layout[7] = {};  // component sizes the slots were carved for
    void* base = nullptr;
    int depth = 0;
    Slot slot[kMaxSlots];
    cudaStream_t s_in = nullptr, s_cmp = nullptr, s_out = nullptr;
    cudaEvent_t fork = nullptr, join_cmp = nullptr, join_out = nullptr;
    bool started[kMaxSlots] = {};
};

std::mutex g_mu;
std::vector<Pipeline*> g_pipes;  // one per device

size_t al(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

extern "C" int tfla_train_step_host(const tfla_dims* dims, int variant, const tfla_inputs* host_in,
                                    const void* d_h_host, const tfla_grads* host_grads, void* h_host,
                                    void* stream) {
    set_error("");
    int rc = tfla_host::validate_dims(dims);
    if (rc) return rc;
    if (variant != TFLA_VARIANT_EXP && variant != TFLA_VARIANT_SIG)
        return set_error("unknown variant"), TFLA_ERR_PARAMETER;
    if (!host_in || !host_in->q || !host_in->k || !host_in->v || !host_in->i_pre || !host_in->f_pre || !d_h_host ||
        !host_grads || !host_grads->dq || !host_grads->dk || !host_grads->dv || !host_grads->d_fpre ||
        !host_grads->d_ipre || !h_host)
        return set_error("train_step_host: missing host tensor"), TFLA_ERR_PARAMETER;

    // one batch row per slice: dims (T, L, d_qk, d_hv, NH, 1)
    tfla_dims sd = *dims;
    sd.n_batch = 1;
    const size_t rows = static_cast<size_t>(sd.n_head) * sd.T, NC = sd.T / sd.L;
    const size_t b_qk = rows * sd.d_qk * 2, b_hv = rows * sd.d_hv * 2, b_g = rows * 4;
    const size_t b_m = sd.n_head * (NC + 1) * 4, b_saved = static_cast<size_t>(sd.n_head) * NC * sd.d_qk * sd.d_hv * 2;
    const size_t wsf = tfla_workspace_bytes(&sd, variant, 0), wsb = tfla_workspace_bytes(&sd, variant, 1);
    // every per-slice call below sees this geometry: validate it once, before
    // any work is enqueued (so no slice can fail after earlier slices' copies)
    if ((rc = tfla_validate_dims(&sd))) return rc;
    if (!wsf || !wsb) return set_error("train_step_host: slice geometry has no workspace plan"), TFLA_ERR_GEOMETRY;
    const size_t need = al(b_qk) * 4 + al(b_hv) * 4 + al(b_g) * 4 + al(b_m) + al(b_g) * 2 + al(b_saved) + al(wsf) +
                        al(wsb);

    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_mu);
    if (static_cast<int>(g_pipes.size()) <= dev) g_pipes.resize(dev + 1, nullptr);
    Pipeline*& P = g_pipes[dev];
    if (!P) {
        P = new Pipeline();
        P->device = dev;
        cudaStreamCreateWithFlags(&P->s_in, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&P->s_cmp, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&P->s_out, cudaStreamNonBlocking);
        cudaEventCreateWithFlags(&P->fork, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&P->join_cmp, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&P->join_out, cudaEventDisableTiming);
        for (Slot& s : P->slot) {
            cudaEventCreateWithFlags(&s.in_done, cudaEventDisableTiming);
            cudaEventCreateWithFlags(&s.cmp_done, cudaEventDisableTiming);
            cudaEventCreateWithFlags(&s.out_done, cudaEventDisableTiming);
        }
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int depth = static_cast<int>(std::min<int64_t>(dims->n_batch, kMaxSlots));
    depth = std::max(2, std::min(depth, static_cast<int>(kSlotBudget / need)));
    // The slot pointers depend on every component size, not only on the total:
    // re-carve whenever any of them (or the depth) changes. Earlier users of the
    // memory (any slot, any stream) must be done before it is re-carved.
    const size_t layout[7] = {b_qk, b_hv, b_g, b_m, b_saved, wsf, wsb};
    const bool same_layout = std::equal(layout, layout + 7, P->layout) && P->depth == depth && P->base;
    if (!same_layout) {
        cudaStreamSynchronize(P->s_in);
        cudaStreamSynchronize(P->s_cmp);
        cudaStreamSynchronize(P->s_out);
        if (P->alloc < need * depth) {
            if (P->base) cudaFree(P->base);
            P->base = nullptr;
            P->alloc = 0;
            if (cudaMalloc(&P->base, need * depth) != cudaSuccess) {
                P->base = nullptr;
                P->bytes = 0;
                P->depth = 0;
                std::fill(P->layout, P->layout + 7, size_t(0));
                std::fill(P->started, P->started + kMaxSlots, false);
                cudaGetLastError();
                return set_error("train_step_host: cudaMalloc of the slice buffers failed"), TFLA_ERR_CUDA;
            }
            P->alloc = need * depth;
        }
        P->bytes = need;
        P->depth = depth;
        std::copy(layout, layout + 7, P->layout);
        std::fill(P->started, P->started + kMaxSlots, false);
        for (int i = 0; i < depth; ++i) {
            uint8_t* p = static_cast<uint8_t*>(P->base) + i * need;
            auto take = [&](size_t n) {
                void* r = p;
                p += al(n);
                return r;
            };
            Slot& s = P->slot[i];
            s.q = take(b_qk), s.k = take(b_qk), s.dq = take(b_qk), s.dk = take(b_qk);
            s.v = take(b_hv), s.dh = take(b_hv), s.h = take(b_hv), s.dv = take(b_hv);
            s.ip = take(b_g), s.fp = take(b_g), s.dfp = take(b_g), s.dip = take(b_g);
            s.m = take(b_m), s.mc = take(b_g), s.hd = take(b_g), s.saved = take(b_saved);
            s.wsf = take(wsf), s.wsb = take(wsb);
            s.wsf_bytes = wsf, s.wsb_bytes = wsb;
        }
    }
    // fork the compute and D2H streams off the caller's stream. The H2D stream
    // does not wait for it: the host inputs are ready when the call is made, so
    // the next step's uploads may overlap this step's downloads (each slot's
    // upload still waits for the previous compute that read the slot)
    cudaEventRecord(P->fork, st);
    cudaStreamWaitEvent(P->s_cmp, P->fork, 0);
    cudaStreamWaitEvent(P->s_out, P->fork, 0);
    // on a failure after work was enqueued: let every enqueued copy finish (the
    // caller may free its host buffers once this returns), keep the message
    auto drain = [&](int code) {
        const std::string msg = tfla_last_error();
        cudaStreamSynchronize(P->s_in);
        cudaStreamSynchronize(P->s_cmp);
        cudaStreamSynchronize(P->s_out);
        std::fill(P->started, P->started + kMaxSlots, false);
        set_error(msg);
        return code;
    };
    auto hp = [](const void* base, size_t slice_bytes, int64_t b) {
        return static_cast<const uint8_t*>(base) + static_cast<size_t>(b) * slice_bytes;
    };
    auto hpo = [](void* base, size_t slice_bytes, int64_t b) {
        return static_cast<uint8_t*>(base) + static_cast<size_t>(b) * slice_bytes;
    };
    for (int64_t b = 0; b < dims->n_batch; ++b) {
        const int i = static_cast<int>(b % P->depth);
        Slot& s = P->slot[i];
        // H2D of slice b once the previous compute on this slot consumed its inputs
        if (P->started[i]) cudaStreamWaitEvent(P->s_in, s.cmp_done, 0);
        cudaMemcpyAsync(s.q, hp(host_in->q, b_qk, b), b_qk, cudaMemcpyHostToDevice, P->s_in);
        cudaMemcpyAsync(s.k, hp(host_in->k, b_qk, b), b_qk, cudaMemcpyHostToDevice, P->s_in);
        cudaMemcpyAsync(s.v, hp(host_in->v, b_hv, b), b_hv, cudaMemcpyHostToDevice, P->s_in);
        cudaMemcpyAsync(s.ip, hp(host_in->i_pre, b_g, b), b_g, cudaMemcpyHostToDevice, P->s_in);
        cudaMemcpyAsync(s.fp, hp(host_in->f_pre, b_g, b), b_g, cudaMemcpyHostToDevice, P->s_in);
        cudaMemcpyAsync(s.dh, hp(d_h_host, b_hv, b), b_hv, cudaMemcpyHostToDevice, P->s_in);
        cudaEventRecord(s.in_done, P->s_in);
        // forward + backward of slice b (outputs overwrite the slot once its D2H is done)
        cudaStreamWaitEvent(P->s_cmp, s.in_done, 0);
        if (P->started[i]) cudaStreamWaitEvent(P->s_cmp, s.out_done, 0);
        const tfla_inputs di{s.q, s.k, s.v, static_cast<const float*>(s.ip), static_cast<const float*>(s.fp)};
        const tfla_fwd_out fo{s.h, nullptr, nullptr, static_cast<float*>(s.m), static_cast<float*>(s.mc),
                              static_cast<float*>(s.hd), nullptr, nullptr, nullptr, s.saved};
        if ((rc = tfla_chunkwise_forward(&sd, variant, &di, &fo, s.wsf, s.wsf_bytes, P->s_cmp))) return drain(rc);
        const tfla_bwd_in bi{s.dh, s.saved, nullptr, static_cast<const float*>(s.m),
                             static_cast<const float*>(s.mc), static_cast<const float*>(s.hd)};
        const tfla_grads go{s.dq, s.dk, s.dv, static_cast<float*>(s.dfp), static_cast<float*>(s.dip)};
        if ((rc = tfla_chunkwise_backward(&sd, variant, &di, &bi, &go, s.wsb, s.wsb_bytes, P->s_cmp))) return drain(rc);
        cudaEventRecord(s.cmp_done, P->s_cmp);
        // D2H of slice b's results
        cudaStreamWaitEvent(P->s_out, s.cmp_done, 0);
        cudaMemcpyAsync(hpo(h_host, b_hv, b), s.h, b_hv, cudaMemcpyDeviceToHost, P->s_out);
        cudaMemcpyAsync(hpo(host_grads->dq, b_qk, b), s.dq, b_qk, cudaMemcpyDeviceToHost, P->s_out);
        cudaMemcpyAsync(hpo(host_grads->dk, b_qk, b), s.dk, b_qk, cudaMemcpyDeviceToHost, P->s_out);
        cudaMemcpyAsync(hpo(host_grads->dv, b_hv, b), s.dv, b_hv, cudaMemcpyDeviceToHost, P->s_out);
        cudaMemcpyAsync(hpo(host_grads->d_fpre, b_g, b), s.dfp, b_g, cudaMemcpyDeviceToHost, P->s_out);
        cudaMemcpyAsync(hpo(host_grads->d_ipre, b_g, b), s.dip, b_g, cudaMemcpyDeviceToHost, P->s_out);
        cudaEventRecord(s.out_done, P->s_out);
        P->started[i] = true;
    }
    // join: the caller's stream continues once every result is in host memory
    cudaEventRecord(P->join_cmp, P->s_cmp);
    cudaEventRecord(P->join_out, P->s_out);
    cudaStreamWaitEvent(st, P->join_cmp, 0);
    cudaStreamWaitEvent(st, P->join_out, 0);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(std::string("train_step_host: ") + cudaGetErrorString(e)), TFLA_ERR_CUDA;
    return TFLA_OK;
}
