// mlstm_b200.hpp -- C++ host API over the C ABI (tfla.h): the reference's
// mlstm:: chunkwise / TFLA entry points, same names and argument meaning,
// on device memory. Header-only; link with libtfla_b200.so and cudart.
//
//   reference (CPU, f64)                        here (B200, bf16 operands)
//   mlstm::Dims            core.hpp:27-39       mlstm::b200::Dims (= mlstm::Dims fields)
//   mlstm::BlockConfig     tiled.hpp:12-22      mlstm::b200::BlockConfig
//   mlstm::SequenceInputs  core.hpp:147-153     mlstm::b200::SequenceInputs (DeviceTensor)
//   chunkwise_forward      chunkwise.hpp:39     mlstm::b200::chunkwise_forward
//   tfla_forward           tiled.hpp:51         mlstm::b200::tfla_forward
//   chunkwise_backward     chunkwise.hpp:52     mlstm::b200::chunkwise_backward
//   tfla_backward          tiled.hpp:88         mlstm::b200::tfla_backward
//   GeometryError / ParameterError / NumericError (core.hpp:11-23): same names.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <map>
#include <mutex>
#include <vector>

#include "tfla/tfla.h"

namespace mlstm::b200 {

struct GeometryError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct ParameterError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct NumericError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(int rc) {
    if (rc == TFLA_OK) return;
    const std::string msg = tfla_last_error();
    switch (rc) {
        case TFLA_ERR_GEOMETRY: throw GeometryError(msg);
        case TFLA_ERR_PARAMETER: throw ParameterError(msg);
        case TFLA_ERR_NUMERIC: throw NumericError(msg);
        default: throw CudaError(msg);
    }
}

enum class Variant { Exp = TFLA_VARIANT_EXP, Sig = TFLA_VARIANT_SIG };

struct Dims {
    long T = 1, L = 1, d_qk = 1, d_hv = 1, n_head = 1, n_batch = 1;
    long n_chunk() const { return T / L; }
    tfla_dims c() const { return {T, L, d_qk, d_hv, n_head, n_batch}; }
    void validate_chunked() const {
        tfla_dims d = c();
        check(tfla_validate_dims(&d));
    }
};

struct BlockConfig {
    long b_lhq = 0, b_lkv = 0, b_dqk = 0, b_dhv = 0;
    tfla_blocks c() const { return {b_lhq, b_lkv, b_dqk, b_dhv}; }
    void validate(const Dims& dims) const {
        tfla_dims d = dims.c();
        tfla_blocks b = c();
        check(tfla_validate_blocks(&d, &b));
    }
    static BlockConfig pick_default(const Dims& dims) {
        tfla_dims d = dims.c();
        tfla_blocks b{};
        check(tfla_pick_default_blocks(&d, &b));
        return {b.b_lhq, b.b_lkv, b.b_dqk, b.b_dhv};
    }
};

// Owning device buffer with a shape (element size fixed at construction).
class DeviceTensor {
  public:
    DeviceTensor() = default;
    DeviceTensor(std::vector<long> shape, size_t elem_bytes) : shape_(std::move(shape)), esize_(elem_bytes) {
        numel_ = 1;
        for (long d : shape_) numel_ *= d;
        if (numel_ > 0 && cudaMalloc(&ptr_, bytes()) != cudaSuccess) throw CudaError("cudaMalloc failed");
    }
    ~DeviceTensor() {
        if (ptr_) cudaFree(ptr_);
    }
    DeviceTensor(DeviceTensor&& o) noexcept { *this = std::move(o); }
    DeviceTensor& operator=(DeviceTensor&& o) noexcept {
        std::swap(ptr_, o.ptr_);
        std::swap(shape_, o.shape_);
        std::swap(numel_, o.numel_);
        std::swap(esize_, o.esize_);
        return *this;
    }
    DeviceTensor(const DeviceTensor&) = delete;
    DeviceTensor& operator=(const DeviceTensor&) = delete;

    void* data() const { return ptr_; }
    template <class T>
    T* as() const { return static_cast<T*>(ptr_); }
    const std::vector<long>& shape() const { return shape_; }
    long numel() const { return numel_; }
    size_t bytes() const { return static_cast<size_t>(numel_) * esize_; }
    bool empty() const { return numel_ == 0; }

    static DeviceTensor bf16(std::vector<long> s) { return DeviceTensor(std::move(s), 2); }
    static DeviceTensor f32(std::vector<long> s) { return DeviceTensor(std::move(s), 4); }

  private:
    void* ptr_ = nullptr;
    std::vector<long> shape_;
    long numel_ = 0;
    size_t esize_ = 0;
};

// q, k [B,H,T,dqk] bf16; v [B,H,T,dhv] bf16; i_pre, f_pre [B,H,T] fp32.
struct SequenceInputs {
    DeviceTensor q, k, v, i_pre, f_pre;
    tfla_inputs c() const { return {q.data(), k.data(), v.data(), i_pre.as<float>(), f_pre.as<float>()}; }
    void validate(const Dims& d) const {
        const std::vector<long> qk{d.n_batch, d.n_head, d.T, d.d_qk};
        const std::vector<long> hv{d.n_batch, d.n_head, d.T, d.d_hv};
        const std::vector<long> g{d.n_batch, d.n_head, d.T};
        if (q.shape() != qk || k.shape() != qk) throw GeometryError("q/k shape mismatch with dims");
        if (v.shape() != hv) throw GeometryError("v shape mismatch with dims");
        if (i_pre.shape() != g || f_pre.shape() != g)
            throw GeometryError("gate pre-activation shape mismatch with dims");
    }
    // all_finite (core.cpp:114-116) as the library's device pass -> NumericError
    void check_finite(const Dims& d, cudaStream_t st = nullptr) const {
        validate(d);
        const tfla_dims cd = d.c();
        const tfla_inputs ci = c();
        check(tfla_check_finite(&cd, &ci, st));
    }
};

// ---- recurrent (decode) path: run_recurrent (recurrent.hpp:42-43) with
// RecurrentOptions::initial_state (recurrent.hpp:23-27); the state is carried
// in place (fp32 C [B,H,dqk,dhv], n [B,H,dqk], m [B,H]).
struct MemoryState {
    DeviceTensor C, n, m;
    static MemoryState zero(const Dims& d, cudaStream_t st = nullptr) {
        MemoryState s{DeviceTensor::f32({d.n_batch, d.n_head, d.d_qk, d.d_hv}),
                      DeviceTensor::f32({d.n_batch, d.n_head, d.d_qk}), DeviceTensor::f32({d.n_batch, d.n_head})};
        cudaMemsetAsync(s.C.data(), 0, s.C.bytes(), st);
        cudaMemsetAsync(s.n.data(), 0, s.n.bytes(), st);
        cudaMemsetAsync(s.m.data(), 0, s.m.bytes(), st);
        return s;
    }
};

struct ChunkStates {
    DeviceTensor C;  // fp32 [B,H,NC+1,dqk,dhv] (empty when not requested)
    DeviceTensor n;  // fp32 [B,H,NC+1,dqk]
    DeviceTensor m;  // fp32 [B,H,NC+1]
};
struct SavedStats {
    DeviceTensor m_combine, h_denom;  // fp32 [B,H,T]
};
struct ChunkwiseForward {
    DeviceTensor h_tilde;  // bf16 [B,H,T,dhv]
    ChunkStates states;
    SavedStats stats;
    DeviceTensor saved_states;  // bf16 [B,H,NC,dqk,dhv]
    DeviceTensor C_final, n_final, m_final;
};
struct Gradients {
    DeviceTensor dq, dk, dv, d_fpre, d_ipre;
};

// Workspace cache (one per process; grown on demand).
class Workspace {
  public:
    void* get(size_t bytes) {
        if (bytes > size_) {
            if (ptr_) cudaFree(ptr_);
            ptr_ = nullptr;
            if (cudaMalloc(&ptr_, bytes) != cudaSuccess) throw CudaError("workspace cudaMalloc failed");
            size_ = bytes;
        }
        return ptr_;
    }
    size_t size() const { return size_; }
    ~Workspace() {
        if (ptr_) cudaFree(ptr_);
    }

  private:
    void* ptr_ = nullptr;
    size_t size_ = 0;
};

// One workspace per stream (calls on one stream are ordered; calls on
// different streams must not share scratch memory).
inline Workspace& default_workspace(cudaStream_t st = nullptr) {
    static std::mutex mu;
    static std::map<cudaStream_t, Workspace> ws;
    std::lock_guard<std::mutex> g(mu);
    return ws[st];
}

namespace detail {
struct OutGateArgs {  // tfla_chunkwise_forward_gated: y = sigmoid(o_pre) * rms_norm(h_tilde; gamma, eps)
    const DeviceTensor* o_pre;
    const DeviceTensor* gamma;
    float eps;
    DeviceTensor* y;
};

inline ChunkwiseForward forward(const SequenceInputs& in, const Dims& d, const BlockConfig* blocks, Variant v,
                                bool all_states, cudaStream_t st, const MemoryState* init = nullptr,
                                const OutGateArgs* og = nullptr) {
    d.validate_chunked();
    if (blocks) blocks->validate(d);
    in.validate(d);
    const long B = d.n_batch, H = d.n_head, T = d.T, NC = d.n_chunk();
    ChunkwiseForward out;
    out.h_tilde = DeviceTensor::bf16({B, H, T, d.d_hv});
    if (all_states) {
        out.states.C = DeviceTensor::f32({B, H, NC + 1, d.d_qk, d.d_hv});
        out.states.n = DeviceTensor::f32({B, H, NC + 1, d.d_qk});
    }
    out.states.m = DeviceTensor::f32({B, H, NC + 1});
    out.stats.m_combine = DeviceTensor::f32({B, H, T});
    out.stats.h_denom = DeviceTensor::f32({B, H, T});
    out.saved_states = DeviceTensor::bf16({B, H, NC, d.d_qk, d.d_hv});
    out.C_final = DeviceTensor::f32({B, H, d.d_qk, d.d_hv});
    out.n_final = DeviceTensor::f32({B, H, d.d_qk});
    out.m_final = DeviceTensor::f32({B, H});
    tfla_fwd_out o{out.h_tilde.data(),          out.states.C.as<float>(),     out.states.n.as<float>(),
                   out.states.m.as<float>(),    out.stats.m_combine.as<float>(), out.stats.h_denom.as<float>(),
                   out.C_final.as<float>(),     out.n_final.as<float>(),      out.m_final.as<float>(),
                   out.saved_states.data()};
    tfla_dims dd = d.c();
    tfla_inputs ii = in.c();
    const size_t wsb = tfla_workspace_bytes(&dd, static_cast<int>(v), 0);
    void* ws = default_workspace(st).get(wsb);
    if (og) {
        if (og->o_pre->shape() != out.h_tilde.shape() || og->gamma->shape() != std::vector<long>{H, d.d_hv})
            throw GeometryError("chunkwise_forward_gated: o_pre / gamma shape mismatch");
        *og->y = DeviceTensor::bf16({B, H, T, d.d_hv});
        check(tfla_chunkwise_forward_gated(&dd, static_cast<int>(v), &ii, &o, og->o_pre->data(),
                                           og->gamma->as<float>(), og->eps, og->y->data(), ws,
                                           default_workspace(st).size(), st));
    } else if (init) {
        if (blocks) throw ParameterError("an initial state is supported on chunkwise_forward only");
        const tfla_state_in si{init->C.as<float>(), init->n.as<float>(), init->m.as<float>()};
        check(tfla_chunkwise_forward_init(&dd, static_cast<int>(v), &ii, &si, &o, ws, default_workspace(st).size(), st));
    } else if (blocks) {
        tfla_blocks bb = blocks->c();
        check(tfla_forward(&dd, &bb, static_cast<int>(v), &ii, &o, ws, default_workspace(st).size(), st));
    } else {
        check(tfla_chunkwise_forward(&dd, static_cast<int>(v), &ii, &o, ws, default_workspace(st).size(), st));
    }
    return out;
}

inline Gradients backward(const SequenceInputs& in, const Dims& d, const BlockConfig* blocks, Variant v,
                          const DeviceTensor& d_h, const ChunkStates& states, const SavedStats& stats,
                          const DeviceTensor* saved_states, cudaStream_t st) {
    d.validate_chunked();
    if (blocks) blocks->validate(d);
    in.validate(d);
    if (states.m.empty() || stats.m_combine.empty() || stats.h_denom.empty() ||
        ((!saved_states || saved_states->empty()) && states.C.empty()))
        throw ParameterError("chunkwise_backward: missing saved forward tensors");
    if (d_h.shape() != in.v.shape()) throw GeometryError("chunkwise_backward: dH shape mismatch");
    Gradients g;
    g.dq = DeviceTensor::bf16(in.q.shape());
    g.dk = DeviceTensor::bf16(in.k.shape());
    g.dv = DeviceTensor::bf16(in.v.shape());
    g.d_fpre = DeviceTensor::f32(in.f_pre.shape());
    g.d_ipre = DeviceTensor::f32(in.i_pre.shape());
    tfla_bwd_in b{d_h.data(), saved_states ? saved_states->data() : nullptr, states.C.as<float>(),
                  states.m.as<float>(), stats.m_combine.as<float>(), stats.h_denom.as<float>()};
    tfla_grads gg{g.dq.data(), g.dk.data(), g.dv.data(), g.d_fpre.as<float>(), g.d_ipre.as<float>()};
    tfla_dims dd = d.c();
    tfla_inputs ii = in.c();
    const size_t wsb = tfla_workspace_bytes(&dd, static_cast<int>(v), 1);
    void* ws = default_workspace(st).get(wsb);
    if (blocks) {
        tfla_blocks bb = blocks->c();
        check(tfla_backward(&dd, &bb, static_cast<int>(v), &ii, &b, &gg, ws, default_workspace(st).size(), st));
    } else {
        check(tfla_chunkwise_backward(&dd, static_cast<int>(v), &ii, &b, &gg, ws, default_workspace(st).size(), st));
    }
    return g;
}
}  // namespace detail

inline ChunkwiseForward chunkwise_forward(const SequenceInputs& in, const Dims& d, Variant v,
                                          cudaStream_t st = nullptr, bool all_states = true) {
    return detail::forward(in, d, nullptr, v, all_states, st);
}
// chunkwise_forward on fp32 operands (the reference's <float, float>
// instantiation, chunkwise.cpp:183-194): in.q / k / v hold fp32 tensors; h and
// the C / n states come back fp32 (tfla_chunkwise_forward_f32, CUDA cores).
inline ChunkwiseForward chunkwise_forward_f32(const SequenceInputs& in, const Dims& d, Variant v,
                                              cudaStream_t st = nullptr, bool all_states = true) {
    d.validate_chunked();
    const long B = d.n_batch, H = d.n_head, T = d.T, NC = d.n_chunk();
    ChunkwiseForward out;
    out.h_tilde = DeviceTensor::f32({B, H, T, d.d_hv});
    if (all_states) {
        out.states.C = DeviceTensor::f32({B, H, NC + 1, d.d_qk, d.d_hv});
        out.states.n = DeviceTensor::f32({B, H, NC + 1, d.d_qk});
    }
    out.states.m = DeviceTensor::f32({B, H, NC + 1});
    out.stats.m_combine = DeviceTensor::f32({B, H, T});
    out.stats.h_denom = DeviceTensor::f32({B, H, T});
    out.C_final = DeviceTensor::f32({B, H, d.d_qk, d.d_hv});
    out.n_final = DeviceTensor::f32({B, H, d.d_qk});
    out.m_final = DeviceTensor::f32({B, H});
    tfla_fwd_out o{out.h_tilde.data(),          out.states.C.as<float>(),     out.states.n.as<float>(),
                   out.states.m.as<float>(),    out.stats.m_combine.as<float>(), out.stats.h_denom.as<float>(),
                   out.C_final.as<float>(),     out.n_final.as<float>(),      out.m_final.as<float>(),
                   nullptr};
    tfla_dims dd = d.c();
    tfla_inputs ii = in.c();
    const size_t wsb = tfla_workspace_bytes(&dd, static_cast<int>(v), 0);
    void* ws = default_workspace(st).get(wsb);
    check(tfla_chunkwise_forward_f32(&dd, static_cast<int>(v), &ii, &o, ws, default_workspace(st).size(), st));
    return out;
}

// chunkwise_forward + the cell output epilogue (eq. 5) fused into the
// H store: y = sigmoid(o_pre) * rms_norm(h_tilde; gamma[head], eps).
inline ChunkwiseForward chunkwise_forward_gated(const SequenceInputs& in, const Dims& d, Variant v,
                                                const DeviceTensor& o_pre, const DeviceTensor& gamma, float eps,
                                                DeviceTensor& y, cudaStream_t st = nullptr, bool all_states = true) {
    const detail::OutGateArgs og{&o_pre, &gamma, eps, &y};
    return detail::forward(in, d, nullptr, v, all_states, st, nullptr, &og);
}
inline ChunkwiseForward tfla_forward(const SequenceInputs& in, const Dims& d, const BlockConfig& blocks, Variant v,
                                     cudaStream_t st = nullptr, bool all_states = true) {
    return detail::forward(in, d, &blocks, v, all_states, st);
}
inline Gradients chunkwise_backward(const SequenceInputs& in, const Dims& d, Variant v, const DeviceTensor& d_h,
                                    const ChunkStates& states, const SavedStats& stats,
                                    const DeviceTensor* saved_states = nullptr, cudaStream_t st = nullptr) {
    return detail::backward(in, d, nullptr, v, d_h, states, stats, saved_states, st);
}
inline Gradients tfla_backward(const SequenceInputs& in, const Dims& d, const BlockConfig& blocks, Variant v,
                               const DeviceTensor& d_h, const ChunkStates& states, const SavedStats& stats,
                               const DeviceTensor* saved_states = nullptr, cudaStream_t st = nullptr) {
    return detail::backward(in, d, &blocks, v, d_h, states, stats, saved_states, st);
}

// ---- split entry points (tiled.hpp:36-84, detail_kernels.hpp:38-44)
struct TfLaDqResult {
    DeviceTensor dq, d_b_cum;  // bf16 [B,H,T,dqk]; fp32 [B,H,T]
};
struct TfLaDkResult {
    DeviceTensor dk, d_a_tail, d_b_cum, d_i_log;
};

namespace detail {
inline tfla_bwd_in bwd_in(const SequenceInputs& in, const Dims& d, const BlockConfig& blocks,
                          const DeviceTensor& d_h, const ChunkStates& states, const SavedStats& stats,
                          const DeviceTensor* saved_states) {
    d.validate_chunked();
    blocks.validate(d);
    in.validate(d);
    if (states.m.empty() || stats.m_combine.empty() || stats.h_denom.empty() ||
        ((!saved_states || saved_states->empty()) && states.C.empty()))
        throw ParameterError("tiled backward: missing saved forward tensors");
    if (d_h.shape() != in.v.shape()) throw GeometryError("tiled backward: dH shape mismatch");
    return {d_h.data(), saved_states ? saved_states->data() : nullptr, states.C.as<float>(), states.m.as<float>(),
            stats.m_combine.as<float>(), stats.h_denom.as<float>()};
}
}  // namespace detail

inline TfLaDqResult tfla_backward_dq(const SequenceInputs& in, const Dims& d, const BlockConfig& blocks, Variant v,
                                     const DeviceTensor& d_h, const ChunkStates& states, const SavedStats& stats,
                                     const DeviceTensor* saved_states = nullptr, cudaStream_t st = nullptr) {
    const tfla_bwd_in b = detail::bwd_in(in, d, blocks, d_h, states, stats, saved_states);
    TfLaDqResult r{DeviceTensor::bf16(in.q.shape()), DeviceTensor::f32(in.f_pre.shape())};
    const tfla_dims dd = d.c();
    const tfla_blocks bb = blocks.c();
    const tfla_inputs ii = in.c();
    void* ws = default_workspace(st).get(tfla_workspace_bytes(&dd, static_cast<int>(v), 1));
    check(tfla_backward_dq(&dd, &bb, static_cast<int>(v), &ii, &b, r.dq.data(), r.d_b_cum.as<float>(), ws,
                           default_workspace(st).size(), st));
    return r;
}
inline TfLaDkResult tfla_backward_dk(const SequenceInputs& in, const Dims& d, const BlockConfig& blocks, Variant v,
                                     const DeviceTensor& d_h, const ChunkStates& states, const SavedStats& stats,
                                     const DeviceTensor* saved_states = nullptr, cudaStream_t st = nullptr) {
    const tfla_bwd_in b = detail::bwd_in(in, d, blocks, d_h, states, stats, saved_states);
    const auto& g = in.f_pre.shape();
    TfLaDkResult r{DeviceTensor::bf16(in.k.shape()), DeviceTensor::f32(g), DeviceTensor::f32(g), DeviceTensor::f32(g)};
    const tfla_dims dd = d.c();
    const tfla_blocks bb = blocks.c();
    const tfla_inputs ii = in.c();
    void* ws = default_workspace(st).get(tfla_workspace_bytes(&dd, static_cast<int>(v), 1));
    check(tfla_backward_dk(&dd, &bb, static_cast<int>(v), &ii, &b, r.dk.data(), r.d_a_tail.as<float>(),
                           r.d_b_cum.as<float>(), r.d_i_log.as<float>(), ws, default_workspace(st).size(), st));
    return r;
}
inline DeviceTensor tfla_backward_dv(const SequenceInputs& in, const Dims& d, const BlockConfig& blocks, Variant v,
                                     const DeviceTensor& d_h, const ChunkStates& states, const SavedStats& stats,
                                     const DeviceTensor* saved_states = nullptr, cudaStream_t st = nullptr) {
    const tfla_bwd_in b = detail::bwd_in(in, d, blocks, d_h, states, stats, saved_states);
    DeviceTensor dv = DeviceTensor::bf16(in.v.shape());
    const tfla_dims dd = d.c();
    const tfla_blocks bb = blocks.c();
    const tfla_inputs ii = in.c();
    void* ws = default_workspace(st).get(tfla_workspace_bytes(&dd, static_cast<int>(v), 1));
    check(tfla_backward_dv(&dd, &bb, static_cast<int>(v), &ii, &b, dv.data(), ws, default_workspace(st).size(), st));
    return dv;
}

// state_recurrence_head over every head: C (fp32), n, m and the bf16 operand copy.
inline ChunkwiseForward state_recurrence(const SequenceInputs& in, const Dims& d, Variant v,
                                         cudaStream_t st = nullptr) {
    d.validate_chunked();
    in.validate(d);
    const long B = d.n_batch, H = d.n_head, NC = d.n_chunk();
    ChunkwiseForward f;
    f.states.C = DeviceTensor::f32({B, H, NC + 1, d.d_qk, d.d_hv});
    f.states.n = DeviceTensor::f32({B, H, NC + 1, d.d_qk});
    f.states.m = DeviceTensor::f32({B, H, NC + 1});
    f.saved_states = DeviceTensor::bf16({B, H, NC, d.d_qk, d.d_hv});
    tfla_fwd_out o{};
    o.c_states = f.states.C.as<float>();
    o.n_states = f.states.n.as<float>();
    o.m_states = f.states.m.as<float>();
    o.saved_states = f.saved_states.data();
    const tfla_dims dd = d.c();
    const tfla_inputs ii = in.c();
    void* ws = default_workspace(st).get(tfla_workspace_bytes(&dd, static_cast<int>(v), 0));
    check(tfla_state_recurrence(&dd, static_cast<int>(v), &ii, &o, ws, default_workspace(st).size(), st));
    return f;
}

// tfla_forward_head over every head, from state_recurrence's states: fills
// f.h_tilde and f.stats.
inline void tfla_forward_parallel(const SequenceInputs& in, const Dims& d, const BlockConfig& blocks, Variant v,
                                  ChunkwiseForward& f, cudaStream_t st = nullptr) {
    d.validate_chunked();
    blocks.validate(d);
    in.validate(d);
    const long B = d.n_batch, H = d.n_head;
    f.h_tilde = DeviceTensor::bf16({B, H, d.T, d.d_hv});
    f.stats.m_combine = DeviceTensor::f32({B, H, d.T});
    f.stats.h_denom = DeviceTensor::f32({B, H, d.T});
    const tfla_states_in s{f.saved_states.empty() ? nullptr : f.saved_states.data(), f.states.C.as<float>(),
                           f.states.n.as<float>(), f.states.m.as<float>()};
    const tfla_dims dd = d.c();
    const tfla_blocks bb = blocks.c();
    const tfla_inputs ii = in.c();
    void* ws = default_workspace(st).get(tfla_workspace_bytes(&dd, static_cast<int>(v), 0));
    check(tfla_forward_parallel(&dd, &bb, static_cast<int>(v), &ii, &s, f.h_tilde.data(),
                                f.stats.m_combine.as<float>(), f.stats.h_denom.as<float>(), ws,
                                default_workspace(st).size(), st));
}

// One training step over HOST buffers (tfla_train_step_host): the reference's
// host-tensor boundary. Host layouts as the device ones; pinned memory for the
// PCIe rate. The outputs are complete when `st` reaches this point.
inline void train_step_host(const Dims& d, Variant v, const tfla_inputs& host_in, const void* d_h_host,
                            const tfla_grads& host_grads, void* h_host, cudaStream_t st = nullptr) {
    d.validate_chunked();
    const tfla_dims cd = d.c();
    check(tfla_train_step_host(&cd, static_cast<int>(v), &host_in, d_h_host, &host_grads, h_host, st));
}

// Folds step_exp / step_sig (recurrent.cpp:9-63) over d.T steps; returns
// h_tilde bf16 [B,H,T,dhv] and leaves the final state in `state`.
inline DeviceTensor recurrent_step(const SequenceInputs& in, const Dims& d, Variant v, MemoryState& state,
                                   cudaStream_t st = nullptr) {
    in.validate(d);
    DeviceTensor h = DeviceTensor::bf16({d.n_batch, d.n_head, d.T, d.d_hv});
    const tfla_dims cd = d.c();
    const tfla_inputs ci = in.c();
    check(tfla_recurrent_step(&cd, static_cast<int>(v), &ci, state.C.as<float>(), state.n.as<float>(),
                              state.m.as<float>(), h.data(), st));
    return h;
}

// chunkwise_forward continuing from an initial state (tfla_chunkwise_forward_init).
inline ChunkwiseForward chunkwise_forward_from(const SequenceInputs& in, const Dims& d, Variant v,
                                               const MemoryState& init, cudaStream_t st = nullptr,
                                               bool all_states = true) {
    return detail::forward(in, d, nullptr, v, all_states, st, &init);
}

// chunkwise_forward_frozen (chunkwise.hpp:42-46): the forward under pinned
// max states / m_combine / h_denom -- what chunkwise_backward differentiates.
inline DeviceTensor chunkwise_forward_frozen(const SequenceInputs& in, const Dims& d, Variant v,
                                             const ChunkStates& frozen_states, const SavedStats& frozen_stats,
                                             cudaStream_t st = nullptr) {
    d.validate_chunked();
    in.validate(d);
    if (!frozen_states.m.data() || !frozen_stats.m_combine.data() || !frozen_stats.h_denom.data())
        throw ParameterError("chunkwise_forward_frozen: missing saved stats");
    DeviceTensor h = DeviceTensor::bf16({d.n_batch, d.n_head, d.T, d.d_hv});
    const tfla_dims cd = d.c();
    const tfla_inputs ci = in.c();
    const size_t ws_bytes = tfla_workspace_bytes(&cd, static_cast<int>(v), 0);
    void* ws = default_workspace(st).get(ws_bytes);
    check(tfla_chunkwise_forward_frozen(&cd, static_cast<int>(v), &ci, frozen_states.m.as<float>(),
                                        frozen_stats.m_combine.as<float>(), frozen_stats.h_denom.as<float>(),
                                        h.data(), ws, ws_bytes, st));
    return h;
}

// mlstm::stab (core.cpp:145-166) for the device kernels: enable the audit,
// then read {checks, violations, max argument} (reset on read).
namespace stab {
struct Counts {
    int64_t checks = 0, violations = 0;
    double max_arg = 0.0;
};
inline void enable(bool on = true) { check(tfla_stab_enable(on ? 1 : 0)); }
inline Counts read() {
    Counts c;
    check(tfla_stab_read(&c.checks, &c.violations, &c.max_arg));
    return c;
}
}  // namespace stab

// detail::kv_block_count / block_needs_mask (tiled.cpp:43-49)
inline long kv_block_count(long i_lq, const BlockConfig& blocks) {
    const tfla_blocks b = blocks.c();
    const int64_t r = tfla_kv_block_count(i_lq, &b);
    if (r < 0) throw ParameterError("kv_block_count: bad arguments");
    return static_cast<long>(r);
}
inline bool block_needs_mask(long i_kv_1based, long i_lq, const BlockConfig& blocks) {
    const tfla_blocks b = blocks.c();
    const int r = tfla_block_needs_mask(i_kv_1based, i_lq, &b);
    if (r < 0) throw ParameterError("block_needs_mask: bad arguments");
    return r != 0;
}

// h = sigmoid(o_pre) * rms_norm(h_tilde; gamma[head], eps)  (eq. 5, transfer.cpp:8-18)
inline DeviceTensor output_norm_gate(const DeviceTensor& h_tilde, const DeviceTensor& o_pre,
                                     const DeviceTensor& gamma, float eps, cudaStream_t st = nullptr) {
    const auto& s = h_tilde.shape();
    if (s.size() != 4 || o_pre.shape() != s || gamma.shape() != std::vector<long>{s[1], s[3]})
        throw GeometryError("output_norm_gate: shape mismatch");
    DeviceTensor h = DeviceTensor::bf16(s);
    const tfla_dims cd{s[2], 1, 1, s[3], s[1], s[0]};
    check(tfla_output_norm_gate(&cd, h_tilde.data(), o_pre.data(), gamma.as<float>(), eps, h.data(), st));
    return h;
}

}  // namespace mlstm::b200
