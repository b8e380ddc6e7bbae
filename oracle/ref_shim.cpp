// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (checker, never the product path).
//
// extern "C" wrappers around the UNMODIFIED reference C++ library compiled
// from its own sources under /root/reference/proj/src (see oracle/Makefile,
// output oracle/_ref/libmlstm_ref.so). Used by tests/ to pin the C
// restatement (oracle/tfla_oracle.c) and to generate tests/golden fixtures,
// and by bench.py's cpu_baseline / --impl reference arm to time the
// reference's own CPU implementation on the host cores.
//
// All arrays are f64, row-major, exactly the reference Tensor layouts.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "mlstm/chunkwise.hpp"
#include "mlstm/core.hpp"
#include "mlstm/gates.hpp"
#include "mlstm/gradcheck.hpp"
#include "mlstm/parallel.hpp"
#ifdef REF_HAVE_PERFMODEL
#include "mlstm/perfmodel.hpp"
#endif
#include "mlstm/recurrent.hpp"
#include "mlstm/transfer.hpp"
#include "mlstm/tiled.hpp"

using namespace mlstm;

namespace {

thread_local std::string g_err;

Dims make_dims(long B, long H, long T, long L, long dqk, long dhv) {
    Dims d;
    d.n_batch = B;
    d.n_head = H;
    d.T = T;
    d.L = L;
    d.d_qk = dqk;
    d.d_hv = dhv;
    return d;
}

Tensor from(const double* p, std::vector<long> shape) {
    Tensor t(std::move(shape));
    std::memcpy(t.data(), p, sizeof(double) * static_cast<size_t>(t.numel()));
    return t;
}

void to(const Tensor& t, double* p) {
    if (p) std::memcpy(p, t.data(), sizeof(double) * static_cast<size_t>(t.numel()));
}

SequenceInputs inputs_from(const Dims& d, const double* q, const double* k, const double* v,
                           const double* ip, const double* fp) {
    SequenceInputs in;
    in.q = from(q, {d.n_batch, d.n_head, d.T, d.d_qk});
    in.k = from(k, {d.n_batch, d.n_head, d.T, d.d_qk});
    in.v = from(v, {d.n_batch, d.n_head, d.T, d.d_hv});
    in.i_pre = from(ip, {d.n_batch, d.n_head, d.T});
    in.f_pre = from(fp, {d.n_batch, d.n_head, d.T});
    return in;
}

int code_of(const std::exception& e) {
    if (dynamic_cast<const GeometryError*>(&e)) return 1;
    if (dynamic_cast<const ParameterError*>(&e)) return 2;
    if (dynamic_cast<const NumericError*>(&e)) return 3;
    return 5;
}

#define GUARD_BEGIN try {
#define GUARD_END                    \
    }                                \
    catch (const std::exception& e) { \
        g_err = e.what();            \
        return code_of(e);           \
    }                                \
    return 0;

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// make_inputs(dims, Rng(seed), scale, gate_scale) (core.cpp:127-143).
int ref_make_inputs(long B, long H, long T, long dqk, long dhv, uint64_t seed, double scale,
                    double gate_scale, double* q, double* k, double* v, double* ip, double* fp) {
    GUARD_BEGIN
    Dims d = make_dims(B, H, T, 1, dqk, dhv);
    Rng rng(seed);
    SequenceInputs in = make_inputs(d, rng, scale, gate_scale);
    to(in.q, q);
    to(in.k, k);
    to(in.v, v);
    to(in.i_pre, ip);
    to(in.f_pre, fp);
    GUARD_END
}

// Rng::fill_normal continuing a stream: n standard normals * scale.
int ref_normals(uint64_t seed, long skip, long n, double scale, double* out) {
    GUARD_BEGIN
    Rng rng(seed);
    for (long i = 0; i < skip; ++i) (void)rng.normal();
    for (long i = 0; i < n; ++i) out[i] = scale * rng.normal();
    GUARD_END
}

// chunkwise_gates (gates.cpp:20-53).
int ref_chunkwise_gates(const double* fp, const double* ip, long T, long L, int variant,
                        double* g, double* b, double* a) {
    GUARD_BEGIN
    ChunkwiseGates cg = chunkwise_gates(fp, ip, T, L, variant ? Variant::Sig : Variant::Exp);
    to(cg.g_sum, g);
    to(cg.b_cum, b);
    to(cg.a_tail, a);
    GUARD_END
}

// chunkwise_forward (chunkwise.cpp:270-302) or tfla_forward (tiled.cpp:258-298)
// when blocks != NULL ({b_lhq, b_lkv, b_dqk, b_dhv}).
int ref_forward(long B, long H, long T, long L, long dqk, long dhv, int variant,
                const long* blocks, const double* q, const double* k, const double* v,
                const double* ip, const double* fp, double* h, double* C, double* n, double* m,
                double* m_comb, double* h_denom) {
    GUARD_BEGIN
    Dims d = make_dims(B, H, T, L, dqk, dhv);
    SequenceInputs in = inputs_from(d, q, k, v, ip, fp);
    Variant var = variant ? Variant::Sig : Variant::Exp;
    ChunkwiseForward out;
    if (blocks) {
        BlockConfig bc{blocks[0], blocks[1], blocks[2], blocks[3]};
        out = tfla_forward(in, d, bc, var);
    } else {
        out = chunkwise_forward(in, d, var);
    }
    to(out.h_tilde, h);
    to(out.states.C, C);
    to(out.states.n, n);
    to(out.states.m, m);
    to(out.stats.m_combine, m_comb);
    to(out.stats.h_denom, h_denom);
    GUARD_END
}

// chunkwise_backward (chunkwise.cpp:396-566) or tfla_backward (tiled.cpp:781-811).
int ref_backward(long B, long H, long T, long L, long dqk, long dhv, int variant,
                 const long* blocks, const double* q, const double* k, const double* v,
                 const double* ip, const double* fp, const double* dh, const double* C,
                 const double* n, const double* m, const double* m_comb, const double* h_denom,
                 double* dq, double* dk, double* dv, double* dfp, double* dip) {
    GUARD_BEGIN
    Dims d = make_dims(B, H, T, L, dqk, dhv);
    SequenceInputs in = inputs_from(d, q, k, v, ip, fp);
    Variant var = variant ? Variant::Sig : Variant::Exp;
    const long NC = T / L;
    ChunkStates st;
    st.C = from(C, {B, H, NC + 1, dqk, dhv});
    st.n = from(n, {B, H, NC + 1, dqk});
    st.m = from(m, {B, H, NC + 1});
    SavedStats ss;
    ss.m_combine = from(m_comb, {B, H, T});
    ss.h_denom = from(h_denom, {B, H, T});
    Tensor dH = from(dh, {B, H, T, dhv});
    Gradients g;
    if (blocks) {
        BlockConfig bc{blocks[0], blocks[1], blocks[2], blocks[3]};
        g = tfla_backward(in, d, bc, var, dH, st, ss);
    } else {
        g = chunkwise_backward(in, d, var, dH, st, ss);
    }
    to(g.dq, dq);
    to(g.dk, dk);
    to(g.dv, dv);
    to(g.d_fpre, dfp);
    to(g.d_ipre, dip);
    GUARD_END
}

// The split entry points tfla_backward_dq / _dk / _dv (tiled.cpp:391-779) and
// detail::backward_state_pass_head per head (chunkwise.cpp:196-237).
int ref_backward_split(long B, long H, long T, long L, long dqk, long dhv, int variant,
                       const long* blocks, const double* q, const double* k, const double* v,
                       const double* ip, const double* fp, const double* dh, const double* C,
                       const double* n, const double* m, const double* m_comb,
                       const double* h_denom, double* dq, double* d_b_q, double* dk,
                       double* d_a_tail, double* d_b_kv, double* d_i_log, double* dv, double* d_g,
                       double* d_c) {
    GUARD_BEGIN
    Dims d = make_dims(B, H, T, L, dqk, dhv);
    SequenceInputs in = inputs_from(d, q, k, v, ip, fp);
    Variant var = variant ? Variant::Sig : Variant::Exp;
    const long NC = T / L;
    ChunkStates st;
    st.C = from(C, {B, H, NC + 1, dqk, dhv});
    st.n = from(n, {B, H, NC + 1, dqk});
    st.m = from(m, {B, H, NC + 1});
    SavedStats ss;
    ss.m_combine = from(m_comb, {B, H, T});
    ss.h_denom = from(h_denom, {B, H, T});
    Tensor dH = from(dh, {B, H, T, dhv});
    BlockConfig bc{blocks[0], blocks[1], blocks[2], blocks[3]};
    TfLaDqResult rq = tfla_backward_dq(in, d, bc, var, dH, st, ss);
    TfLaDkResult rk = tfla_backward_dk(in, d, bc, var, dH, st, ss);
    Tensor rv = tfla_backward_dv(in, d, bc, var, dH, st, ss);
    to(rq.dq, dq);
    to(rq.d_b_cum, d_b_q);
    to(rk.dk, dk);
    to(rk.d_a_tail, d_a_tail);
    to(rk.d_b_cum, d_b_kv);
    to(rk.d_i_log, d_i_log);
    to(rv, dv);
    const long SZ = dqk * dhv;
    std::vector<double> dht(static_cast<size_t>(T * dhv));
    for (long s = 0; s < B * H; ++s) {
        const double* fps = fp + s * T;
        const double* ips = ip + s * T;
        ChunkwiseGates gt = chunkwise_gates(fps, ips, T, L, var);
        for (long t = 0; t < T; ++t)
            for (long x = 0; x < dhv; ++x)
                dht[static_cast<size_t>(t * dhv + x)] =
                    dh[(s * T + t) * dhv + x] / (variant ? 1.0 : h_denom[s * T + t]);
        detail::backward_state_pass_head(q + s * T * dqk, nullptr, d, gt, C + s * (NC + 1) * SZ,
                                         m + s * (NC + 1), m_comb + s * T, dht.data(),
                                         d_c + s * (NC + 1) * SZ, d_g + s * NC, var);
    }
    GUARD_END
}

#ifdef REF_HAVE_PERFMODEL
// The cost model (perfmodel.cpp) at one point: out[42] in the order of
// oracle.Reference.perfmodel. params = {f_causal, f_exp, f_log, f_sig, f_max,
// f_abs, f_mask, bytes_qkv, bytes_if, bytes_cmn}.
int ref_perfmodel_eval(int variant, long B, long H, long T, long L, long dqk, long dhv, const double* params,
                       double flops_per_s, double bytes_per_s, double* out) {
    GUARD_BEGIN
    Dims d = make_dims(B, H, T, L, dqk, dhv);
    const Variant var = variant ? Variant::Sig : Variant::Exp;
    PerfParams p;
    p.f_causal = params[0];
    p.f_exp = params[1];
    p.f_log = params[2];
    p.f_sig = params[3];
    p.f_max = params[4];
    p.f_abs = params[5];
    p.f_mask = params[6];
    p.bytes_qkv = params[7];
    p.bytes_if = params[8];
    p.bytes_cmn = params[9];
    AcceleratorSpec acc{"probe", flops_per_s, bytes_per_s};
    int o = 0;
    for (CountMode mode : {CountMode::Exact, CountMode::Simplified})
        for (const auto& it : flops_chunkwise(d, p, var, mode).items) out[o++] = it.second;
    for (const auto& it : flops_parallel(d, p, var, CountMode::Exact).items) out[o++] = it.second;
    for (const auto& it : flops_recurrent(d, p, var, CountMode::Exact).items) out[o++] = it.second;
    for (Formulation f : {Formulation::Chunkwise, Formulation::Parallel, Formulation::Recurrent}) {
        const MemopCounts m = memops(d, p, var, f);
        out[o++] = m.loaded;
        out[o++] = m.stored;
    }
    const double pqk = static_cast<double>(dqk) / static_cast<double>(dhv);
    out[o++] = chunkwise_flops_model(var, T, L, dqk, dhv, p.f_causal);
    out[o++] = chunkwise_bytes_model(var, T, L, dqk, dhv, p);
    out[o++] = flop_optimal_chunk_size(dhv, pqk, p.f_causal);
    out[o++] = runtime_optimal_chunk_size(dhv, pqk, p.f_causal, p.bytes_cmn, accelerator_intensity(acc));
    out[o++] = theoretical_runtime(d, p, var, acc, static_cast<double>(L), RuntimeBound::Sum);
    out[o++] = theoretical_runtime(d, p, var, acc, static_cast<double>(L), RuntimeBound::Max);
    out[o++] = arithmetic_intensity(d, p, static_cast<double>(L));
    out[o++] = accelerator_intensity(acc);
    out[o++] = roofline(acc, out[o - 2]);
    const std::vector<long> cands = chunk_size_candidates(16, 1024, T);
    out[o++] = static_cast<double>(flop_argmin_chunk_size(dhv, pqk, p.f_causal, cands));
    out[o++] = static_cast<double>(runtime_argmin_chunk_size(dhv, pqk, p.f_causal, p.bytes_cmn, acc, cands));
    GUARD_END
}
#endif

// run_recurrent (recurrent.cpp:65-115): h, C_final, n_final, m_final.
int ref_run_recurrent(long B, long H, long T, long dqk, long dhv, int variant, const double* q,
                      const double* k, const double* v, const double* ip, const double* fp,
                      double* h, double* C_final, double* n_final, double* m_final) {
    GUARD_BEGIN
    Dims d = make_dims(B, H, T, 1, dqk, dhv);
    SequenceInputs in = inputs_from(d, q, k, v, ip, fp);
    RecurrentTrace tr = run_recurrent(in, d, variant ? Variant::Sig : Variant::Exp);
    to(tr.h_tilde, h);
    to(tr.C_final, C_final);
    to(tr.n_final, n_final);
    to(tr.m_final, m_final);
    GUARD_END
}

// rms_norm (transfer.cpp:8-18) over rows of length d.
int ref_rms_norm(long rows, long d, const double* x, const double* gamma, double eps, double* y) {
    GUARD_BEGIN
    for (long r = 0; r < rows; ++r) rms_norm(x + r * d, gamma, d, eps, y + r * d);
    GUARD_END
}

// parallel_forward_exp / parallel_forward_sig (parallel.cpp).
int ref_parallel_forward(long B, long H, long T, long dqk, long dhv, int variant,
                         const double* q, const double* k, const double* v, const double* ip,
                         const double* fp, double* h) {
    GUARD_BEGIN
    Dims d = make_dims(B, H, T, 1, dqk, dhv);
    SequenceInputs in = inputs_from(d, q, k, v, ip, fp);
    Tensor out = variant ? parallel_forward_sig(in, d) : parallel_forward_exp(in, d);
    to(out, h);
    GUARD_END
}

// gradcheck_chunkwise / gradcheck_tiled (gradcheck.cpp:84-101); report[5] =
// {dq, dk, dv, d_fpre, d_ipre} relative errors.
int ref_gradcheck(long T, long L, long dqk, long dhv, int variant, const long* blocks,
                  const double* q, const double* k, const double* v, const double* ip,
                  const double* fp, const double* w, double step, double* report) {
    GUARD_BEGIN
    Dims d = make_dims(1, 1, T, L, dqk, dhv);
    SequenceInputs in = inputs_from(d, q, k, v, ip, fp);
    Tensor wt = from(w, {1, 1, T, dhv});
    Variant var = variant ? Variant::Sig : Variant::Exp;
    GradcheckReport r =
        blocks ? gradcheck_tiled(in, d, BlockConfig{blocks[0], blocks[1], blocks[2], blocks[3]},
                                 var, wt, step)
               : gradcheck_chunkwise(in, d, var, wt, step);
    report[0] = r.dq;
    report[1] = r.dk;
    report[2] = r.dv;
    report[3] = r.d_fpre;
    report[4] = r.d_ipre;
    GUARD_END
}

long long ref_stab_checks() { return stab::checks(); }
long long ref_stab_violations() { return stab::violations(); }
void ref_stab_reset() { stab::reset(); }

// CPU baseline timing: `n_slices` independent (b,h) slices of shape
// (T, L, dqk, dhv), inputs from make_inputs(Rng(seed + slice), 1, 1) and dH ~
// N(0,1), each running the public f64 API forward + backward
// (chunkwise_* when tiled == 0, else tfla_* with pick_default blocks), fanned
// over `threads` std::threads. Returns wall seconds (forward-only and total)
// of the timed region (inputs are generated before it).
int ref_time_slices(long T, long L, long dqk, long dhv, int variant, int tiled, long n_slices,
                    int threads, int with_backward, uint64_t seed, double* fwd_seconds,
                    double* total_seconds) {
    GUARD_BEGIN
    Dims d = make_dims(1, 1, T, L, dqk, dhv);
    Variant var = variant ? Variant::Sig : Variant::Exp;
    std::vector<SequenceInputs> ins(static_cast<size_t>(n_slices));
    std::vector<Tensor> dhs(static_cast<size_t>(n_slices));
    for (long s = 0; s < n_slices; ++s) {
        Rng rng(seed + static_cast<uint64_t>(s));
        ins[static_cast<size_t>(s)] = make_inputs(d, rng, 1.0, 1.0);
        dhs[static_cast<size_t>(s)] = Tensor({1, 1, T, dhv});
        rng.fill_normal(dhs[static_cast<size_t>(s)], 1.0);
    }
    BlockConfig bc = BlockConfig::pick_default(d);
    std::vector<double> fwd_t(static_cast<size_t>(n_slices), 0.0);
    std::vector<std::thread> pool;
    const auto t0 = std::chrono::steady_clock::now();
    const int nt = std::max(1, std::min<int>(threads, static_cast<int>(n_slices)));
    for (int w = 0; w < nt; ++w) {
        pool.emplace_back([&, w] {
            for (long s = w; s < n_slices; s += nt) {
                const auto a = std::chrono::steady_clock::now();
                ChunkwiseForward f = tiled ? tfla_forward(ins[static_cast<size_t>(s)], d, bc, var)
                                           : chunkwise_forward(ins[static_cast<size_t>(s)], d, var);
                const auto b = std::chrono::steady_clock::now();
                fwd_t[static_cast<size_t>(s)] = std::chrono::duration<double>(b - a).count();
                if (with_backward) {
                    Gradients g = tiled ? tfla_backward(ins[static_cast<size_t>(s)], d, bc, var,
                                                        dhs[static_cast<size_t>(s)], f.states,
                                                        f.stats)
                                        : chunkwise_backward(ins[static_cast<size_t>(s)], d, var,
                                                             dhs[static_cast<size_t>(s)], f.states,
                                                             f.stats);
                    (void)g;
                }
            }
        });
    }
    for (auto& t : pool) t.join();
    const auto t1 = std::chrono::steady_clock::now();
    *total_seconds = std::chrono::duration<double>(t1 - t0).count();
    // forward share of the wall time: per-thread sums, max over threads
    double fmax = 0.0;
    for (int w = 0; w < nt; ++w) {
        double acc = 0.0;
        for (long s = w; s < n_slices; s += nt) acc += fwd_t[static_cast<size_t>(s)];
        fmax = std::max(fmax, acc);
    }
    *fwd_seconds = fmax;
    GUARD_END
}

}  // extern "C"
