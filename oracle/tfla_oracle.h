/* tfla_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C f64 restatement of the reference chunkwise mLSTM path
 * (/root/reference/proj/src/{gates,chunkwise}.cpp). It is the parity checker
 * for the CUDA kernels: tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may call it; the product path never does.
 *
 * Pinned against the reference itself: tests/test_oracle.py compares every
 * output with the reference library built from its own sources
 * (oracle/_ref/libmlstm_ref.so) and with the committed golden fixtures in
 * tests/golden/ that the reference produced (tests/golden/make_golden.py).
 *
 * Layouts are the reference Tensor layouts (row-major f64):
 *   q,k [B,H,T,dqk]  v,h,dh [B,H,T,dhv]  i_pre,f_pre [B,H,T]
 *   C [B,H,NC+1,dqk,dhv]  n [B,H,NC+1,dqk]  m [B,H,NC+1]  m_comb,h_denom [B,H,T]
 */
#ifndef TFLA_ORACLE_H_
#define TFLA_ORACLE_H_

#ifdef __cplusplus
extern "C" {
#endif

/* chunkwise_gates (gates.cpp:20-53): g [NC], b [NC*L], a [NC*L]. */
int or_chunkwise_gates(const double* f_pre, const double* i_pre, long T, long L, int variant,
                       double* g, double* b, double* a);

/* chunkwise_forward (chunkwise.cpp:270-302, heads via :80-181, states via :13-68). */
int or_forward(long B, long H, long T, long L, long dqk, long dhv, int variant, const double* q,
               const double* k, const double* v, const double* i_pre, const double* f_pre,
               double* h, double* C, double* n, double* m, double* m_comb, double* h_denom,
               int threads);

/* chunkwise_backward (chunkwise.cpp:396-566, state pass :196-237, assembly :239-266). */
int or_backward(long B, long H, long T, long L, long dqk, long dhv, int variant, const double* q,
                const double* k, const double* v, const double* i_pre, const double* f_pre,
                const double* dh, const double* C, const double* m, const double* m_comb,
                const double* h_denom, double* dq, double* dk, double* dv, double* d_fpre,
                double* d_ipre, int threads);
/* or_backward plus the split-entry-point partials (each nullable): d_b_q =
 * TfLaDqResult::d_b_cum, d_b_kv / d_a / d_i = TfLaDkResult::d_b_cum /
 * d_a_tail / d_i_log [B,H,T] (tiled.hpp:56-69); d_g [B,H,NC] and d_c
 * [B,H,NC+1,dqk,dhv] of backward_state_pass_head (chunkwise.cpp:196-237). */
int or_backward_parts(long B, long H, long T, long L, long dqk, long dhv, int variant,
                      const double* q, const double* k, const double* v, const double* i_pre,
                      const double* f_pre, const double* dh, const double* C, const double* m,
                      const double* m_comb, const double* h_denom, double* dq, double* dk,
                      double* dv, double* d_fpre, double* d_ipre, double* d_b_q, double* d_b_kv,
                      double* d_a, double* d_i, double* d_g, double* d_c, int threads);

/* run_recurrent (recurrent.cpp:65-115) with optional per-head initial state
 * (NULL = zero state): h [B,H,T,dhv], C_final [B,H,dqk,dhv], n_final [B,H,dqk],
 * m_final [B,H]. */
int or_recurrent(long B, long H, long T, long dqk, long dhv, int variant, const double* q,
                 const double* k, const double* v, const double* i_pre, const double* f_pre,
                 const double* C_init, const double* n_init, const double* m_init, double* h,
                 double* C_final, double* n_final, double* m_final);

/* Output epilogue (eq. 5): h = sigmoid(o_pre) * rms_norm(h_tilde; gamma[h], eps),
 * rms_norm as transfer.cpp:8-18, gamma [H][dhv]. */
int or_output_norm_gate(long B, long H, long T, long dhv, const double* h_tilde, const double* o_pre,
                        const double* gamma, double eps, double* h);

#ifdef __cplusplus
}
#endif

#endif
