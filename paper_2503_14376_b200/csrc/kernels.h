// kernels.h -- launch interfaces of the TFLA device kernels (host side).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cuda_bf16.h>

namespace tfla_k {

// Per-position / per-chunk gate vectors shared by every kernel (workspace).
//   b   [BH][T]  inclusive in-chunk cumsum of logsigmoid(f)      (gates.cpp:37-42)
//   ib  [BH][T]  i_bar = i (exp) / logsigmoid(i) (sig)           (detail_kernels.hpp:32-34)
//   mc  [BH][T]  combined stabiliser m_c (exp) / 0 (sig)          (chunkwise.cpp:125-135)
//   ab  [BH][T]  a_bar = exp(a - m_{k+1})                         (chunkwise.cpp:41-43)
//   bb  [BH][T]  fwd: b_bar = exp(b + m_k - m_c); bwd: b_bar / (h_denom * sqrt(d_qk))
//   dinv[BH][T]  bwd only: 1 / h_denom
//   gbar[BH][NC] g_bar = exp(g + m_k - m_{k+1})                   (chunkwise.cpp:37-40)
//   gsum, amax [BH][NC] (f64) per-chunk g and max_j a (scan inputs)
// Stabiliser audit counters (stab.cuh; device memory, enabled by
// tfla_stab_enable / TFLA_STAB_CHECK=1): exp arguments checked, arguments
// above tolerance, and the largest positive argument (fp32 bits, log2 units).
struct StabCounters {
    unsigned long long checks, violations;
    unsigned int max_bits, pad;
};

struct GateWS {
    float *b, *ib, *mc, *ab, *bb, *dinv, *gbar;
    double *gsum, *amax;
    double* gtmp;        // [4][BH][T] f64 b, a, ib, m_intra from the chunk pass (nullable)
    StabCounters* stab;  // nullptr unless the audit is on
};

struct Geom {
    int BH, T, L, NC, dqk, dhv;
};

// K0 forward: gates + max-state scan. Writes m_states [BH][NC+1], m_comb [BH][T]
// (may be nullptr), m_final [BH] (nullable). m_init [BH] (nullable) is the
// initial max state m_0 (0 when absent, chunkwise.cpp:23).
void launch_gates_fwd(const Geom& g, int variant, const float* f_pre, const float* i_pre,
                      const GateWS& ws, float* m_states, float* m_comb, float* m_final,
                      cudaStream_t st, const float* m_init = nullptr);
// K0 forward from given max states m_states [BH][NC+1] (tfla_forward_head's
// input, tiled.hpp:40-44): gate vectors and m_comb only.
// mc_given (nullable): also pin m_comb (chunkwise_forward_frozen, chunkwise.cpp:304-394).
void launch_gates_fwd_given_m(const Geom& g, int variant, const float* f_pre, const float* i_pre,
                              const GateWS& ws, const float* m_states, float* m_comb, cudaStream_t st,
                              const float* mc_given = nullptr);
// chunkwise_gates (gates.hpp:31-35) in f64: g_sum [BH][NC], b_cum / a_tail [BH][T] (each nullable).
void launch_gates_export(const Geom& g, int variant, const float* f_pre, const float* i_pre, double* g_sum,
                         double* b_cum, double* a_tail, cudaStream_t st);
// K0 backward: gates from saved m_states / m_comb / h_denom.
void launch_gates_bwd(const Geom& g, int variant, const float* f_pre, const float* i_pre,
                      const float* m_states, const float* m_comb, const float* h_denom,
                      const GateWS& ws, cudaStream_t st);

// K1 / K3: inter-chunk state recurrence on tcgen05.
//   fwd: C_{k+1} = gbar_k C_k + (a_bar o K_k)^T V_k ;   writes C_0..C_{NC-1} (bf16)
//   bwd: dC_k = gbar_k dC_{k+1} + (w o Q_k)^T dH_k ;   writes dC_1..dC_NC (bf16)
struct ScanArgs {
    Geom g;
    int ntile;          // output column tile N (64 or 128)
    const float* w;     // [BH][T] row weights (a_bar fwd / b_bar/(den sqrt d) bwd)
    const float* gbar;  // [BH][NC]
    // fwd extras (nullable)
    float* c_states;    // fp32 [BH][NC+1][dqk][dhv]
    float* c_final;     // fp32 [BH][dqk][dhv]
    float* u_part;      // fp32 [BH][NC][n_xtiles][dqk] n increments (exp fwd, nullable)
    const float* c_init;  // fp32 [BH][dqk][dhv] initial state C_0 (fwd, nullable = 0)
    // bwd extras
    const __nv_bfloat16* c_saved;  // bf16 [BH][NC][dqk][dhv] (for d_g)
    float* dg_part;                // [BH][NC][n_ptile*n_xtile]
    float* dc_states;              // fp32 [BH][NC+1][dqk][dhv] dC_0..dC_NC (nullable,
                                   // backward_state_pass_head's d_c, chunkwise.cpp:196-237)
    long long* trace;              // debug: clock64 events of CTA (0,0,0) (nullable; state_scan.cu)
};
// a_src: bf16 [BH][T][dqk] (k fwd / q bwd); b_src: bf16 [BH][T][dhv] (v fwd / dh bwd);
// states_out: bf16 [BH][NC][dqk][dhv].
// n states from K1's per-x-tile increments (exp forward).
void launch_nscan(const Geom& g, const float* u_part, const float* gbar, float* n_states, float* n_final,
                  int n_xtiles, cudaStream_t st, const float* n_init = nullptr);

// Recurrent (decode) path, recurrent.cu.
struct RecurrentArgs {
    int T, dhv, variant;
    const __nv_bfloat16 *q, *k, *v;   // [BH][T][dqk|dhv]
    const float *i_pre, *f_pre;       // [BH][T]
    float* c_state;                   // [BH][dqk][dhv] in / out
    float* n_state;                   // [BH][dqk] out (exp, nullable)
    float* m_state;                   // [BH] out (exp, nullable)
    const float* n_in;                // [BH][dqk] initial n: a copy of n_state taken before the launch
    const float* m_in;                // [BH] initial m: a copy of m_state taken before the launch
    StabCounters* stab;               // stabiliser audit (nullable)
    __nv_bfloat16* h;                 // [BH][T][dhv]
};
bool recurrent_supported(int dqk, int dhv);
// the column slices of a head form one cluster (dhv / 64 <= 8): no n / m copy needed
bool recurrent_cluster(int dhv);

// Finiteness check (core.cpp:114-116): sets *flag (device) to 1 if the buffer of
// `bytes` bf16 / fp32 elements holds a NaN or Inf. 16-byte aligned buffers.
void launch_nonfinite(const void* p, size_t bytes, bool is_bf16, unsigned* flag, int n_sm, cudaStream_t st);

// apply_gate_softcap (gates.cpp:61-67): io/fo = cap * tanh(ip/fp / cap) (in place allowed).
void launch_gate_softcap(const float* ip, const float* fp, float* io, float* fo, long n, double cap,
                         cudaStream_t st);

// fp32-operand chunkwise forward on CUDA cores (fwd_f32.cu; the reference's
// <float, float> chunkwise_forward_head, chunkwise.cpp:80-194): fp32 q / k / v
// [BH][T][d], h fp32; C / n states fp32 reference layout (nullable).
struct F32FwdArgs {
    Geom g;
    int variant;
    GateWS gw;
    const float *q, *k, *v;
    float* h;
    float* h_denom;
    float *c_states, *n_states, *c_final, *n_final;
};
bool fwd_f32_supported(const Geom& g);
size_t fwd_f32_smem_bytes(const Geom& g);
int launch_fwd_f32(const F32FwdArgs& a, cudaStream_t st);

// Output epilogue (output.cu): h = sigmoid(o_pre) * rms_norm(h_tilde; gamma[head], eps).
bool output_supported(int dhv);
void launch_output_norm_gate(const __nv_bfloat16* ht, const __nv_bfloat16* op, const float* gamma, float eps,
                             __nv_bfloat16* h, long rows, int T, int NH, int dhv, cudaStream_t st);
void launch_recurrent(const RecurrentArgs& a, int BH, int dqk, cudaStream_t st);

// K1 / K3 column tile: 64, or 32 (opt-in TFLA_SCAN32=1) when the 64-column
// grid has at most one CTA per SM (twice the chains, two per SM).
int scan_ntile_for(const Geom& g);
int launch_state_scan(bool bwd, const void* a_src, const void* b_src, void* states_out,
                      const ScanArgs& a, cudaStream_t st);
// K1 / K3 with the state resident in TMEM (state_scan2.cu): 256-column x
// halves, 128-row p tiles, two CTAs per SM. d_qk % 128 == 0, d_hv % 256 == 0,
// L % 32 == 0 (TFLA_NO_SCAN2=1 forces state_scan.cu). Its n increments come
// as ONE partial per chunk (u_part [BH][NC][1][dqk]) and its d_g partials as
// (d_qk/128)*(d_hv/256) tiles per chunk; a.ntile is ignored.
bool scan2_supported(const Geom& g);
bool scan2_use(const Geom& g, bool bwd);  // the measured policy (state_scan2.cu)
int launch_state_scan2(bool bwd, const void* a_src, const void* b_src, void* states_out,
                       const ScanArgs& a, cudaStream_t st);

}  // namespace tfla_k
