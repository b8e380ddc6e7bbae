/* tfla.h -- C ABI of the B200-native TFLA mLSTM library (libtfla_b200.so).
 *
 * Drop-in boundary for the reference's chunkwise/TFLA hot path
 * (/root/reference/proj/include/mlstm/{chunkwise,tiled}.hpp). Every entry point
 * takes plain device pointers, is stream-ordered, never throws, and returns a
 * status code; the C++ exceptions of the reference map onto codes:
 *   mlstm::GeometryError  (core.hpp:11-13)  -> TFLA_ERR_GEOMETRY  (1)
 *   mlstm::ParameterError (core.hpp:16-18)  -> TFLA_ERR_PARAMETER (2)
 *   mlstm::NumericError   (core.hpp:21-23)  -> TFLA_ERR_NUMERIC   (3)
 * plus TFLA_ERR_CUDA (4) for launch / driver failures. tfla_last_error()
 * returns the message of the last failure on the calling thread.
 *
 * Data layout (row-major, last dim fastest, exactly the reference Tensor
 * layouts of SequenceInputs / ChunkStates / SavedStats / Gradients):
 *   q, k          bf16 [B, NH, T, d_qk]        (reference: f64, core.hpp:147-153)
 *   v, h, d_h     bf16 [B, NH, T, d_hv]
 *   i_pre, f_pre  fp32 [B, NH, T]
 *   c_states      fp32 [B, NH, NC+1, d_qk, d_hv]  (chunkwise.hpp:11-15; index 0 = zero state)
 *   n_states      fp32 [B, NH, NC+1, d_qk]
 *   m_states      fp32 [B, NH, NC+1]
 *   m_combine, h_denom fp32 [B, NH, T]           (chunkwise.hpp:20-23)
 *   saved_states  bf16 [B, NH, NC, d_qk, d_hv]   C_0..C_{NC-1}: the operand copy
 *                 of the inter-chunk states the backward pass consumes.
 *   dq, dk        bf16 [B, NH, T, d_qk]; dv bf16 [B, NH, T, d_hv];
 *   d_fpre, d_ipre fp32 [B, NH, T]              (chunkwise.hpp:32-35)
 * with NC = T / L. Arithmetic: bf16 tensor-core operands, fp32 accumulation,
 * fp32 gates / stabilisers / states.
 *
 * Geometry supported by the sm_100a kernels: L a multiple of 64 (64..1024),
 * d_qk and d_hv multiples of 64 (d_qk <= 512), T % L == 0. Everything the
 * reference accepts but these kernels cannot run returns TFLA_ERR_GEOMETRY
 * with a message naming the constraint -- there is no CPU fallback.
 */
#ifndef TFLA_TFLA_H_
#define TFLA_TFLA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    TFLA_OK = 0,
    TFLA_ERR_GEOMETRY = 1,
    TFLA_ERR_PARAMETER = 2,
    TFLA_ERR_NUMERIC = 3,
    TFLA_ERR_CUDA = 4
};

/* mlstm::Variant (core.hpp:113) */
enum { TFLA_VARIANT_EXP = 0, TFLA_VARIANT_SIG = 1 };

/* mlstm::Dims (core.hpp:27-39). */
typedef struct tfla_dims {
    int64_t T, L, d_qk, d_hv, n_head, n_batch;
} tfla_dims;

/* mlstm::BlockConfig (tiled.hpp:12-22). Validated with the reference rules
 * (tiled.cpp:21-30); on the GPU the sequence tiles are fixed at 128 x 128
 * (tcgen05 M = 128) and b_dhv selects the output column tile (64 or 128)
 * when it is one of those values, otherwise the kernels pick 128. */
typedef struct tfla_blocks {
    int64_t b_lhq, b_lkv, b_dqk, b_dhv;
} tfla_blocks;

/* mlstm::SequenceInputs (core.hpp:147-153), device pointers. All tensors are
 * dense row-major; the bf16 tensors (q, k, v, d_h, h, saved states, dq, dk,
 * dv), the fp32 C states and the workspace are moved by TMA / 16-byte vector
 * accesses and must be 16-byte aligned (TFLA_ERR_PARAMETER otherwise). */
typedef struct tfla_inputs {
    const void* q;      /* bf16 */
    const void* k;      /* bf16 */
    const void* v;      /* bf16 */
    const float* i_pre;
    const float* f_pre;
} tfla_inputs;

/* mlstm::ChunkwiseForward (chunkwise.hpp:25-29) plus the final states the
 * north star asks for. Required: h, m_states, m_combine, h_denom. Optional
 * (NULL = not written): c_states, n_states, c_final, n_final, m_final,
 * saved_states (when NULL the states live in the workspace and a later
 * backward must be given c_states instead). */
typedef struct tfla_fwd_out {
    void* h;
    float* c_states;
    float* n_states;
    float* m_states;
    float* m_combine;
    float* h_denom;
    float* c_final; /* [B, NH, d_qk, d_hv] */
    float* n_final; /* [B, NH, d_qk] */
    float* m_final; /* [B, NH] */
    void* saved_states;
} tfla_fwd_out;

/* Initial memory state for a forward that continues an earlier segment
 * (chunked prefill / stateful long context): the chunkwise analogue of
 * RecurrentOptions::initial_state (recurrent.hpp:23-27), which the reference
 * offers only on run_recurrent. c fp32 [B,NH,d_qk,d_hv], n fp32 [B,NH,d_qk],
 * m fp32 [B,NH] (n, m ignored for mLSTMsig) -- e.g. the c_final / n_final /
 * m_final of the previous segment's forward. */
typedef struct tfla_state_in {
    const float* c;
    const float* n;
    const float* m;
} tfla_state_in;

/* What chunkwise_backward consumes (chunkwise.hpp:52-54): dH, ChunkStates,
 * SavedStats. saved_states (bf16) is used when non-NULL, else c_states (fp32,
 * the reference ChunkStates.C) is converted on the device. */
typedef struct tfla_bwd_in {
    const void* d_h;
    const void* saved_states;
    const float* c_states;
    const float* m_states;
    const float* m_combine;
    const float* h_denom;
} tfla_bwd_in;

/* mlstm::Gradients (chunkwise.hpp:32-35). */
typedef struct tfla_grads {
    void* dq;
    void* dk;
    void* dv;
    float* d_fpre;
    float* d_ipre;
} tfla_grads;

/* Dims::validate_chunked (core.cpp:9-21) plus the kernel constraints above. */
int tfla_validate_dims(const tfla_dims* dims);
/* BlockConfig::validate (tiled.cpp:21-30). */
int tfla_validate_blocks(const tfla_dims* dims, const tfla_blocks* blocks);
/* BlockConfig::pick_default (tiled.cpp:32-39). */
int tfla_pick_default_blocks(const tfla_dims* dims, tfla_blocks* out);

/* detail::kv_block_count (tiled.cpp:43-45): number of kv blocks query block
 * i_lq visits in Alg. 1, ((i_lq + 1) * b_lhq) / b_lkv; -1 on bad arguments. */
int64_t tfla_kv_block_count(int64_t i_lq, const tfla_blocks* blocks);
/* detail::block_needs_mask (tiled.cpp:47-49): 1 when kv block i_kv_1based
 * (1-based, as in the reference loop) needs the causal mask for query block
 * i_lq (the literal, over-inclusive-by-one predicate), 0 if not, -1 on bad
 * arguments. */
int tfla_block_needs_mask(int64_t i_kv_1based, int64_t i_lq, const tfla_blocks* blocks);

/* Device workspace bytes for one forward (pass = 0) or backward (pass = 1). */
size_t tfla_workspace_bytes(const tfla_dims* dims, int variant, int pass);
/* Bytes of the bf16 saved_states buffer. */
size_t tfla_saved_state_bytes(const tfla_dims* dims);

/* chunkwise_forward (chunkwise.hpp:39-40 / chunkwise.cpp:270-302). */
int tfla_chunkwise_forward(const tfla_dims* dims, int variant, const tfla_inputs* in,
                           const tfla_fwd_out* out, void* workspace, size_t workspace_bytes,
                           void* stream);
/* tfla_forward (tiled.hpp:51-52 / tiled.cpp:258-298): same outputs, block
 * config validated like the reference. */
int tfla_forward(const tfla_dims* dims, const tfla_blocks* blocks, int variant,
                 const tfla_inputs* in, const tfla_fwd_out* out, void* workspace,
                 size_t workspace_bytes, void* stream);

/* chunkwise_forward_frozen (chunkwise.hpp:42-46 / chunkwise.cpp:304-394): the
 * forward with the max-state schedule (m_states [B,NH,NC+1]), m_combine and the
 * output denominator h_denom ([B,NH,T]) pinned to saved values -- the function
 * whose exact gradient tfla_chunkwise_backward computes (finite-difference
 * checks differentiate it, gradcheck.cpp:49-64). Writes h bf16 [B,NH,T,d_hv];
 * uses the forward workspace (tfla_workspace_bytes pass 0). mLSTMsig ignores
 * the values but, like the reference, requires the pointers. */
int tfla_chunkwise_forward_frozen(const tfla_dims* dims, int variant, const tfla_inputs* in,
                                  const float* m_states, const float* m_combine, const float* h_denom,
                                  void* h, void* workspace, size_t workspace_bytes, void* stream);

/* chunkwise_backward (chunkwise.hpp:52-54 / chunkwise.cpp:396-566): the exact
 * gradient of chunkwise_forward_frozen (normaliser and max states detached). */
int tfla_chunkwise_backward(const tfla_dims* dims, int variant, const tfla_inputs* in,
                            const tfla_bwd_in* saved, const tfla_grads* grads, void* workspace,
                            size_t workspace_bytes, void* stream);
/* tfla_backward (tiled.hpp:88-90 / tiled.cpp:781-811). */
int tfla_backward(const tfla_dims* dims, const tfla_blocks* blocks, int variant,
                  const tfla_inputs* in, const tfla_bwd_in* saved, const tfla_grads* grads,
                  void* workspace, size_t workspace_bytes, void* stream);

/* Split forward entry points (SURVEY §8(b) "optional split entry points").
 * tfla_state_recurrence: detail::state_recurrence_head (detail_kernels.hpp:
 *   38-44 / chunkwise.cpp:13-68) over every head -- gates, the max-state scan
 *   and the inter-chunk recurrence only. Reads in->k, v, i_pre, f_pre; writes
 *   out->m_states (required), c_states and/or saved_states (at least one),
 *   n_states, c_final, n_final, m_final (nullable); out->m_combine is written
 *   when non-NULL; out->h / h_denom are ignored.
 * tfla_forward_parallel: detail::tfla_forward_head (tiled.hpp:36-44 /
 *   tiled.cpp:59-240) over every head -- the intra-chunk part from the given
 *   states (saved_states bf16, else c_states fp32; n_states and m_states for
 *   mLSTMexp). Writes h, m_combine, h_denom. blocks must be non-NULL. */
typedef struct tfla_states_in {
    const void* saved_states; /* bf16 [B,NH,NC,d_qk,d_hv] C_0..C_{NC-1}, or NULL */
    const float* c_states;    /* fp32 [B,NH,NC+1,d_qk,d_hv] (used when saved_states is NULL) */
    const float* n_states;    /* fp32 [B,NH,NC+1,d_qk] (mLSTMexp) */
    const float* m_states;    /* fp32 [B,NH,NC+1] (mLSTMexp) */
} tfla_states_in;
int tfla_state_recurrence(const tfla_dims* dims, int variant, const tfla_inputs* in, const tfla_fwd_out* out,
                          void* workspace, size_t workspace_bytes, void* stream);
int tfla_forward_parallel(const tfla_dims* dims, const tfla_blocks* blocks, int variant, const tfla_inputs* in,
                          const tfla_states_in* states, void* h, float* m_combine, float* h_denom,
                          void* workspace, size_t workspace_bytes, void* stream);

/* Split backward entry points: each runs ONE gradient kernel of the split
 * (non-fused) path plus what it depends on, for callers that schedule the
 * gradients separately. Same saved-tensor inputs and errors as tfla_backward;
 * blocks must be non-NULL (validated like the reference).
 *   tfla_backward_dq  (tiled.hpp:56-59, 72-74 / tiled.cpp:391-529): dq and the
 *     query-side gate partial d_b_cum [B,H,T] fp32.
 *   tfla_backward_dk  (tiled.hpp:64-69, 76-79 / tiled.cpp:531-670): dk and the
 *     key-side partials d_a_tail, d_b_cum (= -column sums of the gate-matrix
 *     gradient), d_i_log (= +column sums), each [B,H,T] fp32.
 *   tfla_backward_dv  (tiled.hpp:81-84 / tiled.cpp:672-779): dv.
 * tfla_backward's gate gradients equal tfla_assemble_gate_grads over
 * d_g (tfla_backward_state_pass), dq.d_b_cum + dk.d_b_cum, dk.d_a_tail and
 * dk.d_i_log (tiled.cpp:795-808). */
int tfla_backward_dq(const tfla_dims* dims, const tfla_blocks* blocks, int variant,
                     const tfla_inputs* in, const tfla_bwd_in* saved, void* dq, float* d_b_cum,
                     void* workspace, size_t workspace_bytes, void* stream);
int tfla_backward_dk(const tfla_dims* dims, const tfla_blocks* blocks, int variant,
                     const tfla_inputs* in, const tfla_bwd_in* saved, void* dk, float* d_a_tail,
                     float* d_b_cum, float* d_i_log, void* workspace, size_t workspace_bytes,
                     void* stream);
int tfla_backward_dv(const tfla_dims* dims, const tfla_blocks* blocks, int variant,
                     const tfla_inputs* in, const tfla_bwd_in* saved, void* dv, void* workspace,
                     size_t workspace_bytes, void* stream);
/* backward_state_pass_head (chunkwise.hpp:70-76 / chunkwise.cpp:196-237) over
 * every head: d_c fp32 [B,H,NC+1,dqk,dhv] (nullable; entry NC is zero) and
 * d_g fp32 [B,H,NC] (the summed-forget-gate gradients, gbar applied). */
int tfla_backward_state_pass(const tfla_dims* dims, int variant, const tfla_inputs* in,
                             const tfla_bwd_in* saved, float* d_c, float* d_g, void* workspace,
                             size_t workspace_bytes, void* stream);
/* assemble_gate_grads_head (chunkwise.hpp:78-83 / chunkwise.cpp:239-266) over
 * every head: d_g [B,H,NC], d_b_total / d_a / d_i_extra [B,H,T] -> d_fpre,
 * d_ipre [B,H,T], all fp32 device pointers. No workspace. */
int tfla_assemble_gate_grads(const tfla_dims* dims, int variant, const float* f_pre, const float* i_pre,
                             const float* d_g, const float* d_b_total, const float* d_a,
                             const float* d_i_extra, float* d_fpre, float* d_ipre, void* stream);

/* Per-kernel CUDA-event profiling (tracing hook): when enabled, every kernel
 * launch site records an event pair on its stream. tfla_profile_read fills
 * ms[i] (summed device time) and launches[i] for kernel class i < n, then
 * resets; it returns the number of kernel classes. Names via
 * tfla_profile_name(i). */
int tfla_profile_enable(int on);
int tfla_profile_read(double* ms, int64_t* launches, int n);
const char* tfla_profile_name(int id);

/* Stabiliser audit -- the GPU counterpart of stab::exp_guarded / stab::checks /
 * stab::violations (core.hpp, core.cpp:145-166). When enabled (or when the
 * environment has TFLA_STAB_CHECK=1 at first use), every stabilised exponent
 * of the gate kernels and of the gating epilogues of the forward / backward
 * kernels (state recurrence gates, intra-chunk D, b_bar, a_bar, g_bar, the
 * decode step's gates) is noted before the kernels clamp it at 0: checks
 * counts them, violations counts arguments above 2^-10 in log2 units (fp32
 * rounding of an exactly-zero argument stays ~1e-5), max_arg is the largest
 * argument seen (natural-log units). tfla_stab_read synchronises the device,
 * returns the counts since the last read and resets them. Per device. */
int tfla_stab_enable(int on);
int tfla_stab_read(int64_t* checks, int64_t* violations, double* max_arg);

/* One training step with HOST buffers -- the reference-facing boundary
 * (chunkwise_forward + chunkwise_backward over host tensors, chunkwise.hpp:
 * 39-54): host_in (q, k, v bf16, i_pre, f_pre fp32) and d_h_host (bf16) are
 * read, h_host (bf16 h_tilde) and host_grads (dq, dk, dv bf16, d_fpre, d_ipre
 * fp32) are written; the saved forward tensors stay on the device. The batch
 * is streamed in batch-row slices through two device slots on three internal
 * streams (H2D | forward + backward | D2H overlap). The host inputs are read
 * from the time of the call on (they must be ready then); the device work and
 * the host outputs are ordered on `stream`: the outputs are complete when
 * `stream` reaches this point. Pinned host memory gives the PCIe rate;
 * pageable memory works but copies synchronously. */
int tfla_train_step_host(const tfla_dims* dims, int variant, const tfla_inputs* host_in, const void* d_h_host,
                         const tfla_grads* host_grads, void* h_host, void* stream);

/* chunkwise_gates (gates.hpp:21-35 / gates.cpp:20-59) over every head, f64
 * out: g_sum [B,NH,NC], b_cum [B,NH,T], a_tail [B,NH,T] (each nullable). */
int tfla_chunkwise_gates(const tfla_dims* dims, int variant, const float* f_pre, const float* i_pre,
                         double* g_sum, double* b_cum, double* a_tail, void* stream);

/* SequenceInputs::validate's finiteness check (core.cpp:106-117): returns
 * TFLA_ERR_NUMERIC when q, k, v, i_pre or f_pre holds a NaN / Inf. Opt-in
 * (a full read of the inputs); synchronises `stream`. */
int tfla_check_finite(const tfla_dims* dims, const tfla_inputs* in, void* stream);

/* Message of the last failure on this thread ("" if none). */
const char* tfla_last_error(void);

/* chunkwise_forward from an initial state (tfla_state_in; NULL = zero state,
 * identical to tfla_chunkwise_forward). m_states[0] / n_states[0] / c_states[0]
 * and saved_states[0] hold the initial state, so tfla_chunkwise_backward on
 * this forward's outputs differentiates the segment with the initial state
 * held constant (no gradient is returned for it). */
int tfla_chunkwise_forward_init(const tfla_dims* dims, int variant, const tfla_inputs* in,
                                const tfla_state_in* init, const tfla_fwd_out* out, void* workspace,
                                size_t workspace_bytes, void* stream);

/* Recurrent (decode) path: run_recurrent (recurrent.cpp:65-115) with the
 * memory state carried in place, i.e. RecurrentOptions::initial_state
 * (recurrent.hpp:23-27) in and {C,n,m}_final out. Folds step_exp / step_sig
 * (recurrent.cpp:9-63) over dims->T steps for every (batch, head); dims->L is
 * not used. Hands over from tfla_chunkwise_forward's c_final / n_final /
 * m_final (prefill) to token-by-token decode.
 *   in:    q, k bf16 [B,H,T,d_qk]; v bf16 [B,H,T,d_hv]; i_pre, f_pre fp32 [B,H,T]
 *   state: c_state fp32 [B,H,d_qk,d_hv], n_state fp32 [B,H,d_qk], m_state fp32
 *          [B,H]; read as the initial state and overwritten with the final one
 *          (n_state / m_state are ignored and may be NULL for mLSTMsig)
 *   h:     bf16 [B,H,T,d_hv] (pre-norm h_tilde)
 * d_qk in {64, 128, 256}, d_hv a multiple of 64. */
int tfla_recurrent_step(const tfla_dims* dims, int variant, const tfla_inputs* in, float* c_state,
                        float* n_state, float* m_state, void* h, void* stream);

/* apply_gate_softcap (gates.cpp:61-67): i_out = cap tanh(i_pre / cap) and
 * f_out = cap tanh(f_pre / cap) (softcap, gates.cpp:15-18), fp32 [B,H,T]
 * (in place allowed). cap <= 0 is a ParameterError (gates.cpp:16). The
 * reference applies it to the inputs before the forward (mlstm_cli.cpp:135);
 * gradients are then with respect to the capped pre-activations. */
int tfla_apply_gate_softcap(const tfla_dims* dims, const float* i_pre, const float* f_pre, double cap,
                            float* i_out, float* f_out, void* stream);

/* mLSTM cell output epilogue (eq. 5, :109-114): for every (b, h, t)
 * row of d_hv, h = sigmoid(o_pre) * rms_norm(h_tilde; gamma[h], eps) with
 * rms_norm as the reference's transfer.cpp:8-18 (mean over d_hv; rms == 0
 * gives 0). h_tilde, o_pre, h bf16 [B,H,T,d_hv]; gamma fp32 [H, d_hv];
 * eps >= 0 (ParameterError otherwise, transfer.cpp:9). dims->L is not used. */
int tfla_output_norm_gate(const tfla_dims* dims, const void* h_tilde, const void* o_pre, const float* gamma,
                          float eps, void* h, void* stream);

/* chunkwise_forward on fp32 operands (BASELINE config 0 as worded; the
 * reference's <float, float> instantiation, chunkwise.cpp:183-194): q, k, v
 * fp32 [B,NH,T,d] (no bf16 rounding), out->h fp32 [B,NH,T,d_hv], C / n states
 * fp32 in the reference layout (optional), m / m_combine / h_denom as
 * tfla_chunkwise_forward; saved_states is not written. CUDA-core kernel for
 * the reference-precision case: d_hv a multiple of 64, d_qk <= 256,
 * L * d_qk <= 8192 (GeometryError otherwise). Workspace as the forward's. */
int tfla_chunkwise_forward_f32(const tfla_dims* dims, int variant, const tfla_inputs* in, const tfla_fwd_out* out,
                               void* workspace, size_t workspace_bytes, void* stream);

/* chunkwise_forward with the cell output epilogue fused into the H store
 * (eq. 5, :109-114): everything tfla_chunkwise_forward writes, plus
 * y = sigmoid(o_pre) * rms_norm(h_tilde; gamma[h], eps) (transfer.cpp:8-18),
 * i.e. tfla_output_norm_gate(h_tilde = out->h) in the same call. o_pre, y
 * bf16 [B,H,T,d_hv]; gamma fp32 [H,d_hv]; eps >= 0. By default the forward is
 * followed by the tfla_output_norm_gate pass; with TFLA_FUSED_OUT=1 the fused
 * L = 128 forward (d_hv / 128 in {1, 2, 4}) forms y inside its H drain, the
 * x-tile CTAs of a head reducing each row's sum of squares over cluster
 * shared memory (parity-tested, measured slower: DESIGN.md section 9.3). */
int tfla_chunkwise_forward_gated(const tfla_dims* dims, int variant, const tfla_inputs* in,
                                 const tfla_fwd_out* out, const void* o_pre, const float* gamma, float eps,
                                 void* y, void* workspace, size_t workspace_bytes, void* stream);

/* Library / build identification string. */
const char* tfla_version(void);

/* Building-block self test (tcgen05 + TMA + TMEM): D[128,N] = A * B^T.
 * a_mode 0: A bf16 [128][K] K-major via TMA; 1: A given as [K][128] (MN-major
 * via TMA); 2: A [128][K] written by threads (K-major stationary); 3: X [K][128]
 * written by threads, A = X^T (MN-major stationary); 4: A [128][K] written by
 * threads into TMEM (tcgen05.mma A-from-TMEM form). b_mode 0: B [N][K];
 * 1: B given as [K][N]. out fp32 [128][N], out_bf16 bf16 [128][N]. */
int tfla_selftest_gemm(int a_mode, int b_mode, int N, int K, const void* a, const void* b,
                       float* out, void* out_bf16, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* TFLA_TFLA_H_ */
