// bwd_parallel.h -- K4 (dQ / dK / dV) and K7 (gate-gradient assembly) launch interfaces.
#pragma once
#include "kernels.h"

namespace tfla_k {

enum BwdKind { kDQ = 0, kDK = 1, kDV = 2 };

struct BwdArgs {
    Geom g;
    int ntile;    // dV column tile (64 / 128); dQ / dK always use 128-wide d_qk tiles
    int variant;
    GateWS gw;    // b, ib, mc, ab, bb (= b_bar / (den sqrt d)), dinv
    const __nv_bfloat16* q;  // [BH][T][dqk]  (CUDA-core reads in the epilogue)
    const __nv_bfloat16* k;
    float* dbq_part;  // [n_ptile][BH][T]  dQ: row gate partials
    float* da_part;   // [n_ptile][BH][T]  dK: d a_bar partials
    float* colsum;    // [BH][T]           dK: column sums of dD
    float* iq_part;   // [BH][T]           fused: w q.(C_k dh) alone (d_g identity), nullable
    __nv_bfloat16 *dq, *dk, *dv;  // outputs (direct stores in the fused kernel)
    long long* trace;             // debug: per-stage clock64 events of CTA 0 (nullable)
    int l2mode;                   // fused backward: last-use L2 evict-first bits (TFLA_BWDF_L2)
};

struct BwdTensors {
    const void *q, *k, *v, *dh;
    const void* states;   // bf16 [BH][NC][dqk][dhv]: C_k (dQ) or dC_{k+1} (dK, dV)
    void* out;            // dq / dk / dv
};

int launch_bwd_parallel(BwdKind kind, const BwdArgs& a, const BwdTensors& t, cudaStream_t st);
// Wide (256-column) split kernels for L >= 128: dQ / dK when d_qk == 256, dV
// when d_hv % 256 == 0 (TFLA_NO_WIDE_BWD=1 forces the 128-column kernels).
bool bwd_wide_qk(const Geom& g);
bool bwd_wide_v(const Geom& g);
// p tiles of the dQ / dK gate partials (dbq_part / da_part slices).
int bwd_n_ptile(const Geom& g);
// CTA-pair (cta_group::2, M = 256) form of the wide kernels for L >= 256
// (bwd_pair.cu): d_qk == 256, d_hv % 256 == 0; opt-in (TFLA_PAIR_BWD=1).
bool bwd_pair_supported(const Geom& g);
int launch_bwd_pair(BwdKind kind, const BwdArgs& a, const BwdTensors& t, cudaStream_t st);

// Fused dQ/dK/dV for L = 128 (bwd_fused.cu): one CTA per chunk, shared score tiles.
// Writes gate partials with n_ptile = 1.
bool bwd_fused_supported(const Geom& g);
int launch_bwd_fused(const BwdArgs& a, const BwdTensors& t, void* dq, void* dk, void* dv,
                     const void* c_states, const void* dc_states, cudaStream_t st);

// 256-column-group variant of the fused backward (bwd_fused_wide.cu): L = 128,
// d_qk == 256, d_hv % 256 == 0; opt-in (TFLA_WIDE_FUSED_BWD=1, measured slower).
bool bwd_fused_wide_supported(const Geom& g);
int launch_bwd_fused_wide(const BwdArgs& a, const BwdTensors& t, void* dq, void* dk, void* dv,
                          const void* c_states, const void* dc_states, cudaStream_t st);

struct AssembleArgs {
    Geom g;
    int variant;
    int n_ptile, n_tiles;     // p tiles; tiles per chunk in dg_part
    const float* f_pre;
    const float* i_pre;
    const float* gbar;        // [BH][NC]
    const float* dg_part;     // [BH][NC][n_tiles]
    const float* dbq_part;    // [n_ptile][BH][T]
    const float* da_part;     // [n_ptile][BH][T]
    const float* colsum;      // [BH][T]; nullptr: d_b / d_a / d_i_extra given directly
    const float* di_extra;    // [BH][T] d_i_extra when colsum == nullptr
    float* d_fpre;
    float* d_ipre;
};
void launch_assemble(const AssembleArgs& a, cudaStream_t st);

// Split-entry-point partials (tiled.hpp:56-79) from the kernels' scratch:
//   kind kDQ: out0 = sum_p dbq_part                      (TfLaDqResult::d_b_cum)
//   kind kDK: out0 = sum_p da_part, out1 = -colsum, out2 = colsum
//             (TfLaDkResult::d_a_tail / d_b_cum / d_i_log)
void launch_split_partials(BwdKind kind, const Geom& g, int n_ptile, const float* dbq_part,
                           const float* da_part, const float* colsum, float* out0, float* out1,
                           float* out2, cudaStream_t st);
// d_g from per-token partials, without reading the states: with
// U_k = (a_bar o K_k)^T V_k and W_k = (w o Q_k)^T dH_k, the two recurrences
// C_{k+1} = gbar_k C_k + U_k and dC_k = gbar_k dC_{k+1} + W_k give
//   <C_{k+1}, dC_{k+1}> = d_g[k] + <U_k, dC_{k+1}> = d_g[k+1] + <C_{k+1}, W_{k+1}>
// so d_g[k] = d_g[k+1] + I_{k+1} - A_k, d_g[NC-1] = 0 (dC_NC = 0), where
// I_j = sum_{t in j} iq[t] (= w q.(C_j dh)) and A_k = sum_{t in k} da[t].
void launch_dg_from_partials(const Geom& g, const float* iq, const float* da, float* d_g, cudaStream_t st);
// d_g [BH][NC] = gbar * sum of the state-pass partials (chunkwise.cpp:216-221).
void launch_dg_reduce(const Geom& g, int n_tiles, const float* dg_part, const float* gbar, float* d_g,
                      cudaStream_t st);

// fp32 reference-layout states [BH][NC+1][dqk][dhv] -> bf16 [BH][NC][dqk][dhv].
void launch_states_to_bf16(const float* c_states, __nv_bfloat16* out, const Geom& g,
                           cudaStream_t st);

}  // namespace tfla_k
