// fwd_parallel.h -- K2 launch interface.
#pragma once
#include "kernels.h"

namespace tfla_k {

struct FwdArgs {
    Geom g;
    int ntile;    // output column tile (64 / 128)
    int variant;  // 0 exp, 1 sig
    GateWS gw;    // b, ib, mc, bb used
    const __nv_bfloat16* q;   // [BH][T][dqk] (also read on CUDA cores for q.n)
    const float* n_states;    // [BH][NC+1][dqk] (exp)
    const float* qn;          // [BH][T] q_t . n_{c(t)} (exp, from launch_qn)
    float* h_denom;           // [BH][T] (nullable)
    const float* den_fixed;   // [BH][T] frozen denominators (chunkwise_forward_frozen), nullable
};

// qn[t] = q_t . n_{c(t)} for the exp normaliser (one small pass over q).
void launch_qn(const Geom& g, const __nv_bfloat16* q, const float* n_states, float* qn, cudaStream_t st);

// q (via args), k: bf16 [BH][T][dqk]; v, h: bf16 [BH][T][dhv];
// states: bf16 [BH][NC][dqk][dhv] (C_0 .. C_{NC-1}).
int launch_fwd_parallel(const FwdArgs& a, const void* k, const void* v, const void* states,
                        void* h, cudaStream_t st);

}  // namespace tfla_k
