// fwd_fused.h -- K12 launch interface (fused recurrent + parallel forward, L = 128).
#pragma once
#include "kernels.h"

namespace tfla_k {

struct FusedFwdArgs {
    Geom g;
    int variant;          // 0 exp, 1 sig
    GateWS gw;            // b, ib, mc, ab, bb, gbar (from K0)
    __nv_bfloat16* h;     // [BH][T][dhv]
    float* h_denom;       // [BH][T]
    float* n_states;      // fp32 [BH][NC+1][dqk] (exp, nullable)
    float* n_final;       // fp32 [BH][dqk] (exp, nullable)
    float* c_states;      // fp32 [BH][NC+1][dqk][dhv] reference layout (nullable)
    float* c_final;       // fp32 [BH][dqk][dhv] (nullable)
    const float* c_init;  // fp32 [BH][dqk][dhv] initial state C_0 (nullable = zero state)
    const float* n_init;  // fp32 [BH][dqk] initial n_0 (exp, nullable)
    long long* trace;     // debug: per-chunk clock64 events of CTA `trace_cta` (nullable)
    int trace_cta;
    int cluster;          // CTAs (x tiles of one head) sharing the Q/K stages by TMA multicast (set by launch)
    // Fused output epilogue (eq. 5; rms_norm as transfer.cpp:8-18):
    // y = sigmoid(o_pre) * h_tilde / sqrt(mean(h_tilde^2) + eps) * gamma[head],
    // the row's sum of squares reduced over the x-tile CTAs of the head (a
    // cluster, DSMEM). Off when o_pre is null.
    const __nv_bfloat16* o_pre;  // [BH][T][dhv]
    const float* gamma;          // [NH][dhv]
    __nv_bfloat16* y;            // [BH][T][dhv]
    float eps;
    int n_head;
    int ocl;                     // output cluster = dhv / 128 (1, 2 or 4; set by launch)
};

// The output epilogue fuses into K12 when the head's x tiles fit one cluster
// whose partial sums fit the exchange buffer (dhv / 128 in {1, 2, 4}).
bool fwd_fused_out_supported(const Geom& g);

bool fwd_fused_supported(const Geom& g);

// q, k: bf16 [BH][T][dqk]; v: bf16 [BH][T][dhv]; saved: bf16 [BH][NC][dqk][dhv]
// (C_0 .. C_{NC-1}, the backward's operand states).
int launch_fwd_fused(const FusedFwdArgs& a, const void* q, const void* k, const void* v, void* saved,
                     cudaStream_t st);

}  // namespace tfla_k
