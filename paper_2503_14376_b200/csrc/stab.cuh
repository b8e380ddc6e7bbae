// stab.cuh -- opt-in stabiliser audit: the GPU counterpart of the reference's
// stab::exp_guarded (core.cpp:145-166), which counts every stabilised exp and
// every one whose argument is positive (tests assert zero violations,
// test_tiled.cpp:135-145, acceptance.cpp:158). Here every gating site notes its
// exponent argument BEFORE the fminf(arg, 0) clamp, so a wrong m / m_comb shows
// up as a counted violation instead of a silently clamped factor. Arguments are
// in log2 units (the kernels use exp2f); fp32 rounding of b - m_c + ib - b can
// push an exact-zero argument to ~1e-5, so a violation is arg > kStabTol
// (exp factor > 1.0007) -- a stabiliser off by even one log-gate is ~1 unit.
// Disabled (stab == nullptr): one predicated branch per element, no memory.
#pragma once
#include <cuda_runtime.h>

#include "kernels.h"

namespace tfla_k {

constexpr float kStabTol = 1.0f / 1024.0f;

struct StabLocal {
    unsigned checks = 0, viol = 0;
    float amax = 0.f;
    __device__ __forceinline__ void note(float arg_log2) {
        ++checks;
        viol += arg_log2 > kStabTol ? 1u : 0u;
        amax = fmaxf(amax, arg_log2);
    }
    __device__ __forceinline__ void flush(StabCounters* s) const {
        if (!s || !checks) return;
        atomicAdd(&s->checks, static_cast<unsigned long long>(checks));
        if (viol) atomicAdd(&s->violations, static_cast<unsigned long long>(viol));
        if (amax > 0.f) atomicMax(&s->max_bits, __float_as_uint(amax));
    }
};

}  // namespace tfla_k
