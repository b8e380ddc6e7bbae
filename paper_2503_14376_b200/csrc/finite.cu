// finite.cu -- the reference's input finiteness check (SequenceInputs::validate,
// core.cpp:106-117, all_finite core.cpp:114-116) on the device: one grid-stride
// pass over a buffer with 16-byte loads; any NaN / Inf sets a flag. Opt-in
// (tfla_check_finite), since it is a full HBM read of q, k, v and the gates.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"

namespace tfla_k {
namespace {

__device__ __forceinline__ bool bad_bf16x2(uint32_t w) {  // exponent all ones (NaN / Inf) in either half
    return (w & 0x7F800000u) == 0x7F800000u || (w & 0x00007F80u) == 0x00007F80u;
}
__device__ __forceinline__ bool bad_f32(uint32_t w) { return (w & 0x7F800000u) == 0x7F800000u; }

__global__ void nonfinite_kernel(const uint4* __restrict__ p, size_t n16, const uint8_t* __restrict__ tail,
                                 int ntail, int is_bf16, unsigned* flag) {
    bool bad = false;
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n16;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const uint4 v = p[i];
        bad |= is_bf16 ? (bad_bf16x2(v.x) | bad_bf16x2(v.y) | bad_bf16x2(v.z) | bad_bf16x2(v.w))
                       : (bad_f32(v.x) | bad_f32(v.y) | bad_f32(v.z) | bad_f32(v.w));
    }
    if (blockIdx.x == 0) {  // elements past the last full 16-byte word
        const int esz = is_bf16 ? 2 : 4;
        for (int e = threadIdx.x; e < ntail / esz; e += blockDim.x) {
            uint32_t w = 0;
            for (int b = 0; b < esz; ++b) w |= static_cast<uint32_t>(tail[e * esz + b]) << (8 * b);
            bad |= is_bf16 ? (w & 0x7F80u) == 0x7F80u : bad_f32(w);
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1u);
}

}  // namespace

void launch_nonfinite(const void* p, size_t bytes, bool is_bf16, unsigned* flag, int n_sm, cudaStream_t st) {
    const size_t n16 = bytes / 16;
    const int ntail = static_cast<int>(bytes - n16 * 16);
    const size_t want = (n16 + 255) / 256;
    const unsigned grid = static_cast<unsigned>(want < static_cast<size_t>(4 * n_sm) ? (want ? want : 1) : 4 * n_sm);
    nonfinite_kernel<<<grid, 256, 0, st>>>(static_cast<const uint4*>(p), n16,
                                           static_cast<const uint8_t*>(p) + n16 * 16, ntail, is_bf16 ? 1 : 0, flag);
}

}  // namespace tfla_k
