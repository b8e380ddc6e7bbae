// output.cu -- mLSTM cell output epilogue (eq. 5, :109-114):
//   h = sigmoid(o_pre) * rms_norm(h_tilde; gamma_head, eps)
// with rms_norm exactly as transfer.cpp:8-18 (mean over d_hv, rms == 0 -> 0).
// One warp per (b, h, t) row; 16-byte loads of h_tilde / o_pre, fp32 math,
// one shuffle reduction for the sum of squares. HBM-bound: reads 2 x 2 B and
// writes 2 B per element.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"

namespace tfla_k {
namespace {

template <int kMax>  // 16-B chunks per lane: ceil(d_hv / 256)
__global__ void __launch_bounds__(256) output_norm_gate_kernel(const __nv_bfloat16* __restrict__ ht,
                                                                const __nv_bfloat16* __restrict__ op,
                                                                const float* __restrict__ gamma, float eps,
                                                                __nv_bfloat16* __restrict__ h, long rows, int T,
                                                                int NH, int dhv) {
    const long r = static_cast<long>(blockIdx.x) * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    const int head = static_cast<int>((r / T) % NH);
    const uint4* x4 = reinterpret_cast<const uint4*>(ht + r * dhv);
    const uint4* o4 = reinterpret_cast<const uint4*>(op + r * dhv);
    const int nch = dhv / 8;
    uint4 xv[kMax], ov[kMax];
    float sq = 0.f;
#pragma unroll
    for (int i = 0; i < kMax; ++i) {  // both operands in flight before the reduction
        const int c = lane + 32 * i;
        if (c < nch) {
            xv[i] = x4[c];
            ov[i] = o4[c];
        }
    }
#pragma unroll
    for (int i = 0; i < kMax; ++i) {
        const int c = lane + 32 * i;
        if (c < nch) {
            const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&xv[i]);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(p2[e]);
                sq = fmaf(f.x, f.x, fmaf(f.y, f.y, sq));
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    const float rms = sqrtf(sq / static_cast<float>(dhv) + eps);
    const float inv = rms == 0.f ? 0.f : 1.f / rms;
    const float* g = gamma + static_cast<size_t>(head) * dhv;
    uint4* y4 = reinterpret_cast<uint4*>(h + r * dhv);
#pragma unroll
    for (int i = 0; i < kMax; ++i) {
        const int c = lane + 32 * i;
        if (c < nch) {
            const __nv_bfloat162* x2 = reinterpret_cast<const __nv_bfloat162*>(&xv[i]);
            const __nv_bfloat162* o2 = reinterpret_cast<const __nv_bfloat162*>(&ov[i]);
            const float4 g0 = *reinterpret_cast<const float4*>(g + c * 8);
            const float4 g1 = *reinterpret_cast<const float4*>(g + c * 8 + 4);
            const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
            uint4 out;
            uint32_t* w = reinterpret_cast<uint32_t*>(&out);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 xf = __bfloat1622float2(x2[e]);
                const float2 of = __bfloat1622float2(o2[e]);
                const float s0 = 1.f / (1.f + __expf(-of.x)), s1 = 1.f / (1.f + __expf(-of.y));
                const __nv_bfloat162 hv =
                    __floats2bfloat162_rn(s0 * xf.x * inv * gg[2 * e], s1 * xf.y * inv * gg[2 * e + 1]);
                w[e] = *reinterpret_cast<const uint32_t*>(&hv);
            }
            y4[c] = out;
        }
    }
}

// softcap (gates.cpp:15-18) applied to both gate pre-activations
// (apply_gate_softcap, gates.cpp:61-67): x <- c tanh(x / c), f64 math.
__global__ void gate_softcap_kernel(const float* __restrict__ ip, const float* __restrict__ fp, float* io,
                                    float* fo, long n, double cap) {
    for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long>(gridDim.x) * blockDim.x) {
        io[i] = static_cast<float>(cap * tanh(static_cast<double>(ip[i]) / cap));
        fo[i] = static_cast<float>(cap * tanh(static_cast<double>(fp[i]) / cap));
    }
}

}  // namespace

void launch_gate_softcap(const float* ip, const float* fp, float* io, float* fo, long n, double cap,
                         cudaStream_t st) {
    const long blocks = (n + 255) / 256;
    gate_softcap_kernel<<<static_cast<unsigned>(blocks < 4096 ? blocks : 4096), 256, 0, st>>>(ip, fp, io, fo, n, cap);
}

bool output_supported(int dhv) { return dhv % 8 == 0 && dhv <= 2048 && dhv > 0; }

void launch_output_norm_gate(const __nv_bfloat16* ht, const __nv_bfloat16* op, const float* gamma, float eps,
                             __nv_bfloat16* h, long rows, int T, int NH, int dhv, cudaStream_t st) {
    const unsigned grid = static_cast<unsigned>((rows + 7) / 8);
    const int per = (dhv / 8 + 31) / 32;
    if (per <= 1) output_norm_gate_kernel<1><<<grid, 256, 0, st>>>(ht, op, gamma, eps, h, rows, T, NH, dhv);
    else if (per <= 2) output_norm_gate_kernel<2><<<grid, 256, 0, st>>>(ht, op, gamma, eps, h, rows, T, NH, dhv);
    else if (per <= 4) output_norm_gate_kernel<4><<<grid, 256, 0, st>>>(ht, op, gamma, eps, h, rows, T, NH, dhv);
    else output_norm_gate_kernel<8><<<grid, 256, 0, st>>>(ht, op, gamma, eps, h, rows, T, NH, dhv);
}

}  // namespace tfla_k
