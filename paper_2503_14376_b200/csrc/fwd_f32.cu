// fwd_f32.cu -- fp32-operand chunkwise forward on CUDA cores.
//
// BASELINE config 0 as worded ("mLSTMexp chunkwise forward fp32", B=1 NH=2
// S=256 d=64 L=64): the reference's <float, float> instantiation of
// chunkwise_forward_head (chunkwise.cpp:80-194, state_recurrence_head :13-78)
// on fp32 q / k / v without bf16 rounding. The tensor-core kernels take bf16
// operands (tcgen05 kind::f16); this path keeps every operand and product in
// fp32 for the reference-precision case, at sizes where the whole chunk fits
// in shared memory (L * d_qk <= 8192, dqk <= 256).
//
// One CTA per (64-column d_hv tile, head) walks the chunks in order with
// C[:, x tile] and n resident in shared memory. Per chunk k:
//   S_ij  = q_i . k_j / sqrt(d)                          (j <= i)
//   Sb_ij = S_ij exp(b_i - b_j + ib_j - m_c,i)           (exp; sig: no m_c)
//   H_i   = sum_j Sb_ij v_j + b_bar_i (q_i / sqrt(d))^T C_k
//   den_i = max(|sum_j Sb_ij + b_bar_i q_i . n_k / sqrt(d)|, exp(-m_c,i))  (exp; sig: 1)
//   C_{k+1} = gbar_k C_k + sum_j a_bar_j k_j v_j^T,  n_{k+1} = gbar_k n_k + sum_j a_bar_j k_j
// with the gate vectors of K0 (gates.cu: f64 scans, fp32 outputs).
#include <cuda_runtime.h>

#include "kernels.h"

namespace tfla_k {
namespace {

constexpr int kCols = 64;
constexpr int kThreads = 256;

struct F32Smem {
    int dqk, L;
    __host__ __device__ int kstride() const { return dqk + 1; }  // padded K rows (no bank conflicts)
    __host__ __device__ int offC() const { return 0; }                        // [dqk][64]
    __host__ __device__ int offQ() const { return offC() + dqk * kCols; }     // [L][dqk]
    __host__ __device__ int offK() const { return offQ() + L * dqk; }         // [L][dqk + 1]
    __host__ __device__ int offV() const { return offK() + L * kstride(); }   // [L][64]
    __host__ __device__ int offS() const { return offV() + L * kCols; }       // [L][L + 1]
    __host__ __device__ int offN() const { return offS() + L * (L + 1); }     // [dqk]
    __host__ __device__ int offR() const { return offN() + dqk; }             // [L] row sums
    __host__ __device__ int floats() const { return offR() + L; }
};

__global__ void __launch_bounds__(kThreads) fwd_f32_kernel(F32FwdArgs a) {
    extern __shared__ float sm[];
    const Geom& G = a.g;
    const int T = G.T, L = G.L, NC = G.NC, dqk = G.dqk, dhv = G.dhv;
    const F32Smem lay{dqk, L};
    float* C = sm + lay.offC();
    float* Q = sm + lay.offQ();
    float* K = sm + lay.offK();
    float* V = sm + lay.offV();
    float* S = sm + lay.offS();
    float* nv = sm + lay.offN();
    float* rowv = sm + lay.offR();
    const int ks = lay.kstride(), ss = L + 1;
    const int xt = blockIdx.x, bh = blockIdx.y, x0 = xt * kCols;
    const int tid = threadIdx.x;
    const bool is_exp = a.variant == 0;
    const float rs = rsqrtf(static_cast<float>(dqk));
    const size_t hb = static_cast<size_t>(bh) * T;

    for (int i = tid; i < dqk * kCols; i += kThreads) C[i] = 0.f;
    for (int i = tid; i < dqk; i += kThreads) nv[i] = 0.f;
    __syncthreads();

    auto emit_state = [&](int c, float* cs, float* ns) {  // state entering chunk c
        if (cs)
            for (int i = tid; i < dqk * kCols; i += kThreads)
                cs[((static_cast<size_t>(bh) * (NC + 1) + c) * dqk + i / kCols) * dhv + x0 + i % kCols] = C[i];
        if (ns && xt == 0)
            for (int p = tid; p < dqk; p += kThreads) ns[(static_cast<size_t>(bh) * (NC + 1) + c) * dqk + p] = nv[p];
    };

    for (int c = 0; c < NC; ++c) {
        emit_state(c, a.c_states, is_exp ? a.n_states : nullptr);
        const size_t t0 = hb + static_cast<size_t>(c) * L;
        for (int i = tid; i < L * dqk; i += kThreads) {
            const int r = i / dqk, p = i % dqk;
            Q[r * dqk + p] = a.q[(t0 + r) * dqk + p];
            K[r * ks + p] = a.k[(t0 + r) * dqk + p];
        }
        for (int i = tid; i < L * kCols; i += kThreads) V[i] = a.v[(t0 + i / kCols) * dhv + x0 + i % kCols];
        __syncthreads();
        // gated scores
        for (int idx = tid; idx < L * L; idx += kThreads) {
            const int i = idx / L, j = idx % L;
            float sb = 0.f;
            if (j <= i) {
                float s = 0.f;
                for (int p = 0; p < dqk; ++p) s = fmaf(Q[i * dqk + p], K[j * ks + p], s);
                const float bi = a.gw.b[t0 + i], bj = a.gw.b[t0 + j], ibj = a.gw.ib[t0 + j];
                const float arg = is_exp ? bi - bj + ibj - a.gw.mc[t0 + i] : bi - bj + ibj;
                sb = s * rs * expf(fminf(arg, 0.f));  // the stabiliser keeps arg <= 0 (up to rounding)
            }
            S[i * ss + j] = sb;
        }
        __syncthreads();
        // row sums + (exp) the denominator's inter term q_i . n_k
        for (int i = tid; i < L; i += kThreads) {
            float r = 0.f;
            for (int j = 0; j <= i; ++j) r += S[i * ss + j];
            float qn = 0.f;
            if (is_exp)
                for (int p = 0; p < dqk; ++p) qn = fmaf(Q[i * dqk + p], nv[p], qn);
            const float w = a.gw.bb[t0 + i] * rs;
            float den = 1.f;
            if (is_exp) den = fmaxf(fabsf(r + w * qn), expf(-a.gw.mc[t0 + i]));
            rowv[i] = 1.f / den;
            if (xt == 0 && a.h_denom) a.h_denom[t0 + i] = den;
        }
        __syncthreads();
        // H = (Sb V + w (Q C)) / den
        for (int idx = tid; idx < L * kCols; idx += kThreads) {
            const int i = idx / kCols, x = idx % kCols;
            float hi = 0.f, hc = 0.f;
            for (int j = 0; j <= i; ++j) hi = fmaf(S[i * ss + j], V[j * kCols + x], hi);
            for (int p = 0; p < dqk; ++p) hc = fmaf(Q[i * dqk + p], C[p * kCols + x], hc);
            a.h[(t0 + i) * dhv + x0 + x] = (hi + a.gw.bb[t0 + i] * rs * hc) * rowv[i];
        }
        __syncthreads();
        // state update: C <- gbar C + sum_j a_bar_j k_j v_j^T ; n <- gbar n + sum_j a_bar_j k_j
        const float gb = a.gw.gbar[static_cast<size_t>(bh) * NC + c];
        for (int idx = tid; idx < dqk * kCols; idx += kThreads) {
            const int p = idx / kCols, x = idx % kCols;
            float u = 0.f;
            for (int j = 0; j < L; ++j) u = fmaf(a.gw.ab[t0 + j] * K[j * ks + p], V[j * kCols + x], u);
            C[idx] = fmaf(gb, C[idx], u);
        }
        if (is_exp)
            for (int p = tid; p < dqk; p += kThreads) {
                float u = 0.f;
                for (int j = 0; j < L; ++j) u = fmaf(a.gw.ab[t0 + j], K[j * ks + p], u);
                nv[p] = fmaf(gb, nv[p], u);
            }
        __syncthreads();
    }
    emit_state(NC, a.c_states, is_exp ? a.n_states : nullptr);
    if (a.c_final)
        for (int i = tid; i < dqk * kCols; i += kThreads)
            a.c_final[(static_cast<size_t>(bh) * dqk + i / kCols) * dhv + x0 + i % kCols] = C[i];
    if (a.n_final && xt == 0)
        for (int p = tid; p < dqk; p += kThreads) a.n_final[static_cast<size_t>(bh) * dqk + p] = is_exp ? nv[p] : 0.f;
}

}  // namespace

size_t fwd_f32_smem_bytes(const Geom& g) { return static_cast<size_t>(F32Smem{g.dqk, g.L}.floats()) * 4; }

bool fwd_f32_supported(const Geom& g) {
    return g.dhv % kCols == 0 && g.dqk <= 256 && g.L * g.dqk <= 8192 && fwd_f32_smem_bytes(g) <= 232448;
}

int launch_fwd_f32(const F32FwdArgs& a, cudaStream_t st) {
    const size_t smem = fwd_f32_smem_bytes(a.g);
    cudaFuncSetAttribute(fwd_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    fwd_f32_kernel<<<dim3(a.g.dhv / kCols, a.g.BH), kThreads, smem, st>>>(a);
    return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

}  // namespace tfla_k
