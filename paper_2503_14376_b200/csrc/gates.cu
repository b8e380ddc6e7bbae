// gates.cu -- K0: chunkwise log gates and stabilisers (f64 scans, fp32 out).
//
// Restates gates.cpp:20-53 (b = inclusive in-chunk cumsum of logsig(f),
// a = reverse tail sum + i_bar, g = b_{L-1}), the max-state recurrence of
// chunkwise.cpp:33-44 (m_0 = 0, m_{k+1} = max(g_k + m_k, max_j a_{k,j})) and
// the combine stabiliser of chunkwise.cpp:110-135. The in-chunk row max is
// separable, max_{j<=i}(b_i - b_j + i_j) = b_i + prefmax_{j<=i}(i_j - b_j), so
// every stabiliser is known before any matmul runs.
// One CTA per (chunk, head), one thread per position (L <= 1024).
#include <cuda_runtime.h>
#include <math.h>

#include "kernels.h"
#include "stab.cuh"

namespace tfla_k {
namespace {

__device__ __forceinline__ double logsig(double x) { return fmin(x, 0.0) - log1p(exp(-fabs(x))); }

// Block-wide inclusive scan (op = sum or max) over blockDim.x <= 1024 threads.
template <bool kMax>
__device__ double block_scan(double v, double* sh) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        double u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v = kMax ? fmax(v, u) : v + u;
    }
    if (lane == 31) sh[wid] = v;
    __syncthreads();
    if (wid == 0) {
        double t = lane < nw ? sh[lane] : (kMax ? -INFINITY : 0.0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            double u = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t = kMax ? fmax(t, u) : t + u;
        }
        sh[lane] = t;
    }
    __syncthreads();
    if (wid > 0) {
        const double pre = sh[wid - 1];
        v = kMax ? fmax(v, pre) : v + pre;
    }
    __syncthreads();
    return v;
}

__device__ double block_max(double v, double* sh) {
    double r = block_scan<true>(v, sh);
    __shared__ double last;
    if (threadIdx.x == blockDim.x - 1) last = r;
    __syncthreads();
    return last;
}

struct ChunkGates {
    double fbar, b, a, ib, g, amax, mintra;
};

// Per-thread view of one chunk's gates (thread j = chunk position j).
// kStab = false skips the two max scans (amax, m_intra) the backward does not need.
template <bool kStab = true>
__device__ ChunkGates chunk_gates(const float* f, const float* ip, int variant, double* sh) {
    const int j = threadIdx.x, L = blockDim.x;
    ChunkGates r;
    r.fbar = logsig(static_cast<double>(f[j]));
    r.ib = variant == 0 ? static_cast<double>(ip[j]) : logsig(static_cast<double>(ip[j]));
    r.b = block_scan<false>(r.fbar, sh);
    // reverse inclusive scan: thread j holds fbar of position L-1-j
    __shared__ double fb_s[1024];
    fb_s[j] = r.fbar;
    __syncthreads();
    const double rev = block_scan<false>(fb_s[L - 1 - j], sh);  // sum_{u >= L-1-j} fbar_u
    __shared__ double tail_s[1024];
    tail_s[L - 1 - j] = rev - fb_s[L - 1 - j];                  // sum_{u > L-1-j}
    __syncthreads();
    r.a = tail_s[j] + r.ib;
    __shared__ double g_s;
    if (j == L - 1) g_s = r.b;
    __syncthreads();
    r.g = g_s;
    if (kStab) {
        r.amax = block_max(r.a, sh);
        r.mintra = r.b + block_scan<true>(r.ib - r.b, sh);
    } else {
        r.amax = r.mintra = 0.0;
    }
    return r;
}

// chunkwise_gates (gates.hpp:31-35 / gates.cpp:20-59) exported in f64.
__global__ void gates_export_kernel(const float* __restrict__ f_pre, const float* __restrict__ i_pre, int T,
                                    int NC, int variant, double* g_sum, double* b_cum, double* a_tail) {
    __shared__ double sh[32];
    const int c = blockIdx.x, bh = blockIdx.y, L = blockDim.x;
    const size_t base = static_cast<size_t>(bh) * T + static_cast<size_t>(c) * L;
    ChunkGates r = chunk_gates(f_pre + base, i_pre + base, variant, sh);
    if (b_cum) b_cum[base + threadIdx.x] = r.b;
    if (a_tail) a_tail[base + threadIdx.x] = r.a;
    if (g_sum && threadIdx.x == 0) g_sum[static_cast<size_t>(bh) * NC + c] = r.g;
}

__global__ void gates_chunk_kernel(const float* __restrict__ f_pre, const float* __restrict__ i_pre,
                                   int T, int NC, int variant, double* gsum, double* amax, double* gtmp,
                                   size_t BT) {
    __shared__ double sh[32];
    const int c = blockIdx.x, bh = blockIdx.y, L = blockDim.x;
    const size_t base = static_cast<size_t>(bh) * T + static_cast<size_t>(c) * L;
    ChunkGates r = chunk_gates(f_pre + base, i_pre + base, variant, sh);
    if (gtmp) {  // the finalize pass reads these instead of repeating the block scans
        const size_t t = base + threadIdx.x;
        gtmp[t] = r.b;
        gtmp[BT + t] = r.a;
        gtmp[2 * BT + t] = r.ib;
        gtmp[3 * BT + t] = r.mintra;
    }
    if (threadIdx.x == 0) {
        gsum[static_cast<size_t>(bh) * NC + c] = r.g;
        amax[static_cast<size_t>(bh) * NC + c] = r.amax;
    }
}

__global__ void gates_finalize_kernel(const float* __restrict__ f_pre,
                                      const float* __restrict__ i_pre, int T, int NC, int variant,
                                      GateWS ws, float* m_states, float* m_comb, float* m_final,
                                      const float* __restrict__ m_init,
                                      const float* __restrict__ m_given,
                                      const float* __restrict__ mc_given) {
    __shared__ double sh[32];
    __shared__ double m_pair[2];
    const int c = blockIdx.x, bh = blockIdx.y, L = blockDim.x, j = threadIdx.x;
    const size_t base = static_cast<size_t>(bh) * T + static_cast<size_t>(c) * L;
    ChunkGates r;
    if (ws.gtmp) {  // from the chunk pass
        const size_t BT = static_cast<size_t>(gridDim.y) * T, t = base + j;
        r.b = ws.gtmp[t];
        r.a = ws.gtmp[BT + t];
        r.ib = ws.gtmp[2 * BT + t];
        r.mintra = ws.gtmp[3 * BT + t];
        __shared__ double g_s;
        if (j == L - 1) g_s = r.b;
        __syncthreads();
        r.g = g_s;
    } else {
        r = chunk_gates(f_pre + base, i_pre + base, variant, sh);
    }
    if (j == 0) {
        if (variant == 0 && m_given) {  // caller's max states (tfla_forward_head input)
            const float* mg = m_given + static_cast<size_t>(bh) * (NC + 1);
            m_pair[0] = mg[c];
            m_pair[1] = mg[c + 1];
        } else if (variant == 0) {  // m_c, m_{c+1} from mscan_kernel (ws.gsum now holds m_1..m_NC)
            const double* ms = ws.gsum + static_cast<size_t>(bh) * NC;
            // m_0 = 0 (chunkwise.cpp:23) or the caller's initial max state
            m_pair[0] = c == 0 ? (m_init ? static_cast<double>(m_init[bh]) : 0.0) : ms[c - 1];
            m_pair[1] = ms[c];
        } else {
            m_pair[0] = m_pair[1] = 0.0;
        }
    }
    __syncthreads();
    const double mk = m_pair[0], mk1 = m_pair[1];
    const size_t t = base + j;
    double mc, abar, bbar, gbar;
    if (variant == 0) {
        // chunkwise_forward_frozen (chunkwise.cpp:304-394) pins m_comb as well
        mc = mc_given ? static_cast<double>(mc_given[t]) : fmax(r.b + mk, r.mintra);
        abar = exp(r.a - mk1);
        bbar = exp(r.b + mk - mc);
        gbar = exp(r.g + mk - mk1);
        if (ws.stab) {  // stab::exp_guarded at chunkwise.cpp:40-43, 130
            constexpr double kL2e = 1.4426950408889634;
            StabLocal sl;
            sl.note(static_cast<float>((r.a - mk1) * kL2e));
            sl.note(static_cast<float>((r.b + mk - mc) * kL2e));
            if (j == 0) sl.note(static_cast<float>((r.g + mk - mk1) * kL2e));
            sl.flush(ws.stab);
        }
    } else {
        mc = 0.0;
        abar = exp(r.a);
        bbar = exp(r.b);
        gbar = exp(r.g);
    }
    ws.b[t] = static_cast<float>(r.b);
    ws.ib[t] = static_cast<float>(r.ib);
    ws.mc[t] = static_cast<float>(mc);
    ws.ab[t] = static_cast<float>(abar);
    ws.bb[t] = static_cast<float>(bbar);
    if (m_comb) m_comb[t] = static_cast<float>(mc);
    if (j == 0) ws.gbar[static_cast<size_t>(bh) * NC + c] = static_cast<float>(gbar);
    if (j == 0 && m_states) {
        m_states[static_cast<size_t>(bh) * (NC + 1) + c] = static_cast<float>(mk);
        if (c == NC - 1) {
            m_states[static_cast<size_t>(bh) * (NC + 1) + NC] = static_cast<float>(mk1);
            if (m_final) m_final[bh] = static_cast<float>(mk1);
        }
    }
}

// Max-state recurrence m_{k+1} = max(g_k + m_k, amax_k), m_0 = 0
// (chunkwise.cpp:33-44) as a warp scan of max-plus maps f_k(m) = max(m + g_k, a_k):
// f2 o f1 = (g1 + g2, max(a1 + g2, a2)). One warp per head, 32 chunks per step;
// overwrites gsum[k] with m_{k+1} (the chunk sums are consumed here only).
__global__ void mscan_kernel(double* __restrict__ gsum, const double* __restrict__ amax, int NC,
                             const float* __restrict__ m_init) {
    const int bh = blockIdx.x, lane = threadIdx.x;
    double* gs = gsum + static_cast<size_t>(bh) * NC;
    const double* am = amax + static_cast<size_t>(bh) * NC;
    double m = m_init ? static_cast<double>(m_init[bh]) : 0.0;
    for (int k0 = 0; k0 < NC; k0 += 32) {
        const int k = k0 + lane;
        double G = k < NC ? gs[k] : 0.0, A = k < NC ? am[k] : -INFINITY;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {  // inclusive scan: (G, A) = f_k o ... o f_{k-o+1} style
            const double Gp = __shfl_up_sync(0xffffffffu, G, o), Ap = __shfl_up_sync(0xffffffffu, A, o);
            if (lane >= o) {
                A = fmax(Ap + G, A);
                G = Gp + G;
            }
        }
        const double mk1 = fmax(m + G, A);
        if (k < NC) gs[k] = mk1;
        m = __shfl_sync(0xffffffffu, mk1, 31);
    }
}

__global__ void gates_bwd_kernel(const float* __restrict__ f_pre, const float* __restrict__ i_pre,
                                 int T, int NC, int dqk, int variant, const float* m_states,
                                 const float* m_comb, const float* h_denom, GateWS ws) {
    __shared__ double sh[32];
    const int c = blockIdx.x, bh = blockIdx.y, L = blockDim.x, j = threadIdx.x;
    const size_t base = static_cast<size_t>(bh) * T + static_cast<size_t>(c) * L;
    ChunkGates r = chunk_gates<false>(f_pre + base, i_pre + base, variant, sh);  // m_c comes saved
    const size_t t = base + j;
    const double rs = 1.0 / sqrt(static_cast<double>(dqk));
    double mc = 0.0, den = 1.0, abar, bbar, gbar;
    if (variant == 0) {
        const double mk = m_states[static_cast<size_t>(bh) * (NC + 1) + c];
        const double mk1 = m_states[static_cast<size_t>(bh) * (NC + 1) + c + 1];
        mc = m_comb[t];
        den = h_denom[t];
        abar = exp(r.a - mk1);        // chunkwise.cpp:542-544
        bbar = exp(r.b + mk - mc);    // chunkwise.cpp:508-510
        gbar = exp(r.g + mk - mk1);   // chunkwise.cpp:209-211
        if (ws.stab) {
            constexpr double kL2e = 1.4426950408889634;
            StabLocal sl;
            sl.note(static_cast<float>((r.a - mk1) * kL2e));
            sl.note(static_cast<float>((r.b + mk - mc) * kL2e));
            if (j == 0) sl.note(static_cast<float>((r.g + mk - mk1) * kL2e));
            sl.flush(ws.stab);
        }
    } else {
        abar = exp(r.a);
        bbar = exp(r.b);
        gbar = exp(r.g);
    }
    ws.b[t] = static_cast<float>(r.b);
    ws.ib[t] = static_cast<float>(r.ib);
    ws.mc[t] = static_cast<float>(mc);
    ws.ab[t] = static_cast<float>(abar);
    ws.bb[t] = static_cast<float>(bbar * rs / den);
    ws.dinv[t] = static_cast<float>(1.0 / den);
    if (j == 0) ws.gbar[static_cast<size_t>(bh) * NC + c] = static_cast<float>(gbar);
}

}  // namespace

void launch_gates_fwd(const Geom& g, int variant, const float* f_pre, const float* i_pre,
                      const GateWS& ws, float* m_states, float* m_comb, float* m_final,
                      cudaStream_t st, const float* m_init) {
    dim3 grid(g.NC, g.BH);
    if (variant != 0) m_init = nullptr;  // mLSTMsig carries no max state
    gates_chunk_kernel<<<grid, g.L, 0, st>>>(f_pre, i_pre, g.T, g.NC, variant, ws.gsum, ws.amax, ws.gtmp,
                                             static_cast<size_t>(g.BH) * g.T);
    if (variant == 0) mscan_kernel<<<g.BH, 32, 0, st>>>(ws.gsum, ws.amax, g.NC, m_init);
    gates_finalize_kernel<<<grid, g.L, 0, st>>>(f_pre, i_pre, g.T, g.NC, variant, ws, m_states,
                                                m_comb, m_final, m_init, nullptr, nullptr);
}

void launch_gates_fwd_given_m(const Geom& g, int variant, const float* f_pre, const float* i_pre,
                              const GateWS& ws, const float* m_states, float* m_comb, cudaStream_t st,
                              const float* mc_given) {
    dim3 grid(g.NC, g.BH);
    GateWS w = ws;
    w.gtmp = nullptr;  // no chunk pass ran: the finalize pass computes the scans itself
    gates_finalize_kernel<<<grid, g.L, 0, st>>>(f_pre, i_pre, g.T, g.NC, variant, w, nullptr, m_comb,
                                                nullptr, nullptr, m_states, mc_given);
}

void launch_gates_export(const Geom& g, int variant, const float* f_pre, const float* i_pre, double* g_sum,
                         double* b_cum, double* a_tail, cudaStream_t st) {
    gates_export_kernel<<<dim3(g.NC, g.BH), g.L, 0, st>>>(f_pre, i_pre, g.T, g.NC, variant, g_sum, b_cum, a_tail);
}

void launch_gates_bwd(const Geom& g, int variant, const float* f_pre, const float* i_pre,
                      const float* m_states, const float* m_comb, const float* h_denom,
                      const GateWS& ws, cudaStream_t st) {
    dim3 grid(g.NC, g.BH);
    gates_bwd_kernel<<<grid, g.L, 0, st>>>(f_pre, i_pre, g.T, g.NC, g.dqk, variant, m_states,
                                           m_comb, h_denom, ws);
}

}  // namespace tfla_k
