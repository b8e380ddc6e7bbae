// ubench_tmem.cu -- TMEM load / store throughput on one SM (design evidence for
// the fused forward: the per-chunk C round trip is TMEM-read bound).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -Ipaper_2503_14376_b200/csrc profiles/ubench_tmem.cu -o /tmp/ubench_tmem
// Prints cycles per 32x32b.x32 load / store per warp for 4 / 8 / 16 warps.
#include <cstdio>
#include <cuda_runtime.h>

#include "tc.cuh"

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
        "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
        "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}

__global__ void bench(int mode, int iters, long long* out, float* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tc::tmem_alloc(&slot, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t base = tc::tmem_row_addr(slot);
    const int nw = blockDim.x >> 5;
    // warps sharing a lane quarter split the 512 columns
    const int share = nw / 4, part = warp / 4;
    const int ncol = 512 / share;
    float acc = 0.f;
    uint32_t r[32];
    for (int i = 0; i < 32; ++i) r[i] = threadIdx.x + i;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        for (int c = 0; c < ncol; c += 32) {
            const uint32_t a = base + part * ncol + c;
            if (mode == 0) {
                float v[32];
                tc::tmem_ld32(a, v);
                tc::tmem_ld_wait();
                for (int i = 0; i < 32; ++i) acc += v[i];
            } else if (mode == 1) {
                tmem_st32(a, r);
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            } else {
                float v[32];
                tc::tmem_ld32(a, v);
                tc::tmem_ld_wait();
                for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(v[i] * 0.5f);
                tmem_st32(a, r);
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) *out = t1 - t0;
    if (acc == 1234.5f) *sink = acc;
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(slot, 512);
}

int main() {
    long long* d;
    float* s;
    cudaMalloc(&d, 8);
    cudaMalloc(&s, 4);
    const char* names[] = {"ld", "st", "ld+st"};
    for (int mode = 0; mode < 3; ++mode)
        for (int nw : {4, 8, 16}) {
            const int iters = 200;
            bench<<<1, nw * 32>>>(mode, iters, d, s);
            long long cyc;
            cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
            const double bytes = 128.0 * 512 * 4 * iters;  // whole TMEM per iteration
            printf("%-6s warps=%2d  %8.1f B/cyc/SM  (%lld cyc, err=%s)\n", names[mode], nw, bytes / cyc, cyc,
                   cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
