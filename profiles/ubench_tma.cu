// ubench_tma.cu -- per-SM TMA ingest rate (design evidence for the state scans:
// is ~20-24 B/cycle/SM a TMA / L2 limit or the kernel's own pipeline?).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -Ipaper_2503_14376_b200/csrc profiles/ubench_tma.cu -lcuda -o /tmp/ubench_tma
// Each CTA streams its own [rows][cols] bf16 slab through a ring of `stages`
// stages of `boxes` TMA boxes (box_cols x box_rows, SWIZZLE_128B); one consumer
// thread waits each stage and releases it. Prints bytes / SM cycle and TB/s.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc.cuh"

struct P {
    int stages, boxes, box_rows, iters, l2_resident, issuers;
};

__global__ void __launch_bounds__(160, 1)
    ingest(const __grid_constant__ CUtensorMap map, P p, long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int box_bytes = 128 * p.box_rows;
    const int stage_bytes = box_bytes * p.boxes;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.stages * stage_bytes);
    uint64_t* empty = full + p.stages;
    if (threadIdx.x == 0) {
        for (int s = 0; s < p.stages; ++s) {
            tc::mbar_init(&full[s], p.issuers);
            tc::mbar_init(&empty[s], 1);
        }
        tc::fence_barrier_init();
    }
    __syncthreads();
    // l2_resident 1: eight shared slabs (8 CTAs read the same rows at once);
    // 2: each CTA re-reads its own 512 rows (L2-resident, no sharing)
    const int slab = p.l2_resident == 1 ? (blockIdx.x & 7) : blockIdx.x;
    const int wrap = p.l2_resident == 2 ? 1024 : 1 << 30;
    const long long t0 = clock64();
    // issuers: the stage's boxes are split over this many producer warps (lane 0 each)
    const int w = threadIdx.x >> 5;
    if (w >= 1 && w <= p.issuers && (threadIdx.x & 31) == 0) {
        const int me = w - 1;
        const int per = p.boxes / p.issuers;
        for (int i = 0; i < p.iters; ++i) {
            const int s = i % p.stages;
            tc::mbar_wait(&empty[s], ((i / p.stages) & 1) ^ 1);
            tc::mbar_arrive_expect_tx(&full[s], per * box_bytes);
            for (int b = me * per; b < (me + 1) * per; ++b)
                tc::tma_load_3d(smem + s * stage_bytes + b * box_bytes, &map, &full[s], 64 * b,
                                (i * p.box_rows) % wrap, slab);
        }
    } else if (threadIdx.x == 0) {
        for (int i = 0; i < p.iters; ++i) {
            const int s = i % p.stages;
            tc::mbar_wait(&full[s], (i / p.stages) & 1);
            tc::mbar_arrive(&empty[s]);
        }
        cyc[blockIdx.x] = clock64() - t0;
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int cols = 256;  // K rows of the 7B shape: 512 B pitch, a box takes 64 columns
    struct Case {
        int grid, stages, boxes, box_rows, l2, issuers;
    };
    std::vector<Case> cases = {
        {128, 4, 3, 64, 0, 1},  {128, 8, 3, 64, 0, 1},  {148, 4, 3, 64, 0, 1},  {148, 8, 3, 64, 0, 1},
        {296, 4, 3, 64, 0, 1},  {148, 3, 4, 128, 0, 1}, {148, 6, 4, 64, 0, 1},  {148, 3, 2, 256, 0, 1},
        {148, 4, 3, 64, 1, 1},  {148, 8, 3, 64, 1, 1},  {148, 3, 4, 128, 1, 1}, {128, 8, 3, 64, 1, 1},
        {148, 4, 3, 64, 2, 1},  {148, 8, 3, 64, 2, 1},  {148, 3, 4, 128, 2, 1}, {296, 4, 3, 64, 2, 1},
        {148, 8, 3, 64, 2, 3},  {148, 6, 4, 64, 2, 2},  {148, 6, 4, 64, 2, 4},  {148, 3, 2, 256, 2, 1},
        {148, 3, 2, 256, 2, 2}, {148, 8, 3, 64, 1, 3},  {128, 8, 3, 64, 0, 3},  {148, 6, 4, 64, 0, 4},
        {148, 3, 4, 128, 0, 4}, {148, 3, 2, 256, 0, 2},
    };
    const int rows_per_slab = 16384;
    for (const Case& c : cases) {
        const int slabs = c.l2 == 1 ? 8 : c.grid;
        void* buf = nullptr;
        const size_t bytes = static_cast<size_t>(slabs) * rows_per_slab * cols * 2;
        if (cudaMalloc(&buf, bytes) != cudaSuccess) return 1;
        cudaMemset(buf, 0, bytes);
        CUtensorMap map;
        cuuint64_t dims[3] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows_per_slab),
                              static_cast<cuuint64_t>(slabs)};
        cuuint64_t strides[2] = {static_cast<cuuint64_t>(cols) * 2,
                                 static_cast<cuuint64_t>(cols) * 2 * rows_per_slab};
        cuuint32_t box[3] = {64, static_cast<cuuint32_t>(c.box_rows), 1};
        cuuint32_t es[3] = {1, 1, 1};
        if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return 2;
        P p{c.stages, c.boxes, c.box_rows, rows_per_slab / c.box_rows, c.l2, c.issuers};
        const int smem = c.stages * c.boxes * 128 * c.box_rows + 2 * 8 * c.stages;
        cudaFuncSetAttribute(ingest, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        long long* cyc = nullptr;
        cudaMalloc(&cyc, c.grid * sizeof(long long));
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a);
            ingest<<<c.grid, 160, smem>>>(map, p, cyc);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        if (cudaGetLastError() != cudaSuccess) return 3;
        std::vector<long long> h(c.grid);
        cudaMemcpy(h.data(), cyc, c.grid * sizeof(long long), cudaMemcpyDeviceToHost);
        double mc = 0;
        for (long long v : h) mc += v;
        mc /= c.grid;
        const double per_cta = static_cast<double>(p.iters) * c.boxes * 128 * c.box_rows;
        printf("issuers %d grid %3d stages %d boxes %d x (64 x %3d) stage %3d KB %s: %6.1f B/cycle/CTA, %5.2f TB/s (%.3f ms)\n",
               c.issuers, c.grid, c.stages, c.boxes, c.box_rows, c.boxes * c.box_rows * 128 / 1024,
               c.l2 == 1 ? "L2 shared x8" : c.l2 == 2 ? "L2 own slab " : "HBM         ", per_cta / mc, per_cta * c.grid / (best * 1e-3) / 1e12, best);
        cudaFree(cyc);
        cudaFree(buf);
    }
    (void)sms;
    return 0;
}
