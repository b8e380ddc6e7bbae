// selftest.cu -- building-block self test for the tcgen05/TMA machinery that
// every TFLA kernel relies on: D[128,N] = A[128,K] * B[N,K]^T with A and B in
// each supported shared-memory form (TMA-loaded K-major / MN-major operands,
// thread-written "stationary" operands read K-major or MN-major), a two-stage
// TMA->MMA ring, TMEM epilogue loads and a swizzled TMA store of the bf16
// result. Exposed as tfla_selftest_gemm() for the GPU test-suite.
#include <cuda_runtime.h>

#include "host_util.h"
#include "tc.cuh"
#include "tfla/tfla.h"

namespace {

constexpr int kStages = 2;
constexpr int kStageA = 128 * 64 * 2;  // 16 KB
constexpr int kStageB = 256 * 64 * 2;  // 32 KB
constexpr int kStageBytes = kStageA + kStageB;
constexpr int kStatBytes = 128 * 256 * 2;  // 64 KB
constexpr int kOutBytes = 128 * 256 * 2;   // 64 KB
constexpr int kSmemBytes = kStages * kStageBytes + kStatBytes + kOutBytes + 1024 + 256;

struct SelfTestArgs {
    int a_mode, b_mode, N, K;
    const __nv_bfloat16* a_raw;  // for stationary modes
    float* out;
};

__global__ void __launch_bounds__(192, 1)
    selftest_gemm_kernel(const __grid_constant__ CUtensorMap map_a,
                         const __grid_constant__ CUtensorMap map_b,
                         const __grid_constant__ CUtensorMap map_out, SelfTestArgs args) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint8_t* stages = smem;
    uint8_t* stat = smem + kStages * kStageBytes;
    uint8_t* outs = stat + kStatBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(outs + kOutBytes);
    uint64_t* full = bars;              // [kStages]
    uint64_t* empty = bars + kStages;   // [kStages]
    uint64_t* accfull = bars + 2 * kStages;
    uint64_t* statfull = accfull + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(statfull + 1);

    const int N = args.N, K = args.K, nkb = K / 64;
    const int warp = tc::warp_id();
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        tc::mbar_init(accfull, 1);
        tc::mbar_init(statfull, 128);
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    const bool stationary = args.a_mode >= 2;  // 2, 3: thread-written smem; 4: TMEM
    if (warp == 0) {
        if (tc::elect_one()) {
            for (int kb = 0; kb < nkb; ++kb) {
                const int s = kb % kStages;
                const uint32_t ph = (kb / kStages) & 1;
                tc::mbar_wait(&empty[s], ph ^ 1);
                uint8_t* sa = stages + s * kStageBytes;
                uint8_t* sb = sa + kStageA;
                uint32_t bytes = N * 64 * 2 + (stationary ? 0 : kStageA);
                tc::mbar_arrive_expect_tx(&full[s], bytes);
                if (args.a_mode == 0) {
                    tc::tma_load_2d(sa, &map_a, &full[s], kb * 64, 0);
                } else if (args.a_mode == 1) {
                    for (int m = 0; m < 2; ++m)
                        tc::tma_load_2d(sa + m * 64 * 128, &map_a, &full[s], m * 64, kb * 64);
                }
                if (args.b_mode == 0) {
                    tc::tma_load_2d(sb, &map_b, &full[s], kb * 64, 0);
                } else {
                    for (int m = 0; m < N / 64; ++m)
                        tc::tma_load_2d(sb + m * 64 * 128, &map_b, &full[s], m * 64, kb * 64);
                }
            }
        }
    } else if (warp == 1) {
        if (stationary) tc::mbar_wait(statfull, 0);
        tc::tc_fence_after();
        const uint32_t idesc =
            tc::idesc_bf16(128, N, (args.a_mode == 1 || args.a_mode == 3) ? 1 : 0, args.b_mode);
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % kStages;
            const uint32_t ph = (kb / kStages) & 1;
            tc::mbar_wait(&full[s], ph);
            tc::tc_fence_after();
            const uint32_t sa = tc::smem_u32(stages + s * kStageBytes);
            const uint32_t sb = sa + kStageA;
            if (tc::elect_one()) {
                for (int ks = 0; ks < 4; ++ks) {
                    uint64_t ad;
                    if (args.a_mode == 0)
                        ad = tc::kmajor_desc(sa, 128, ks);
                    else if (args.a_mode == 1)
                        ad = tc::mnmajor_desc(sa, 64, ks);
                    else if (args.a_mode == 2)
                        ad = tc::kmajor_desc(tc::smem_u32(stat), 128, kb * 4 + ks);
                    else
                        ad = tc::mnmajor_desc(tc::smem_u32(stat), K, kb * 4 + ks);
                    uint64_t bd = args.b_mode == 0 ? tc::kmajor_desc(sb, N, ks)
                                                   : tc::mnmajor_desc(sb, 64, ks);
                    if (args.a_mode == 4)  // A from TMEM: 16 K elements = 8 packed columns
                        tc::mma_bf16_ts(tmem, tmem + 256 + (kb * 4 + ks) * 8, bd, idesc, (kb | ks) ? 1u : 0u);
                    else
                        tc::mma_bf16(tmem, ad, bd, idesc, (kb | ks) ? 1u : 0u);
                }
                tc::mma_commit(&empty[s]);
                if (kb == nkb - 1) tc::mma_commit(accfull);
            }
            __syncwarp();
        }
    } else {
        const int et = threadIdx.x - 64;  // 0..127
        if (args.a_mode == 4) {
            // a_raw is A[128][K]; thread (lane quarter, lane) owns row r: bf16 pairs
            // packed per 32-bit TMEM column at columns 256 + k/2.
            const int r = (warp & 3) * 32 + tc::lane_id();
            for (int c = 0; c < K / 64; ++c) {
                uint32_t w[32];
                for (int j = 0; j < 32; ++j)
                    w[j] = *reinterpret_cast<const uint32_t*>(args.a_raw + r * K + c * 64 + 2 * j);
                tc::tmem_st32(tc::tmem_row_addr(tmem) + 256 + c * 32, w);
            }
            tc::tmem_st_wait();
            tc::tc_fence_before();
            tc::mbar_arrive(statfull);
        } else if (stationary) {
            // a_mode 2: a_raw is A[128][K]; write it as a K-major [128][K] tile.
            // a_mode 3: a_raw is X[K][128] (A = X^T); write X as [K][128] tile.
            const int rows = args.a_mode == 2 ? 128 : K;
            const int cols = args.a_mode == 2 ? K : 128;
            for (int r = et; r < rows; r += 128) {
                for (int c8 = 0; c8 < cols / 8; ++c8) {
                    uint4 v = *reinterpret_cast<const uint4*>(args.a_raw + r * cols + c8 * 8);
                    const uint32_t atom = c8 >> 3, chunk = (c8 & 7) ^ (r & 7);
                    *reinterpret_cast<uint4*>(stat + atom * rows * 128 + r * 128 + chunk * 16) = v;
                }
            }
            tc::fence_proxy_async_smem();
            tc::mbar_arrive(statfull);
        }
        tc::mbar_wait(accfull, 0);
        tc::tc_fence_after();
        const int row = (warp & 3) * 32 + tc::lane_id();
        for (int c = 0; c < N / 32; ++c) {
            float v[32];
            tc::tmem_ld32(tc::tmem_row_addr(tmem) + c * 32, v);
            tc::tmem_ld_wait();
            for (int j = 0; j < 32; ++j) args.out[row * N + c * 32 + j] = v[j];
            for (int j = 0; j < 4; ++j) tc::sw128_store8(outs, row, c * 4 + j, 128, v + 8 * j);
        }
        tc::fence_proxy_async_smem();
        tc::named_bar_sync(1, 128);
        if (et == 0) {
            for (int a = 0; a < N / 64; ++a) tc::tma_store_2d(&map_out, outs + a * 128 * 128, a * 64, 0);
            tc::tma_store_commit();
            tc::tma_store_wait_all<0>();
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

}  // namespace

extern "C" int tfla_selftest_gemm(int a_mode, int b_mode, int N, int K, const void* a,
                                  const void* b, float* out, void* out_bf16, void* stream) {
    using namespace tfla_host;
    if (a_mode < 0 || a_mode > 4 || b_mode < 0 || b_mode > 1 || N < 64 || N > 256 || N % 64 ||
        K < 64 || K > 256 || K % 64) {
        set_error("tfla_selftest_gemm: bad arguments");
        return TFLA_ERR_PARAMETER;
    }
    CUtensorMap ma{}, mb{}, mo{};
    bool ok = true;
    if (a_mode == 0) ok &= make_tmap_bf16(&ma, a, 128, K, 64, 128);
    else if (a_mode == 1) ok &= make_tmap_bf16(&ma, a, K, 128, 64, 64);
    else ok &= make_tmap_bf16(&ma, a, 128, 64, 64, 64);  // unused placeholder
    if (b_mode == 0) ok &= make_tmap_bf16(&mb, b, N, K, 64, N);
    else ok &= make_tmap_bf16(&mb, b, K, N, 64, 64);
    ok &= make_tmap_bf16(&mo, out_bf16, 128, N, 64, 128);
    if (!ok) return TFLA_ERR_CUDA;
    SelfTestArgs args{a_mode, b_mode, N, K, static_cast<const __nv_bfloat16*>(a), out};
    cudaFuncSetAttribute(selftest_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kSmemBytes);
    selftest_gemm_kernel<<<1, 192, kSmemBytes, static_cast<cudaStream_t>(stream)>>>(ma, mb, mo,
                                                                                   args);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string("selftest launch: ") + cudaGetErrorString(e));
        return TFLA_ERR_CUDA;
    }
    return TFLA_OK;
}
