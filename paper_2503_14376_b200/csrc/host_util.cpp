#include "host_util.h"

#include <mutex>

namespace tfla_host {

namespace {
thread_local std::string g_last_error;

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

bool encode(CUtensorMap* map, CUtensorMapDataType dt, uint32_t esize, const void* ptr,
            uint64_t rows, uint64_t cols, uint32_t box_cols, uint32_t box_rows,
            uint64_t outer = 0) {
    auto fn = get_encode_fn();
    if (!fn) {
        set_error("cuTensorMapEncodeTiled unavailable (no CUDA driver)");
        return false;
    }
    cuuint64_t gdim[3] = {cols, rows, outer};
    cuuint64_t gstride[2] = {cols * esize, cols * rows * esize};
    cuuint32_t box[3] = {box_cols, box_rows, 1};
    cuuint32_t estride[3] = {1, 1, 1};
    const cuuint32_t rank = outer ? 3 : 2;
    CUresult r = fn(map, dt, rank, const_cast<void*>(ptr), gdim, gstride, box, estride,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (code " + std::to_string(int(r)) + ")");
        return false;
    }
    return true;
}
}  // namespace

void set_error(const std::string& msg) { g_last_error = msg; }
const char* last_error() { return g_last_error.c_str(); }

bool make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols,
                    uint32_t box_cols, uint32_t box_rows) {
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ptr, rows, cols, box_cols, box_rows);
}

bool make_tmap_bf16_3d(CUtensorMap* map, const void* ptr, uint64_t outer, uint64_t rows,
                       uint64_t cols, uint32_t box_cols, uint32_t box_rows) {
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ptr, rows, cols, box_cols, box_rows,
                  outer);
}

bool make_tmap_f32(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols,
                   uint32_t box_cols, uint32_t box_rows) {
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, ptr, rows, cols, box_cols, box_rows);
}

}  // namespace tfla_host
