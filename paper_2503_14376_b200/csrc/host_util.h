// host_util.h -- host-side helpers shared by the C-ABI translation units:
// TMA tensor-map encoding (driver entry point fetched through the runtime, so
// the library does not link libcuda directly) and error bookkeeping.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <string>

namespace tfla_host {

// true when the environment variable is set to a non-empty value other than "0"
bool env_flag(const char* name);

// SM count of the current device (cached per device)
int num_sms();
// Persistent grid size: min(n_tiles, #SMs), lowered to the nearest value
// coprime to `period` (>= #SMs / 2) so static tile striding mixes tile kinds.
int coprime_grid(long n_tiles, int period);

// Opt the kernel into `bytes` of dynamic shared memory on the current device
// (once per kernel and device; thread-safe).
void ensure_smem_attr(const void* func, int bytes);

// Thread-local last error message behind tfla_last_error().
void set_error(const std::string& msg);
const char* last_error();

// Row-major bf16 2D tensor [rows][cols]; the TMA box is {box_cols, box_rows}
// with the 128-byte swizzle (box_cols * 2 must be <= 128).
bool make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols,
                    uint32_t box_cols, uint32_t box_rows);

// Row-major bf16 3D tensor [outer][rows][cols] (e.g. [B*NH][T][d]); box
// {box_cols, box_rows, 1}. Rows beyond `rows` are zero-filled on load and
// clipped on store, so tiles never bleed into the next head.
bool make_tmap_bf16_3d(CUtensorMap* map, const void* ptr, uint64_t outer, uint64_t rows,
                       uint64_t cols, uint32_t box_cols, uint32_t box_rows);

// Same for fp32 [rows][cols] (box_cols * 4 <= 128).
// 32-column boxes with the 64-byte swizzle (32-column state-scan tiles)
bool make_tmap_bf16_3d_sw64(CUtensorMap* map, const void* ptr, uint64_t outer, uint64_t rows,
                            uint64_t cols, uint32_t box_rows);
bool make_tmap_f32(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols,
                   uint32_t box_cols, uint32_t box_rows);

}  // namespace tfla_host

// ---------------------------------------------------------------- profiling
// Optional per-kernel CUDA-event timing (tfla_profile_*): when enabled, every
// launch site records an event pair on the launching stream.
namespace tfla_host {

enum ProfId {
    P_GATES_FWD = 0,
    P_SCAN_FWD,
    P_FWD_PARALLEL,
    P_GATES_BWD,
    P_STATES_BF16,
    P_SCAN_BWD,
    P_BWD_DQ,
    P_BWD_DK,
    P_BWD_DV,
    P_ASSEMBLE,
    P_BWD_FUSED,
    P_QN,
    P_FWD_FUSED,
    P_COUNT
};

const char* prof_name(int id);

class ProfScope {
  public:
    ProfScope(int id, cudaStream_t st, int launches);
    ~ProfScope();

  private:
    int id_;
    cudaStream_t st_;
    cudaEvent_t start_ = nullptr;
};

void prof_enable(bool on);
int prof_read(double* ms, int64_t* launches, int n);

}  // namespace tfla_host
