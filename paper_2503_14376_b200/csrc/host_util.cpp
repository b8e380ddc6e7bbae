#include "host_util.h"
#include "workspace.h"
#include <cstring>
#include <vector>

#include <cstdlib>
#include <mutex>
#include <set>
#include <utility>

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
            uint64_t outer = 0, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
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
                    CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (code " + std::to_string(int(r)) + ")");
        return false;
    }
    return true;
}
}  // namespace

void set_error(const std::string& msg) { g_last_error = msg; }

int num_sms() {  // of the current device, cached per device
    static std::mutex mu;
    static int cache[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    int& n = cache[dev & 63];
    if (!n) {
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

void ensure_smem_attr(const void* func, int bytes) {
    // cudaFuncSetAttribute applies to the current device only: record
    // (kernel, device) pairs so every device of a multi-GPU process gets it
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    if (done.insert({func, dev}).second)
        cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

bool env_flag(const char* name) {
    const char* v = std::getenv(name);
    return v && *v && std::string(v) != "0";
}
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

bool make_tmap_bf16_3d_sw64(CUtensorMap* map, const void* ptr, uint64_t outer, uint64_t rows,
                            uint64_t cols, uint32_t box_rows) {
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ptr, rows, cols, 32, box_rows, outer,
                  CU_TENSOR_MAP_SWIZZLE_64B);
}

bool make_tmap_f32(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols,
                   uint32_t box_cols, uint32_t box_rows) {
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, ptr, rows, cols, box_cols, box_rows);
}

}  // namespace tfla_host

// ---------------------------------------------------------------- profiling
#include <vector>

namespace tfla_host {
namespace {
struct ProfRec {
    int id;
    cudaEvent_t a, b;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof;
int64_t g_launch[P_COUNT] = {};
const char* kNames[P_COUNT] = {"gates_fwd",    "state_scan_fwd", "fwd_parallel", "gates_bwd",
                               "states_to_bf16", "state_scan_bwd", "bwd_dq",     "bwd_dk",
                               "bwd_dv",       "assemble",       "bwd_fused",      "qn",
                               "fwd_fused"};
}  // namespace

int coprime_grid(long n_tiles, int period) {
    int g = num_sms();
    if (n_tiles <= g) return static_cast<int>(n_tiles);
    auto gcd = [](int a, int b) {
        while (b) {
            const int t = a % b;
            a = b;
            b = t;
        }
        return a;
    };
    int c = g;
    while (period > 1 && c > g / 2 && gcd(c, period) != 1) --c;
    return c > g / 2 ? c : g;
}

const char* prof_name(int id) { return (id >= 0 && id < P_COUNT) ? kNames[id] : ""; }

ProfScope::ProfScope(int id, cudaStream_t st, int launches) : id_(id), st_(st) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (!g_prof_on) return;
    g_launch[id] += launches;
    cudaEventCreate(&start_);
    cudaEventRecord(start_, st_);
}

ProfScope::~ProfScope() {
    if (!start_) return;
    cudaEvent_t end;
    cudaEventCreate(&end);
    cudaEventRecord(end, st_);
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof.push_back({id_, start_, end});
}

void prof_enable(bool on) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof_on = on;
}

int prof_read(double* ms, int64_t* launches, int n) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (int i = 0; i < n && i < P_COUNT; ++i) {
        ms[i] = 0.0;
        launches[i] = g_launch[i];
    }
    for (auto& r : g_prof) {
        cudaEventSynchronize(r.b);
        float t = 0.f;
        cudaEventElapsedTime(&t, r.a, r.b);
        if (r.id < n) ms[r.id] += t;
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    g_prof.clear();
    for (int i = 0; i < P_COUNT; ++i) g_launch[i] = 0;
    return P_COUNT;
}

}  // namespace tfla_host

// ---------------------------------------------------------------- stabiliser audit
namespace tfla_host {
namespace {
std::mutex g_stab_mu;
std::vector<tfla_k::StabCounters*> g_stab;  // per device, nullptr = off
bool g_stab_env_read = false;
}  // namespace

static int cur_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}

static tfla_k::StabCounters* stab_enable_locked(int dev) {
    if (static_cast<int>(g_stab.size()) <= dev) g_stab.resize(dev + 1, nullptr);
    if (!g_stab[dev]) {
        void* p = nullptr;
        if (cudaMalloc(&p, sizeof(tfla_k::StabCounters)) != cudaSuccess) return nullptr;
        cudaMemset(p, 0, sizeof(tfla_k::StabCounters));
        cudaDeviceSynchronize();
        g_stab[dev] = static_cast<tfla_k::StabCounters*>(p);
    }
    return g_stab[dev];
}

tfla_k::StabCounters* stab_counters() {
    std::lock_guard<std::mutex> lk(g_stab_mu);
    const int dev = cur_device();
    if (!g_stab_env_read) {
        g_stab_env_read = true;
        if (env_flag("TFLA_STAB_CHECK")) stab_enable_locked(dev);
    }
    return dev < static_cast<int>(g_stab.size()) ? g_stab[dev] : nullptr;
}

}  // namespace tfla_host

extern "C" {
int tfla_stab_enable(int on) {
    std::lock_guard<std::mutex> lk(tfla_host::g_stab_mu);
    tfla_host::g_stab_env_read = true;
    const int dev = tfla_host::cur_device();
    if (on) {
        if (!tfla_host::stab_enable_locked(dev)) {
            tfla_host::set_error("tfla_stab_enable: cudaMalloc failed");
            return TFLA_ERR_CUDA;
        }
    } else if (dev < static_cast<int>(tfla_host::g_stab.size()) && tfla_host::g_stab[dev]) {
        cudaDeviceSynchronize();
        cudaFree(tfla_host::g_stab[dev]);
        tfla_host::g_stab[dev] = nullptr;
    }
    return TFLA_OK;
}

int tfla_stab_read(int64_t* checks, int64_t* violations, double* max_arg) {
    std::lock_guard<std::mutex> lk(tfla_host::g_stab_mu);
    const int dev = tfla_host::cur_device();
    tfla_k::StabCounters h{};
    if (dev < static_cast<int>(tfla_host::g_stab.size()) && tfla_host::g_stab[dev]) {
        if (cudaDeviceSynchronize() != cudaSuccess ||
            cudaMemcpy(&h, tfla_host::g_stab[dev], sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) {
            tfla_host::set_error("tfla_stab_read: device error");
            return TFLA_ERR_CUDA;
        }
        cudaMemset(tfla_host::g_stab[dev], 0, sizeof(h));
        cudaDeviceSynchronize();
    }
    if (checks) *checks = static_cast<int64_t>(h.checks);
    if (violations) *violations = static_cast<int64_t>(h.violations);
    if (max_arg) {
        float f;
        memcpy(&f, &h.max_bits, sizeof(f));
        *max_arg = static_cast<double>(f) / 1.4426950408889634;  // natural-log units, like exp_guarded
    }
    return TFLA_OK;
}

int tfla_profile_enable(int on) {
    tfla_host::prof_enable(on != 0);
    return 0;
}
int tfla_profile_read(double* ms, int64_t* launches, int n) {
    return tfla_host::prof_read(ms, launches, n);
}
const char* tfla_profile_name(int id) { return tfla_host::prof_name(id); }
}
