// capi.cpp -- C-ABI entry points: validation (mirroring Dims::validate_chunked,
// core.cpp:9-21, and BlockConfig::validate / pick_default, tiled.cpp:21-39),
// workspace sizing, and error reporting. The forward / backward drivers live
// in tfla_fwd.cu / tfla_bwd.cu.
#include <cstdio>
#include <string>

#include "capi_internal.h"
#include "host_util.h"
#include "tfla/tfla.h"

using tfla_host::set_error;

namespace {

int64_t largest_divisor_up_to(int64_t n, int64_t cap) {
    for (int64_t d = n < cap ? n : cap; d >= 1; --d)
        if (n % d == 0) return d;
    return 1;
}

}  // namespace

namespace tfla_host {

int validate_dims(const tfla_dims* d) {
    if (!d) {
        set_error("dims is NULL");
        return TFLA_ERR_PARAMETER;
    }
    // Dims::validate (core.cpp:9-16)
    if (d->T < 1) return set_error("T must be >= 1"), TFLA_ERR_GEOMETRY;
    if (d->L < 1) return set_error("L must be >= 1"), TFLA_ERR_GEOMETRY;
    if (d->d_qk < 1) return set_error("d_qk must be >= 1"), TFLA_ERR_GEOMETRY;
    if (d->d_hv < 1) return set_error("d_hv must be >= 1"), TFLA_ERR_GEOMETRY;
    if (d->n_head < 1) return set_error("n_head must be >= 1"), TFLA_ERR_GEOMETRY;
    if (d->n_batch < 1) return set_error("n_batch must be >= 1"), TFLA_ERR_GEOMETRY;
    // Dims::validate_chunked (core.cpp:18-21)
    if (d->T % d->L != 0) return set_error("T not divisible by L"), TFLA_ERR_GEOMETRY;
    // sm_100a kernel constraints (tcgen05 M=128 tiles, 64-wide SW128 atoms)
    if (d->L % 64 != 0 || d->L > 1024)
        return set_error("B200 kernels need L a multiple of 64 in [64, 1024]"), TFLA_ERR_GEOMETRY;
    if (d->d_qk % 64 != 0 || d->d_qk > 512)
        return set_error("B200 kernels need d_qk a multiple of 64, <= 512"), TFLA_ERR_GEOMETRY;
    if (d->d_hv % 64 != 0 || d->d_hv > 4096)
        return set_error("B200 kernels need d_hv a multiple of 64, <= 4096"), TFLA_ERR_GEOMETRY;
    // bound every factor before forming a product (no int64 overflow), then the
    // products: (b, h) slices index a grid y / z dimension, rows fit in int32
    if (d->n_head > 65535 || d->n_batch > 65535 || d->n_head * d->n_batch > 65535)
        return set_error("B*NH must stay <= 65535 per call (shard larger batches)"), TFLA_ERR_GEOMETRY;
    if (d->T >= (int64_t(1) << 31) || d->T >= ((int64_t(1) << 31) / (d->n_head * d->n_batch)) + 1 ||
        d->T * d->n_head * d->n_batch >= (int64_t(1) << 31))
        return set_error("B*NH*T must stay below 2^31 rows"), TFLA_ERR_GEOMETRY;
    return TFLA_OK;
}

int check_aligned(std::initializer_list<const void*> ptrs, const char* where) {
    for (const void* p : ptrs)
        if (p && (reinterpret_cast<uintptr_t>(p) & 15u))
            return set_error(std::string(where) + ": device pointers must be 16-byte aligned"),
                   TFLA_ERR_PARAMETER;
    return TFLA_OK;
}

int validate_blocks(const tfla_dims* d, const tfla_blocks* b) {
    if (!b) {
        set_error("blocks is NULL");
        return TFLA_ERR_PARAMETER;
    }
    // BlockConfig::validate (tiled.cpp:21-30)
    if (b->b_lhq < 1 || b->b_lkv < 1 || b->b_dqk < 1 || b->b_dhv < 1)
        return set_error("block sizes must be >= 1"), TFLA_ERR_GEOMETRY;
    if (b->b_lhq < b->b_lkv) return set_error("b_lhq must be >= b_lkv"), TFLA_ERR_GEOMETRY;
    if (d->L % b->b_lhq != 0 || d->L % b->b_lkv != 0)
        return set_error("sequence block sizes must divide L"), TFLA_ERR_GEOMETRY;
    if (b->b_lhq % b->b_lkv != 0) return set_error("b_lkv must divide b_lhq"), TFLA_ERR_GEOMETRY;
    if (d->d_qk % b->b_dqk != 0) return set_error("b_dqk must divide d_qk"), TFLA_ERR_GEOMETRY;
    if (d->d_hv % b->b_dhv != 0) return set_error("b_dhv must divide d_hv"), TFLA_ERR_GEOMETRY;
    return TFLA_OK;
}

}  // namespace tfla_host

extern "C" {

int tfla_validate_dims(const tfla_dims* dims) {
    set_error("");
    return tfla_host::validate_dims(dims);
}

int tfla_validate_blocks(const tfla_dims* dims, const tfla_blocks* blocks) {
    set_error("");
    if (!dims) return set_error("dims is NULL"), TFLA_ERR_PARAMETER;
    return tfla_host::validate_blocks(dims, blocks);
}

int tfla_pick_default_blocks(const tfla_dims* dims, tfla_blocks* out) {
    set_error("");
    if (!dims || !out) return set_error("NULL argument"), TFLA_ERR_PARAMETER;
    // BlockConfig::pick_default (tiled.cpp:32-39)
    out->b_lhq = largest_divisor_up_to(dims->L, 32);
    out->b_lkv = largest_divisor_up_to(out->b_lhq, 8);
    out->b_dqk = largest_divisor_up_to(dims->d_qk, 16);
    out->b_dhv = largest_divisor_up_to(dims->d_hv, 32);
    return TFLA_OK;
}

// detail::kv_block_count / block_needs_mask (tiled.cpp:43-49): the TFLA
// Alg. 1 kv-loop bound of query block i_lq and the literal (over-inclusive by
// one block, test_tiled.cpp:52-57) mask predicate of kv block i_kv (1-based).
// The sm_100a kernels tile the chunk in 128 x 128 blocks and mask inside the
// diagonal tile; these are the reference's host-side block bookkeeping.
int64_t tfla_kv_block_count(int64_t i_lq, const tfla_blocks* blocks) {
    if (!blocks || blocks->b_lkv < 1 || blocks->b_lhq < 1 || i_lq < 0) return -1;
    return ((i_lq + 1) * blocks->b_lhq) / blocks->b_lkv;
}

int tfla_block_needs_mask(int64_t i_kv_1based, int64_t i_lq, const tfla_blocks* blocks) {
    if (!blocks || blocks->b_lkv < 1 || blocks->b_lhq < 1) return -1;
    return i_kv_1based * blocks->b_lkv >= i_lq * blocks->b_lhq ? 1 : 0;
}

const char* tfla_last_error(void) { return tfla_host::last_error(); }

const char* tfla_version(void) { return "tfla_b200 0.1 (sm_100a, tcgen05/TMA)"; }

}  // extern "C"
