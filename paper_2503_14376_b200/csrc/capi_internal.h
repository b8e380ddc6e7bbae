// capi_internal.h -- declarations shared by the C-ABI translation units.
#pragma once
#include "tfla/tfla.h"

#include <cstdint>
#include <initializer_list>

namespace tfla_host {
int validate_dims(const tfla_dims* d);
int validate_blocks(const tfla_dims* d, const tfla_blocks* b);
// Every device tensor is read / written by TMA or 16-byte vector accesses:
// non-NULL pointers must be 16-byte aligned (ParameterError otherwise).
int check_aligned(std::initializer_list<const void*> ptrs, const char* where);
}  // namespace tfla_host
