// capi_internal.h -- declarations shared by the C-ABI translation units.
#pragma once
#include "tfla/tfla.h"

namespace tfla_host {
int validate_dims(const tfla_dims* d);
int validate_blocks(const tfla_dims* d, const tfla_blocks* b);
}  // namespace tfla_host
