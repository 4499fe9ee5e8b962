#pragma once
#include <cuda.h>

#include "../../include/moe.h"

namespace moe {
// 2-D bf16 tensor map, SWIZZLE_128B, element coordinates (inner, outer).
// row_elems: row pitch in elements. box_inner must be 64 (128 B swizzle span).
moe_status make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_elems,
                          uint32_t box_inner, uint32_t box_outer, const char* what);
}  // namespace moe
