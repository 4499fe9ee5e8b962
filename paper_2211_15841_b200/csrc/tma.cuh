#pragma once
#include <cuda.h>

#include "../../include/moe.h"

namespace moe {
// 2-D bf16 tensor map, SWIZZLE_128B, element coordinates (inner, outer).
// row_elems: row pitch in elements. box_inner * 2 bytes must equal the
// swizzle span (64 elements for 128 B, 32 for 64 B).
moe_status make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_elems,
                          uint32_t box_inner, uint32_t box_outer, const char* what, int swizzle_bytes = 128);
// MN-major operand map: the row-major [outer, inner] matrix viewed as 3-D
// {64, outer, inner/64} (strides: row pitch, 128 B) with box {64, 64, nchunk}:
// one TMA box fills nchunk MN-chunks of 64 K-rows ([chunk][64][128 B] in smem,
// SWIZZLE_128B). inner must be a multiple of 64.
moe_status make_tmap_bf16_mn(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_elems,
                             uint32_t nchunk, const char* what);
// fp32 [outer, inner] map with 32 x 32 boxes, SWIZZLE_128B (router logits store).
moe_status make_tmap_f32(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_elems,
                         const char* what);
// Epilogue store / H-prefetch maps: 32 x 32 boxes, 64 B swizzle.
inline moe_status make_tmap_epi(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                                uint64_t row_elems, const char* what) {
  return make_tmap_bf16(map, base, inner, outer, row_elems, 32, 32, what, 64);
}
// Wide epilogue store maps: 64 x 32 boxes (4 KB: 32 rows of 128 B), 128 B
// swizzle — twice the bytes per TMA store of make_tmap_epi (TMA store
// throughput grows with the box: scripts/micro/tma_store_bw.cu).
inline moe_status make_tmap_epi_wide(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                                     uint64_t row_elems, const char* what) {
  return make_tmap_bf16(map, base, inner, outer, row_elems, 64, 32, what, 128);
}
// Tall epilogue store maps: 64 x 64 boxes (8 KB: 64 rows of 128 B), 128 B
// swizzle — two warps of adjacent TMEM lane quarters stage one box together.
inline moe_status make_tmap_epi_tall(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                                     uint64_t row_elems, const char* what) {
  return make_tmap_bf16(map, base, inner, outer, row_elems, 64, 64, what, 128);
}
}  // namespace moe
