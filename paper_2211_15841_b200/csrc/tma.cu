// tma.cu — host-side creation of TMA tensor maps (cuTensorMapEncodeTiled,
// resolved through the runtime's driver entry point so the library does not
// link libcuda directly).
#include <cuda.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "tma.cuh"
#include "gemm_util.cuh"

namespace moe {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

moe_status make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_elems,
                          uint32_t box_inner, uint32_t box_outer, const char* what, int swizzle_bytes) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return set_error(MOE_ECUDA, "cuTensorMapEncodeTiled unavailable (driver entry point)");
  if (!base) return set_error(MOE_EINVAL, "%s: NULL pointer", what);
  if (reinterpret_cast<uintptr_t>(base) % 16)
    return set_error(MOE_EINVAL, "%s: pointer must be 16-byte aligned for TMA", what);
  if ((row_elems * 2) % 16) return set_error(MOE_ESHAPE, "%s: row pitch must be a multiple of 16 bytes", what);
  if (outer == 0) outer = 1;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_elems * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(MOE_ECUDA, "%s: cuTensorMapEncodeTiled failed (%d) dims=[%llu,%llu] box=[%u,%u]", what, (int)r,
                     (unsigned long long)inner, (unsigned long long)outer, box_inner, box_outer);
  return MOE_OK;
}

moe_status make_tmap_f32(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_elems,
                         const char* what) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return set_error(MOE_ECUDA, "cuTensorMapEncodeTiled unavailable (driver entry point)");
  if (!base) return set_error(MOE_EINVAL, "%s: NULL pointer", what);
  if (reinterpret_cast<uintptr_t>(base) % 16)
    return set_error(MOE_EINVAL, "%s: pointer must be 16-byte aligned for TMA", what);
  if ((row_elems * 4) % 16) return set_error(MOE_ESHAPE, "%s: row pitch must be a multiple of 16 bytes", what);
  if (outer == 0) outer = 1;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_elems * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(MOE_ECUDA, "%s: cuTensorMapEncodeTiled (f32) failed (%d)", what, (int)r);
  return MOE_OK;
}

moe_status make_tmap_bf16_mn(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_elems,
                             uint32_t nchunk, const char* what) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return set_error(MOE_ECUDA, "cuTensorMapEncodeTiled unavailable (driver entry point)");
  if (!base) return set_error(MOE_EINVAL, "%s: NULL pointer", what);
  if (reinterpret_cast<uintptr_t>(base) % 16)
    return set_error(MOE_EINVAL, "%s: pointer must be 16-byte aligned for TMA", what);
  if (inner % 64) return set_error(MOE_ESHAPE, "%s: MN extent %llu must be a multiple of 64", what,
                                   (unsigned long long)inner);
  if (outer == 0) outer = 1;
  cuuint64_t dims[3] = {64, outer, inner / 64};
  cuuint64_t strides[2] = {row_elems * 2, 128};
  cuuint32_t box[3] = {64, (cuuint32_t)BK, nchunk};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(MOE_ECUDA, "%s: cuTensorMapEncodeTiled (3-D MN) failed (%d) dims=[64,%llu,%llu] box=[64,64,%u]",
                     what, (int)r, (unsigned long long)outer, (unsigned long long)(inner / 64), nchunk);
  return MOE_OK;
}

}  // namespace moe
