// Semantics check of TMA tile::gather4 on sm_100a: 4 arbitrary rows of a 2-D
// bf16 tensor into shared memory, SWIZZLE_128B, with an out-of-range row index.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void g4(const __grid_constant__ CUtensorMap map, int r0, int r1, int r2, int r3, int col, uint16_t* out) {
  __shared__ __align__(1024) uint16_t buf[4 * 64];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(4 * 64 * 2));
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5, %6}], [%7];" ::"r"(su32(buf)),
        "l"(&map), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(&bar))
        : "memory");
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0,1,0,p;\n}"
                   : "=r"(done) : "r"(su32(&bar)) : "memory");
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4 * 64; i += blockDim.x) out[i] = buf[i];
}

int main() {
  const int rows = 1000, cols = 256;
  uint16_t* h = new uint16_t[rows * cols];
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) h[r * cols + c] = (uint16_t)((r * 7 + c) & 0x7fff) | 1;  // nonzero
  uint16_t *d, *o;
  cudaMalloc(&d, rows * cols * 2);
  cudaMalloc(&o, 4 * 64 * 2);
  cudaMemcpy(d, h, rows * cols * 2, cudaMemcpyHostToDevice);
  for (int sw = 0; sw < 2; ++sw) {
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE,
                                        sw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode box {64,1} swizzle %d: %d\n", sw, (int)r);
    int rr[4] = {5, 999, 1000 /* out of range */, 17};
    g4<<<1, 128>>>(map, rr[0], rr[1], rr[2], rr[3], 64, o);
    cudaError_t e = cudaDeviceSynchronize();
    printf("launch: %s\n", cudaGetErrorString(e));
    uint16_t out[256];
    cudaMemcpy(out, o, 512, cudaMemcpyDeviceToHost);
    for (int q = 0; q < 4; ++q) {
      int ok = 0, zero = 0;
      for (int c = 0; c < 64; ++c) {
        // position of element (q, c) in smem: row q, 16B chunk c/8 swizzled with row (q & 7)
        const int chunk = sw ? ((c / 8) ^ (q & 7)) : (c / 8);
        const uint16_t got = out[q * 64 + chunk * 8 + (c % 8)];
        const uint16_t want = rr[q] < rows ? h[rr[q] * cols + 64 + c] : 0;
        ok += got == want;
        zero += got == 0;
      }
      printf("  row slot %d (src row %d): %d/64 match (%d zeros)\n", q, rr[q], ok, zero);
    }
  }
  return 0;
}
