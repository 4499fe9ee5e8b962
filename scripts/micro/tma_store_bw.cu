// Microbenchmark: TMA (cp.async.bulk.tensor) store throughput from per-warp
// smem staging buffers vs. box shape and stores in flight, all SMs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tma_store_bw.cu -o tma_store_bw -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int DEPTH>
__global__ void __launch_bounds__(32 * 16, 1) store_kernel(const __grid_constant__ CUtensorMap map, int box_rows,
                                                           int box_bytes, int iters, int warps, int rows_total,
                                                           int fence, int chunks, int inner_box) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp >= warps) return;
  uint8_t* buf = smem + warp * DEPTH * box_bytes;
  const int gw = blockIdx.x * warps + warp;
  const int nw = gridDim.x * warps;
  int slot = 0;
  for (int it = 0; it < iters; ++it) {
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(DEPTH - 1) : "memory");
    __syncwarp();
    uint4* b = reinterpret_cast<uint4*>(buf + slot * box_bytes);
    for (int i = lane; i < box_bytes / 16; i += 32) b[i] = make_uint4(it, i, gw, 7);
    if (fence) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      const long long id = (long long)it * nw + gw;
      const int row = (int)(((id / chunks) * box_rows) % rows_total);
      const int col = (int)(id % chunks) * inner_box;
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&map),
                   "r"(smem_u32(buf + slot * box_bytes)), "r"(col), "r"(row)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    slot = (slot + 1) % DEPTH;
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const long long rows_total = 1 << 18;  // rows of the destination
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  struct Shape { int inner_elems, rows; CUtensorMapSwizzle sw; const char* name; int chunks = 1; };
  Shape shapes[] = {{32, 32, CU_TENSOR_MAP_SWIZZLE_64B, "32x32 sw64 in 256B rows (4 chunks)", 4},
                    {64, 32, CU_TENSOR_MAP_SWIZZLE_128B, "32x64 sw128 in 256B rows (2 chunks)", 2},
                    {32, 32, CU_TENSOR_MAP_SWIZZLE_64B, "32x32 sw64 in 1024B rows (16 chunks)", 16},
                    {64, 32, CU_TENSOR_MAP_SWIZZLE_128B, "32x64 sw128 in 1024B rows (8 chunks)", 8},{32, 32, CU_TENSOR_MAP_SWIZZLE_64B, "32x32 sw64 (2KB, 64B rows)"},
                    {64, 32, CU_TENSOR_MAP_SWIZZLE_128B, "32x64 sw128 (4KB, 128B rows)"},
                    {64, 64, CU_TENSOR_MAP_SWIZZLE_128B, "64x64 sw128 (8KB)"},
                    {64, 128, CU_TENSOR_MAP_SWIZZLE_128B, "128x64 sw128 (16KB)"},
                    {128, 32, CU_TENSOR_MAP_SWIZZLE_NONE, "32x128 noswz (8KB, 256B rows)"},
                    {256, 32, CU_TENSOR_MAP_SWIZZLE_NONE, "32x256 noswz (16KB, 512B rows)"}};
  for (auto& s : shapes) {
    const long long inner = (long long)s.inner_elems * s.chunks;  // destination row = chunks boxes wide
    void* dst;
    cudaMalloc(&dst, rows_total * inner * 2);
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows_total};
    cuuint64_t strides[1] = {(cuuint64_t)inner * 2};
    cuuint32_t box[2] = {(cuuint32_t)s.inner_elems, (cuuint32_t)s.rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dst, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, s.sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d for %s\n", r, s.name); continue; }
    const int box_bytes = s.inner_elems * s.rows * 2;
    for (int warps : {4, 8, 16}) {
      for (int depth : {1, 2, 4}) {
        const int smem = warps * depth * box_bytes;
        if (smem > 200 * 1024) continue;
        const long long total_bytes = 2LL << 30;
        const int iters = (int)(total_bytes / box_bytes / (sms * warps));
        auto launch = [&](int fence) {
          if (depth == 1) { cudaFuncSetAttribute(store_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            store_kernel<1><<<sms, 512, smem>>>(map, s.rows, box_bytes, iters, warps, (int)rows_total, fence, s.chunks, s.inner_elems); }
          if (depth == 2) { cudaFuncSetAttribute(store_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            store_kernel<2><<<sms, 512, smem>>>(map, s.rows, box_bytes, iters, warps, (int)rows_total, fence, s.chunks, s.inner_elems); }
          if (depth == 4) { cudaFuncSetAttribute(store_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            store_kernel<4><<<sms, 512, smem>>>(map, s.rows, box_bytes, iters, warps, (int)rows_total, fence, s.chunks, s.inner_elems); }
        };
        launch(1);
        cudaEvent_t a, b;
        cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        launch(1);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        cudaError_t e = cudaGetLastError();
        const double bytes = (double)iters * sms * warps * box_bytes;
        printf("%-32s warps=%2d depth=%d : %7.1f GB/s  (%.3f ms) %s\n", s.name, warps, depth, bytes / ms / 1e6, ms,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
    }
    cudaFree(dst);
  }
  return 0;
}
