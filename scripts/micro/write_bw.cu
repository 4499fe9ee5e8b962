// HBM write-only bandwidth by store form (16-byte st.global, 32-byte
// st.global.v8, cudaMemset), 298 MB (the SDD's two bf16 outputs at MoE-XS) and
// 149 MB (one output); CUDA events, best of 10. The denominators behind the
// SDD's write-bound floor.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 write_bw.cu -o write_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void w16(uint4* __restrict__ dst, size_t n) {
  const size_t nt = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += nt)
    dst[i] = make_uint4((unsigned)i, 1u, 2u, 3u);
}

__global__ void w32(uint32_t* __restrict__ dst, size_t n32) {
  const size_t nt = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n32; i += nt) {
    uint32_t* p = dst + i * 8;
    asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "r"((unsigned)i) : "memory");
  }
}

// Each warp writes whole contiguous 4 KB chunks (like a TMA store box).
__global__ void wchunk(uint4* __restrict__ dst, size_t nchunks) {
  const int lane = threadIdx.x & 31;
  const size_t w = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5, nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  for (size_t c = w; c < nchunks; c += nw) {
    uint4* p = dst + c * 256;
#pragma unroll
    for (int j = 0; j < 8; ++j) p[j * 32 + lane] = make_uint4((unsigned)c, j, lane, 0);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t sizes[2] = {298ull << 20, 149ull << 20};
  uint8_t* buf;
  cudaMalloc(&buf, sizes[0]);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (size_t bytes : sizes) {
    for (int form = 0; form < 4; ++form) {
      for (int occ : {4, 8}) {
        if (form == 3 && occ == 8) continue;
        float best = 1e9f;
        for (int r = 0; r < 12; ++r) {
          cudaEventRecord(a);
          if (form == 0) w16<<<sms * occ, 256>>>((uint4*)buf, bytes / 16);
          else if (form == 1) w32<<<sms * occ, 256>>>((uint32_t*)buf, bytes / 32);
          else if (form == 2) wchunk<<<sms * occ, 256>>>((uint4*)buf, bytes / 4096);
          else cudaMemsetAsync(buf, 0, bytes);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (r >= 2 && ms < best) best = ms;
        }
        const char* nm[4] = {"st.v4 (16 B)", "st.v8 (32 B)", "4 KB chunk/warp", "cudaMemset"};
        printf("%4zu MB %-16s ctas=%d x 256: %7.1f us  %6.0f GB/s\n", bytes >> 20, nm[form], sms * occ, best * 1e3,
               bytes / (best * 1e-3) / 1e9);
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
