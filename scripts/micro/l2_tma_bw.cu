// Microbenchmark: L2 -> SMEM delivery rate of TMA loads on all SMs.
// Modes: each CTA streams 16 KB boxes (128 rows x 64 bf16, SWIZZLE_128B) from an
// L2-resident buffer into an S-stage ring (a consumer warp only waits/frees).
//   distinct : every CTA reads different boxes
//   shared G : groups of G CTAs read the same box sequence at the same time
//   mcast C  : clusters of C CTAs; each loads 1/C of the box and multicasts it
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 l2_tma_bw.cu -o l2bw -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  uint32_t done;
  do {
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}"
                 : "=r"(done) : "r"(su32(b)), "r"(ph) : "memory");
  } while (!done);
}
__device__ __forceinline__ void mbar_wait_test(uint64_t* b, uint32_t ph) {
  uint32_t done;
  do {
    asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}"
                 : "=r"(done) : "r"(su32(b)), "r"(ph) : "memory");
  } while (!done);
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* b, uint32_t cta) {
  // arrive on CTA `cta`'s copy of barrier b
  uint32_t a = su32(b), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(cta));
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
__device__ __forceinline__ uint32_t ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

constexpr int S = 32;  // max ring stages

// mode 0 distinct, 1 shared(G), 2 multicast cluster C (launched with cluster dims C)
struct Maps { CUtensorMap m[4]; };
template <int C>
__global__ void __launch_bounds__(128, 1) bw_kernel(const __grid_constant__ Maps maps, int nmaps, int iters, int nboxes,
                                                  int mode, int G, int BOX, int NS, int rows_per_box) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* buf = (uint8_t*)(((uintptr_t)smem + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[S], empty[S];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = C > 1 ? ctarank() : 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], C);  // every CTA of the cluster must free a stage before it is refilled
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  
  if (C > 1) cluster_sync(); else __syncthreads();
  const int b = blockIdx.x;
  mode &= 3;
  if (G == 900) {
    // every lane of warp 0 owns one stage and issues its own boxes
    if (warp == 0 && lane < NS) {
      const int s = lane;
      for (int i = 0; i < iters / NS; ++i) {
        if (i > 0) mbar_wait(&full[s], (i - 1) & 1);
        const int box = (int)(((long long)(b * NS + lane) * iters + i) % nboxes);
        mbar_expect(&full[s], BOX);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
            ::"r"(su32(buf + s * BOX)), "l"(&maps.m[0]), "r"(0), "r"(box * rows_per_box), "r"(su32(&full[s])) : "memory");
      }
      mbar_wait(&full[s], ((iters / NS) - 1) & 1);
    }
  } else if (G == 555 || G == 556 || G == 557) {
    const int P = G - 553;  // 2, 3, 4 producer warps
    if (warp < P && lane == 0) {
      const int ns = NS / P;
      for (int i = 0; i < iters / P; ++i) {
        const int s = warp * ns + i % ns;
        const uint32_t ph = (i / ns) & 1;
        if (i >= ns) mbar_wait(&full[s], ph ^ 1);
        const int box = (int)(((long long)(b * P + warp) * iters + i) % nboxes);
        mbar_expect(&full[s], BOX);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
            ::"r"(su32(buf + s * BOX)), "l"(&maps.m[0]), "r"(0), "r"(box * rows_per_box), "r"(su32(&full[s])) : "memory");
      }
      for (int s = warp * ns; s < (warp + 1) * ns; ++s) mbar_wait(&full[s], ((iters / P) / ns - 1) & 1);
    }
  } else if (G >= 600 && G < 700) {
    // P = G - 600 producer warps (stage s issued by warp s % P), one consumer
    // warp (warp 3) freeing every stage on all CTAs of the cluster; with C > 1
    // each CTA loads 1/C of the box and multicasts it
    const int P = G - 600;
    if (warp < P && lane == 0) {
      for (int i = 0; i < iters; ++i) {
        const int s = i % NS;
        if (s % P != warp) continue;
        const uint32_t ph = (i / NS) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        const int box = mode == 0 ? (int)(((long long)b * iters + i) % nboxes)
                                  : (int)(((long long)(b / C) * 7919 + i) % nboxes);
        mbar_expect(&full[s], BOX);
        if (C == 1) {
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
              ::"r"(su32(buf + s * BOX)), "l"(&maps.m[0]), "r"(0), "r"(box * rows_per_box), "r"(su32(&full[s])) : "memory");
        } else {
          const int rows = rows_per_box / C;
          const uint16_t mask = (uint16_t)((1u << C) - 1);
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, "
              "{%2, %3}], [%4], %5;"
              ::"r"(su32(buf + s * BOX + rank * rows * 128)), "l"(&maps.m[0]), "r"(0),
              "r"(box * rows_per_box + (int)rank * rows), "r"(su32(&full[s])), "h"(mask) : "memory");
        }
      }
    } else if (warp == 3 && lane == 0) {
      for (int i = 0; i < iters; ++i) {
        const int s = i % NS;
        mbar_wait(&full[s], (i / NS) & 1);
        if (C == 1) mbar_arrive(&empty[s]);
        else for (int c = 0; c < C; ++c) mbar_arrive_cluster(&empty[s], c);
      }
    }
  } else if (warp == 0 && lane == 0) {
    for (int i = 0; i < iters; ++i) {
      const int s = i % NS;
      const uint32_t ph = (i / NS) & 1;
      if (G == 777) { if (i >= NS) mbar_wait(&full[s], ph ^ 1); }
      else mbar_wait(&empty[s], ph ^ 1);
      int box;
      if (mode == 0) box = (int)(((long long)b * iters + i) % nboxes);
      else if (mode == 1) box = (int)(((long long)(b / G) * 7919 + i) % nboxes);
      else box = (int)(((long long)(b / C) * 7919 + i) % nboxes);
      mbar_expect(&full[s], BOX);
      const CUtensorMap& map = maps.m[i % nmaps];
      if (C == 1) {
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
            ::"r"(su32(buf + s * BOX)), "l"(&map), "r"(0), "r"(box * rows_per_box), "r"(su32(&full[s])) : "memory");
      } else {
        const int rows = rows_per_box / C;
        const uint16_t mask = (uint16_t)((1u << C) - 1);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, "
            "{%2, %3}], [%4], %5;"
            ::"r"(su32(buf + s * BOX + rank * rows * 128)), "l"(&map), "r"(0), "r"(box * rows_per_box + (int)rank * rows),
            "r"(su32(&full[s])), "h"(mask) : "memory");
      }
    }
  } else if (warp == 1 && lane == 0 && G != 777) {
    for (int i = 0; i < iters; ++i) {
      const int s = i % NS;
      mbar_wait(&full[s], (i / NS) & 1);
      if (C == 1) mbar_arrive(&empty[s]);
      else for (int c = 0; c < C; ++c) mbar_arrive_cluster(&empty[s], c);
    }
  }
  __syncwarp();
  if (C > 1) cluster_sync();
}

#ifndef MODES_MAIN
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long bytes = 32LL << 20;
  void* src;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  cudaEvent_t a, e;
  cudaEventCreate(&a);
  cudaEventCreate(&e);
  for (int rows : {32, 64}) {
    const int inner = 64;
    const int BOX = rows * inner * 2;
    const int nboxes = (int)(bytes / BOX);
    Maps maps;
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)nboxes * rows};
    cuuint64_t strides[1] = {(cuuint64_t)inner * 2};
    cuuint32_t box[2] = {(cuuint32_t)inner, (cuuint32_t)rows}, es[2] = {1, 1};
    cuTensorMapEncodeTiled(&maps.m[0], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int ring_kb = 128;
    const int NS = ring_kb * 1024 / BOX;
    const int smem = ring_kb * 1024 + 1024;
    cudaFuncSetAttribute(bw_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int G : {777, 557, 900}) {
      const int grid = sms;
      const int iters = (int)((1LL << 30) / ((long long)grid * BOX)) / 16 * 16;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        bw_kernel<1><<<grid, 128, smem>>>(maps, 1, iters, nboxes, 0, G, BOX, NS, rows);
        cudaEventRecord(e);
        cudaEventSynchronize(e);
      }
      float ms;
      cudaEventElapsedTime(&ms, a, e);
      const double delivered = (double)grid * iters * BOX;
      printf("box %5d B ring %3d KB producers %d : %8.1f GB/s total (%.1f GB/s per CTA) %s\n", BOX, ring_kb,
             G == 777 ? 1 : (G == 900 ? 32 : G - 553), delivered / ms / 1e6, delivered / ms / 1e6 / grid,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
#else
// MODES_MAIN: distinct vs shared (G CTAs read the same box sequence) vs
// multicast (cluster of C CTAs, each issues 1/C of the box to all): is the
// ~98 GB/s per SM TMA delivery limit on the SM side or the L2 side?
template <int C>
static double run(const Maps& maps, int sms, int mode, int G, int BOX, int NS, int rows, int nboxes, int smem) {
  cudaFuncSetAttribute(bw_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int grid = sms / C * C;
  const int iters = (int)((1LL << 30) / ((long long)grid * BOX)) / 16 * 16;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaEvent_t a, e;
  cudaEventCreate(&a);
  cudaEventCreate(&e);
  float ms = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, bw_kernel<C>, maps, 1, iters, nboxes, mode, G, BOX, NS, rows);
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    cudaEventElapsedTime(&ms, a, e);
  }
  const double delivered = (double)grid * iters * BOX;  // bytes landed in shared memory
  printf("mode %d G %d C %d: %8.1f GB/s delivered to smem (%.1f GB/s per CTA) %s\n", mode, G, C, delivered / ms / 1e6,
         delivered / ms / 1e6 / grid, cudaGetErrorString(cudaGetLastError()));
  return delivered / ms / 1e6;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long bytes = 32LL << 20;
  void* src;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  const int rows = 128, inner = 64, BOX = rows * inner * 2;
  const int nboxes = (int)(bytes / BOX);
  Maps maps;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)nboxes * rows};
  cuuint64_t strides[1] = {(cuuint64_t)inner * 2};
  cuuint32_t box[2] = {(cuuint32_t)inner, (cuuint32_t)rows}, es[2] = {1, 1};
  cuTensorMapEncodeTiled(&maps.m[0], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint32_t box2[2] = {(cuuint32_t)inner, (cuuint32_t)(rows / 2)}, box4[2] = {(cuuint32_t)inner, (cuuint32_t)(rows / 4)};
  Maps m2 = maps, m4 = maps;
  cuTensorMapEncodeTiled(&m2.m[0], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box2, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuTensorMapEncodeTiled(&m4.m[0], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box4, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int ring = 128 * 1024, NS = ring / BOX, smem = ring + 1024;
  // 3 producer warps + a consumer: distinct vs cluster multicast
  for (int P : {1, 2, 3}) {
    run<1>(maps, sms, 0, 600 + P, BOX, NS, rows, nboxes, smem);
    run<2>(m2, sms, 2, 600 + P, BOX, NS, rows, nboxes, smem);
    run<4>(m4, sms, 2, 600 + P, BOX, NS, rows, nboxes, smem);
  }
  run<1>(maps, sms, 0, 1, BOX, NS, rows, nboxes, smem);
  run<1>(maps, sms, 1, 2, BOX, NS, rows, nboxes, smem);
  run<1>(maps, sms, 1, 4, BOX, NS, rows, nboxes, smem);
  run<2>(m2, sms, 2, 1, BOX, NS, rows, nboxes, smem);
  run<4>(m4, sms, 2, 1, BOX, NS, rows, nboxes, smem);
  return 0;
}
#endif
