// Calibration: the tcgen05 GEMM engine (bsgemm.cu) in DENSE mode on plain
// GEMMs, to separate mainloop efficiency from the block-sparse walks.
// C[M,N] (bf16) = A[M,K] . B[N,K]^T, both K-major.  Links the library objects.
// Build (repo root): nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2211_15841_b200/csrc \
//   scripts/micro/gemm_calib.cu build/*.o -o /tmp/gemm_calib -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "bsgemm.cuh"
#include "tma.cuh"

using namespace moe;

int main(int argc, char** argv) {
  struct Sh { int M, N, K, bn; };
  Sh shapes[] = {{8192, 8192, 8192, 256}, {8192, 8192, 2048, 256}, {8192, 8192, 512, 256},
                 {16384, 2048, 512, 256}, {36864, 512, 2048, 256}, {8192, 8192, 8192, 128}};
  for (auto s : shapes) {
    __nv_bfloat16 *A, *B, *C;
    cudaMalloc(&A, (size_t)s.M * s.K * 2);
    cudaMalloc(&B, (size_t)s.N * s.K * 2);
    cudaMalloc(&C, (size_t)s.M * s.N * 2);
    cudaMemset(A, 0x3c, (size_t)s.M * s.K * 2);
    cudaMemset(B, 0x3b, (size_t)s.N * s.K * 2);
    GemmLaunch L{};
    L.name = "calib";
    L.mode = DENSE;
    L.bn = s.bn;
    L.a_mn = false;
    L.b_mn = false;
    L.p.m_tiles = s.M / 128;
    L.p.n_tiles = s.N / s.bn;
    L.p.splits = 1;
    L.p.k_iters_total = L.p.kiters_split = s.K / 64;
    L.p.epi = EPI_STORE;
    L.p.rows_valid = s.M;
    L.max_tiles = L.p.m_tiles * L.p.n_tiles;
    make_tmap_bf16(&L.ta, A, s.K, s.M, s.K, 64, 128, "A");
    make_tmap_bf16(&L.tb, B, s.K, s.N, s.K, 64, s.bn, "B");
    make_tmap_epi(&L.tc, C, s.N, s.M, s.N, "C");
    L.td = L.tc;
    for (int i = 0; i < 3; ++i) gemm_launch(L, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int reps = 10;
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) gemm_launch(L, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= reps;
    const double fl = 2.0 * s.M * s.N * s.K;
    const double by = 2.0 * ((double)s.M * s.K + (double)s.N * s.K + (double)s.M * s.N);
    printf("M=%6d N=%5d K=%5d BN=%d : %8.3f us  %7.1f TFLOP/s  %6.1f GB/s(min bytes)  %s\n", s.M, s.N, s.K, s.bn,
           ms * 1e3, fl / ms / 1e9, by / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    cudaFree(A);
    cudaFree(B);
    cudaFree(C);
  }
  return 0;
}
