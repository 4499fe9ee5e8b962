// gemm_util.cuh — constants and epilogue helpers shared by the 1-CTA
// (bsgemm.cu) and CTA-pair (bsgemm2.cu) tcgen05 GEMM kernels.
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/moe.h"
#include "sm100.cuh"

namespace moe {

using namespace sm100;

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int NUM_EPI_WARPS = 8;                  // 2 per TMEM lane quarter (column halves)
constexpr int NUM_THREADS = 64 + 32 * NUM_EPI_WARPS;
constexpr int A_BYTES = BM * BK * 2;
constexpr int EPI_COLS = 32;                      // epilogue chunk: 32 rows x 32 columns per warp
constexpr int EPI_BUF = 32 * EPI_COLS * 2;        // one warp's chunk, bf16, 64B-swizzled rows
constexpr int EPI_BYTES = NUM_EPI_WARPS * 2 * EPI_BUF;  // double buffered
constexpr int SMEM_LIMIT = 232448;                // 227 KB opt-in
constexpr int SMEM_FIXED = 1024 + 512;            // alignment slack + barriers
constexpr int kMaxRouterTopK = 8;
constexpr int kPrefetch = 0;  // L2 prefetch distance in K-steps (0: off; measured slower at 8)

// tanh on the SFU (MUFU.TANH, max rel. error ~2^-11, below the bf16 output ulp)
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// gelu, tanh approximation (reading R2): 0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3)))
__device__ __forceinline__ float act_fwd(int kind, float x) {
  if (kind == MOE_ACT_GELU_TANH) {
    const float x2 = x * x;
    const float u = x * fmaf(0.7978845608028654f * 0.044715f, x2, 0.7978845608028654f);
    const float hx = 0.5f * x;
    return fmaf(hx, tanh_fast(u), hx);
  }
  if (kind == MOE_ACT_RELU) return x > 0.f ? x : 0.f;
  return x;
}
__device__ __forceinline__ float act_grad(int kind, float x) {
  if (kind == MOE_ACT_GELU_TANH) {
    const float x2 = x * x;
    const float u = x * fmaf(0.7978845608028654f * 0.044715f, x2, 0.7978845608028654f);
    const float t = tanh_fast(u);
    const float du = fmaf(0.7978845608028654f * 3.0f * 0.044715f, x2, 0.7978845608028654f);
    return fmaf(0.5f * x * du, fmaf(-t, t, 1.0f), 0.5f * (1.0f + t));
  }
  if (kind == MOE_ACT_RELU) return x > 0.f ? 1.f : 0.f;
  return 1.f;
}

__device__ __forceinline__ void unpack8(const uint4& w, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 v = __bfloat1622float2(h[i]);
    f[2 * i] = v.x;
    f[2 * i + 1] = v.y;
  }
}

// 64B swizzle (TMA SWIZZLE_64B): 16-byte chunk j of row r lives at chunk j ^ ((r >> 1) & 3).
__device__ __forceinline__ int swz64(int j, int row) { return (j ^ ((row >> 1) & 3)) << 4; }

// Write 32 fp32 values of this thread's row as bf16 into a 64B-swizzled
// [32 rows][64 B] staging buffer (row = lane): conflict-free 16-byte stores.
// Explicit st.shared (a generic store would force a full MEMBAR before the
// async-proxy fence).
__device__ __forceinline__ void stage_row(uint8_t* buf, int lane, const float* v) {
  const uint32_t row = smem_u32(buf) + lane * 64;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(row + swz64(j, lane)),
                 "r"(pack_bf16x2(v[8 * j + 0], v[8 * j + 1])), "r"(pack_bf16x2(v[8 * j + 2], v[8 * j + 3])),
                 "r"(pack_bf16x2(v[8 * j + 4], v[8 * j + 5])), "r"(pack_bf16x2(v[8 * j + 6], v[8 * j + 7]))
                 : "memory");
  }
}
// Read this thread's 32 bf16 values back from a 64B-swizzled staging row.
__device__ __forceinline__ void load_row(const uint8_t* buf, int lane, float* f) {
  const uint32_t row = smem_u32(buf) + lane * 64;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint4 w;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                 : "r"(row + swz64(j, lane))
                 : "memory");
    unpack8(w, f + 8 * j);
  }
}

// Activation over a 32-value chunk with the kind hoisted out of the element
// loop (independent elements -> the SFU latency is overlapped).
__device__ __forceinline__ void act_fwd32(int kind, float* v) {
  if (kind == MOE_ACT_GELU_TANH) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = act_fwd(MOE_ACT_GELU_TANH, v[i]);
  } else if (kind == MOE_ACT_RELU) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = act_fwd(MOE_ACT_RELU, v[i]);
  }
}
// v <- act(v) and g <- act'(v) over a 32-value chunk (one tanh per element
// serves both; the forward saves g for the SDD^T epilogue).
__device__ __forceinline__ void act_fwd_deriv32(int kind, float* v, float* g) {
  if (kind == MOE_ACT_GELU_TANH) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float x = v[i];
      const float x2 = x * x;
      const float u = x * fmaf(0.7978845608028654f * 0.044715f, x2, 0.7978845608028654f);
      const float t = tanh_fast(u);
      const float du = fmaf(0.7978845608028654f * 3.0f * 0.044715f, x2, 0.7978845608028654f);
      const float hx = 0.5f * x;
      v[i] = fmaf(hx, t, hx);
      g[i] = fmaf(hx * du, fmaf(-t, t, 1.0f), fmaf(0.5f, t, 0.5f));
    }
  } else if (kind == MOE_ACT_RELU) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      g[i] = v[i] > 0.f ? 1.f : 0.f;
      v[i] = v[i] > 0.f ? v[i] : 0.f;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i) g[i] = 1.f;
  }
}
// v *= act'(h) over a 32-value chunk.
__device__ __forceinline__ void act_grad_mul32(int kind, float* v, const float* h) {
  if (kind == MOE_ACT_GELU_TANH) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] *= act_grad(MOE_ACT_GELU_TANH, h[i]);
  } else if (kind == MOE_ACT_RELU) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] *= act_grad(MOE_ACT_RELU, h[i]);
  }
}

}  // namespace moe
