// gemm_util.cuh — constants and epilogue helpers shared by the 1-CTA
// (bsgemm.cu) and CTA-pair (bsgemm2.cu) tcgen05 GEMM kernels.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/moe.h"
#include "act_code_table.h"
#include "sm100.cuh"

namespace moe {

using namespace sm100;

constexpr int BM = 128;
#ifndef MOE_BK
#define MOE_BK 64
#endif
constexpr int BK = MOE_BK;        // K per pipeline stage (64: 128B-swizzled K-major rows; 32: 64B-swizzled)
constexpr int KPB = 128 / BK;     // stages per 128 x 128 sparse block
constexpr int KSW = BK * 2;       // K-major row bytes = TMA / UMMA swizzle span
static_assert(BK == 32 || BK == 64, "BK must be 32 or 64");
#ifndef MOE_PAIR_EPW
#define MOE_PAIR_EPW 8
#endif
constexpr int NUM_EPI_WARPS = MOE_PAIR_EPW;       // CTA-pair kernels: NUM_EPI_WARPS / 4 per TMEM lane quarter
constexpr int NUM_THREADS = 64 + 32 * NUM_EPI_WARPS;
constexpr int A_BYTES = BM * BK * 2;
constexpr int EPI_COLS = 32;                      // epilogue chunk: 32 rows x 32 columns per warp
constexpr int EPI_BUF = 32 * EPI_COLS * 2;        // one warp's chunk, bf16, 64B-swizzled rows
constexpr int EPI_BYTES = NUM_EPI_WARPS * 2 * EPI_BUF;  // double buffered
constexpr int SMEM_LIMIT = 232448;                // 227 KB opt-in
constexpr int SMEM_FIXED = 1024 + 512;            // alignment slack + barriers
constexpr int kMaxRouterTopK = 8;

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
// Write 32 fp32 values as bf16 into half `hh` (columns 32hh..32hh+31) of this
// thread's 128-byte row in a 128B-swizzled [32 rows][128 B] staging buffer
// (TMA SWIZZLE_128B: 16-byte chunk j of row r at chunk j ^ (r & 7));
// conflict-free 16-byte stores.
__device__ __forceinline__ void stage_row_half128(uint8_t* buf, int lane, const float* v, int hh) {
  const uint32_t row = smem_u32(buf) + lane * 128;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int cj = 4 * hh + j;
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(row + ((cj ^ (lane & 7)) << 4)),
                 "r"(pack_bf16x2(v[8 * j + 0], v[8 * j + 1])), "r"(pack_bf16x2(v[8 * j + 2], v[8 * j + 3])),
                 "r"(pack_bf16x2(v[8 * j + 4], v[8 * j + 5])), "r"(pack_bf16x2(v[8 * j + 6], v[8 * j + 7]))
                 : "memory");
  }
}
// Read half `hh` (columns 32hh..32hh+31) of this thread's 128B-swizzled row
// (the layout stage_row_half128 writes and a SWIZZLE_128B TMA load leaves).
__device__ __forceinline__ void load_row_half128(const uint8_t* buf, int lane, float* f, int hh) {
  const uint32_t row = smem_u32(buf) + lane * 128;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int cj = 4 * hh + j;
    uint4 w;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                 : "r"(row + ((cj ^ (lane & 7)) << 4))
                 : "memory");
    unpack8(w, f + 8 * j);
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
// serves both; the forward saves g for the SDD^T epilogue). gelu runs on the
// packed fp32x2 pipe (FFMA2/FMUL2: half the issue slots, same fp32 rounding).
// MOE_TANH_F16X2=1 (experiment): the two tanh of a pair on one MUFU.TANH.F16x2
// (fp16 argument and result, rel. error ~2^-11 < the bf16 outputs' ulp)
#ifndef MOE_TANH_F16X2
#define MOE_TANH_F16X2 0
#endif
__device__ __forceinline__ float2 tanh2_fast(float2 u) {
#if MOE_TANH_F16X2
  const __half2 h = __floats2half2_rn(u.x, u.y);
  uint32_t r;
  asm("tanh.approx.f16x2 %0, %1;" : "=r"(r) : "r"(*reinterpret_cast<const uint32_t*>(&h)));
  return __half22float2(*reinterpret_cast<const __half2*>(&r));
#else
  return make_float2(tanh_fast(u.x), tanh_fast(u.y));
#endif
}
__device__ __forceinline__ void act_fwd_deriv32(int kind, float* v, float* g) {
  if (kind == MOE_ACT_GELU_TANH) {
    const float2 c0 = make_float2(0.7978845608028654f, 0.7978845608028654f);
    const float2 c1 = make_float2(0.7978845608028654f * 0.044715f, 0.7978845608028654f * 0.044715f);
    const float2 c3 = make_float2(0.7978845608028654f * 3.0f * 0.044715f, 0.7978845608028654f * 3.0f * 0.044715f);
    const float2 half = make_float2(0.5f, 0.5f), one = make_float2(1.f, 1.f);
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      const float2 x = make_float2(v[i], v[i + 1]);
      const float2 x2 = __fmul2_rn(x, x);
      const float2 u = __fmul2_rn(x, __ffma2_rn(c1, x2, c0));
      const float2 t = tanh2_fast(u);
      const float2 du = __ffma2_rn(c3, x2, c0);
      const float2 hx = __fmul2_rn(half, x);
      const float2 a = __ffma2_rn(hx, t, hx);
      const float2 omt2 = __ffma2_rn(make_float2(-t.x, -t.y), t, one);
      const float2 gd = __ffma2_rn(__fmul2_rn(hx, du), omt2, __ffma2_rn(half, t, half));
      v[i] = a.x;
      v[i + 1] = a.y;
      g[i] = gd.x;
      g[i + 1] = gd.y;
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
// v *= g over a 32-value chunk (packed fp32x2 multiplies).
__device__ __forceinline__ void mul32(float* v, const float* g) {
#pragma unroll
  for (int i = 0; i < 32; i += 2) {
    const float2 r = __fmul2_rn(make_float2(v[i], v[i + 1]), make_float2(g[i], g[i + 1]));
    v[i] = r.x;
    v[i + 1] = r.y;
  }
}
// ---- branch-coded activation (DESIGN reading R24) ----------------------------
// The forward saves only A = act(H) in bf16. gelu has two pre-images for
// A < 0 (either side of its minimum at kGeluXMin): the mantissa LSB of a
// negative A holds the branch (1: h < kGeluXMin), chosen as the nearest bf16
// with that parity (<= 1 ulp from a; the sign follows h, so an A that
// underflows to +0 for very negative h stays negative). A >= 0 is RNE bf16.
// relu needs no code (act' = A > 0). The SDD^T decodes act'(H) from A's 16 bits
// through kActCodeTable (act_code_table.h, staged in shared memory).
// Two coded bf16 values packed as a bf16x2 word (low half: element 0), branch-free:
// RNE where x >= 0; where x < 0 the truncated magnitude with the sign set, +1 if
// its LSB differs from the branch bit (|A| <= 0.17 there, so the +1 never
// carries out of its half).
__device__ __forceinline__ uint32_t code_bf16x2(float2 a, float2 x) {
  const uint32_t rne = pack_bf16x2(a.x, a.y);
  const uint32_t ax = __float_as_uint(a.x), ay = __float_as_uint(a.y);
  const uint32_t t = __byte_perm(ax, ay, 0x7632) | 0x80008000u;          // high halves, sign set
  const float2 d = __fadd2_rn(x, make_float2(-kGeluXMin, -kGeluXMin));  // < 0: left of the minimum
  // branch bits: the signs of d at bits 0 and 16 (bytes 3 of d.x, d.y to bytes 0 and 2)
  const uint32_t b = (__byte_perm(__float_as_uint(d.x), __float_as_uint(d.y), 0x0703) >> 7) & 0x00010001u;
  const uint32_t neg = t + ((t ^ b) & 0x00010001u);
  uint32_t m;  // 0xffff in each half whose x is negative (prmt sign replication of bytes 3 and 7)
  asm("prmt.b32 %0, %1, %2, 0xffbb;" : "=r"(m) : "r"(__float_as_uint(x.x)), "r"(__float_as_uint(x.y)));
  return (neg & m) | (rne & ~m);
}
// v <- act(v) (gelu, relu) and w[i/2] <- the bf16x2 words of the coded A (gelu:
// branch-coded; relu: RNE). Same fp32 arithmetic as act_fwd.
__device__ __forceinline__ void act_fwd_code32(int kind, float* v, uint32_t* w) {
  if (kind == MOE_ACT_GELU_TANH) {
    const float2 c0 = make_float2(0.7978845608028654f, 0.7978845608028654f);
    const float2 c1 = make_float2(0.7978845608028654f * 0.044715f, 0.7978845608028654f * 0.044715f);
    const float2 half = make_float2(0.5f, 0.5f);
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      const float2 x = make_float2(v[i], v[i + 1]);
      const float2 x2 = __fmul2_rn(x, x);
      const float2 u = __fmul2_rn(x, __ffma2_rn(c1, x2, c0));
      const float2 t = make_float2(tanh_fast(u.x), tanh_fast(u.y));
      const float2 hx = __fmul2_rn(half, x);
      const float2 a = __ffma2_rn(hx, t, hx);
      w[i / 2] = code_bf16x2(a, x);
      v[i] = a.x;
      v[i + 1] = a.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = kind == MOE_ACT_RELU ? fmaxf(v[i], 0.f) : v[i];
#pragma unroll
    for (int i = 0; i < 32; i += 2) w[i / 2] = pack_bf16x2(v[i], v[i + 1]);
  }
}
// Table indices of two coded keys (a bf16x2 word), branch-free: each key is
// clamped to its sign's key range (negative keys keep their branch LSB at the
// low end) and rebased; positive keys index [0, kActCodeNPos), negative keys
// [kActCodeNPos, kActCodeN).
__device__ __forceinline__ uint32_t act_code_idx2(uint32_t w) {
  constexpr uint32_t P_LO = (uint32_t)kActCodeELo << 7, P_HI = ((uint32_t)kActCodeEHiPos << 7) | 0x7fu;
  constexpr uint32_t N_LO = 0x8000u | P_LO, N_HI = 0x8000u | ((uint32_t)kActCodeEHiNeg << 7) | 0x7fu;
  const uint32_t sm = (w >> 15) & 0x00010001u;                            // 1 per negative key
  const uint32_t lo = (P_LO * 0x00010001u) | (sm << 15) | (w & sm);
  const uint32_t hi = P_HI * 0x00010001u + sm * (N_HI - P_HI);
  const uint32_t c = __vminu2(__vmaxu2(w, lo), hi);
  const uint32_t base = P_LO * 0x00010001u + sm * (N_LO - (uint32_t)kActCodeNPos - P_LO);
  return c - base;
}
// v *= act'(H) decoded from the 16 bf16x2 words w of coded A (32 values);
// tab_smem: the fp32 decode table in shared memory.
__device__ __forceinline__ void act_code_mul32(int kind, float* v, const uint32_t* w, uint32_t tab_smem) {
  if (kind == MOE_ACT_GELU_TANH) {
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      const uint32_t idx = act_code_idx2(w[i / 2]);
      float g0, g1;
      asm volatile("ld.shared.f32 %0, [%1];" : "=f"(g0) : "r"(tab_smem + 4 * (idx & 0xffffu)));
      asm volatile("ld.shared.f32 %0, [%1];" : "=f"(g1) : "r"(tab_smem + 4 * (idx >> 16)));
      const float2 r = __fmul2_rn(make_float2(v[i], v[i + 1]), make_float2(g0, g1));
      v[i] = r.x;
      v[i + 1] = r.y;
    }
  } else if (kind == MOE_ACT_RELU) {
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      const uint32_t lo = w[i / 2] & 0xffffu, hi = w[i / 2] >> 16;
      v[i] = (lo != 0u && lo < 0x8000u) ? v[i] : 0.f;
      v[i + 1] = (hi != 0u && hi < 0x8000u) ? v[i + 1] : 0.f;
    }
  }
}
// the decode table (fp16 bits) in global memory; the SDD^T kernels expand it
// to fp32 in shared memory (all threads, before the block's first barrier)
static __device__ __align__(16) const uint16_t g_act_code_tab[kActCodeN] = MOE_ACT_CODE_TABLE_INIT;
constexpr int ACT_CODE_BYTES = kActCodeN * 4;
__device__ __forceinline__ void act_code_table_to_smem(uint8_t* dst, const uint16_t* src) {
  float* d = reinterpret_cast<float*>(dst);
  for (int i = threadIdx.x; i < kActCodeN; i += blockDim.x) d[i] = __half2float(__ushort_as_half(__ldg(src + i)));
}

// Raw 16 bf16x2 words of half `hh` of this thread's 128B-swizzled row.
__device__ __forceinline__ void load_row_half128_raw(const uint8_t* buf, int lane, uint32_t* w, int hh) {
  const uint32_t row = smem_u32(buf) + lane * 128;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int cj = 4 * hh + j;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(w[4 * j]), "=r"(w[4 * j + 1]), "=r"(w[4 * j + 2]), "=r"(w[4 * j + 3])
                 : "r"(row + ((cj ^ (lane & 7)) << 4))
                 : "memory");
  }
}
// Raw 16 bf16x2 words of this thread's 64B-swizzled staging row.
__device__ __forceinline__ void load_row_raw(const uint8_t* buf, int lane, uint32_t* w) {
  const uint32_t row = smem_u32(buf) + lane * 64;
#pragma unroll
  for (int j = 0; j < 4; ++j)
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(w[4 * j]), "=r"(w[4 * j + 1]), "=r"(w[4 * j + 2]), "=r"(w[4 * j + 3])
                 : "r"(row + swz64(j, lane))
                 : "memory");
}
// Stage 16 bf16x2 words (32 values) as half `hh` of a 128B-swizzled row / as a 64B-swizzled row.
__device__ __forceinline__ void stage_row_half128_raw(uint8_t* buf, int lane, const uint32_t* w, int hh) {
  const uint32_t row = smem_u32(buf) + lane * 128;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int cj = 4 * hh + j;
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(row + ((cj ^ (lane & 7)) << 4)), "r"(w[4 * j]),
                 "r"(w[4 * j + 1]), "r"(w[4 * j + 2]), "r"(w[4 * j + 3])
                 : "memory");
  }
}
__device__ __forceinline__ void stage_row_raw(uint8_t* buf, int lane, const uint32_t* w) {
  const uint32_t row = smem_u32(buf) + lane * 64;
#pragma unroll
  for (int j = 0; j < 4; ++j)
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(row + swz64(j, lane)), "r"(w[4 * j]),
                 "r"(w[4 * j + 1]), "r"(w[4 * j + 2]), "r"(w[4 * j + 3])
                 : "memory");
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
