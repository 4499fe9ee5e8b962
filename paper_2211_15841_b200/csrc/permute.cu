// permute.cu — padded permutation kernels ("we pad each group of tokens
// with zeros to the nearest multiple of 128 and fuse this operation into
// custom permutation kernels"), the weighted un-permutation (P:279-280,
// §2.4) and their backward passes, plus the unpadded expert-order
// permutation used for expert-parallel dispatch.
//
// All kernels are HBM-bandwidth-bound row copies. Design for latency: every
// warp owns ROWS rows at once (ROWS = 8 / VEC, VEC = 16-byte vectors per lane
// per row), loads all their indices with one coalesced load + shuffles, issues
// all row loads, then all stores — 8 x 16 B in flight per lane. Copies are
// input-driven (one index load per row); the zero pad rows of every expert
// group are written by a second phase of the same kernel. Grid = SMs x 8 CTAs
// of 8 warps, grid-stride, reading device-side sizes (no host sync).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <float.h>
#include <stdlib.h>

#include "common.cuh"
#include "permute.cuh"

namespace moe {

constexpr int kWarpsPerCta = 8;

__device__ __forceinline__ void bf16x8_to_f32(const uint4& w, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 v = __bfloat1622float2(h[i]);
    f[2 * i] = v.x;
    f[2 * i + 1] = v.y;
  }
}
__device__ __forceinline__ uint4 f32_to_bf16x8(const float* f) {
  uint4 w;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&w);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return w;
}

__device__ __forceinline__ int warp_global() { return (blockIdx.x * blockDim.x + threadIdx.x) >> 5; }
__device__ __forceinline__ int warps_total() { return (gridDim.x * blockDim.x) >> 5; }

// Zero the pad rows of every expert group: rows [start_e + c_e, start_e + pc_e).
template <int VEC>
__device__ void zero_pad_rows(uint4* __restrict__ dst, const int32_t* __restrict__ counts,
                              const int32_t* __restrict__ padded_bins, int E, int bs) {
  const int lane = threadIdx.x & 31;
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (int w = warp_global(); w < E * bs; w += warps_total()) {
    const int e = w / bs, j = w - e * bs;
    const int c = __ldg(counts + e);
    const int pc = ((c + bs - 1) / bs) * bs;
    if (j >= pc - c) continue;
    uint4* row = dst + (size_t)(__ldg(padded_bins + e) - pc + c + j) * VEC * 32;
#pragma unroll
    for (int u = 0; u < VEC; ++u) row[lane + 32 * u] = z;
  }
}

// dst[map[i]] = src[i / k] for i < R (rows of h = VEC*256 bf16); optional pad zeroing.
template <int VEC>
__global__ void __launch_bounds__(256) scatter_rows_kernel(const uint4* __restrict__ src, const int32_t* __restrict__ map,
                                                            uint4* __restrict__ dst, int R, int k,
                                                            const int32_t* __restrict__ counts,
                                                            const int32_t* __restrict__ padded_bins, int E, int bs) {
  pdl_trigger();
  pdl_wait();
  constexpr int ROWS = 8 / VEC;
  constexpr int RV = VEC * 32;  // uint4 per row
  const int lane = threadIdx.x & 31;
  for (int base = warp_global() * ROWS; base < R; base += warps_total() * ROWS) {
    const int my = base + lane;
    const int midx = (lane < ROWS && my < R) ? __ldg(map + my) : -1;
    uint4 v[ROWS][VEC];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      const int i = base + r;
      if (i < R) {
        const uint4* s = src + (size_t)(i / k) * RV;
#pragma unroll
        for (int u = 0; u < VEC; ++u) v[r][u] = __ldg(s + lane + 32 * u);
      }
    }
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      const int d = __shfl_sync(0xffffffffu, midx, r);
      if (base + r < R && d >= 0) {  // d < 0: assignment dropped by a capacity
        uint4* o = dst + (size_t)d * RV;
#pragma unroll
        for (int u = 0; u < VEC; ++u) o[lane + 32 * u] = v[r][u];
      }
    }
  }
  if (counts) zero_pad_rows<VEC>(dst, counts, padded_bins, E, bs);
}

// y[t] = sum_{j ascending} g[t,j] * rows[map[t*k+j]]   (fp32 accumulate, bf16 out)
template <int VEC>
__global__ void __launch_bounds__(256) combine_kernel(const uint4* __restrict__ rows, const int32_t* __restrict__ map,
                                                       const float* __restrict__ gates, uint4* __restrict__ y, int T,
                                                       int k) {
  pdl_trigger();
  pdl_wait();
  constexpr int ROWS = 8 / VEC;
  constexpr int RV = VEC * 32;
  const int lane = threadIdx.x & 31;
  for (int base = warp_global() * ROWS; base < T; base += warps_total() * ROWS) {
    float acc[ROWS][VEC][8];
#pragma unroll
    for (int r = 0; r < ROWS; ++r)
#pragma unroll
      for (int u = 0; u < VEC; ++u)
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[r][u][q] = 0.f;
    for (int j = 0; j < k; ++j) {
      const int t_l = base + lane;
      const bool lv = lane < ROWS && t_l < T;
      const int midx = lv ? __ldg(map + (size_t)t_l * k + j) : 0;
      const float g = (lv && gates) ? __ldg(gates + (size_t)t_l * k + j) : 1.0f;
      uint4 v[ROWS][VEC];
#pragma unroll
      for (int r = 0; r < ROWS; ++r) {
        const int m = __shfl_sync(0xffffffffu, midx, r);
        if (base + r < T && m >= 0) {
          const uint4* s = rows + (size_t)m * RV;
#pragma unroll
          for (int u = 0; u < VEC; ++u) v[r][u] = __ldg(s + lane + 32 * u);
        } else {  // a dropped slot (capacity) contributes zero
#pragma unroll
          for (int u = 0; u < VEC; ++u) v[r][u] = make_uint4(0u, 0u, 0u, 0u);
        }
      }
#pragma unroll
      for (int r = 0; r < ROWS; ++r) {
        const float gr = __shfl_sync(0xffffffffu, g, r);
        if (base + r < T) {
#pragma unroll
          for (int u = 0; u < VEC; ++u) {
            float f[8];
            bf16x8_to_f32(v[r][u], f);
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[r][u][q] = fmaf(gr, f[q], acc[r][u][q]);
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      if (base + r < T) {
        uint4* o = y + (size_t)(base + r) * RV;
#pragma unroll
        for (int u = 0; u < VEC; ++u) o[lane + 32 * u] = f32_to_bf16x8(acc[r][u]);
      }
    }
  }
}

// dy_rows[map[i]] = g_i * dy[t]; dgates[i] = <y_rows[map[i]], dy[t]>, i = t*k + j.
// Optionally fused router backward (P:98 softmax chain rule):
// dlogits[t,:] = p * (dp - <p,dp>), p = softmax(logits[t,:]), dp[e] = sum_{j: idx_j = e} dgates_j.
// Each warp owns TPW tokens at once: all index, gate, dy-row and logit loads
// are issued together, then the gathered y rows of every slot, so a warp keeps
// ~TPW*(2 + k) row loads in flight instead of a dependent chain per token.
template <int VEC, int TPW, int EQ>
__global__ void __launch_bounds__(256) scatter_bwd_kernel(
    const uint4* __restrict__ dy, const uint4* __restrict__ y_rows, const int32_t* __restrict__ map,
    const float* __restrict__ gates, uint4* __restrict__ dy_rows, float* __restrict__ dgates, int T, int k,
    const float* __restrict__ logits, const int32_t* __restrict__ expert_idx, int E,
    __nv_bfloat16* __restrict__ dlogits_bf16, float* __restrict__ dlogits_f32, const int32_t* __restrict__ counts,
    const int32_t* __restrict__ padded_bins, int bs, int renorm, const float* __restrict__ aux_c) {
  pdl_trigger();
  pdl_wait();
  constexpr int RV = VEC * 32;
  // EQ: logits per lane per token (E <= 32 * EQ)
  const int lane = threadIdx.x & 31;
  const bool want_dg = dgates != nullptr;
  const bool want_dl = logits && (dlogits_bf16 || dlogits_f32);
  const int EQn = (E + 31) / 32;
  for (int base = warp_global() * TPW; base < T; base += warps_total() * TPW) {
    // lane l < TPW*k holds slot (token base + l / k, j = l % k)
    const int tl = lane / k, jl = lane - tl * k;
    const bool sl = lane < TPW * k && base + tl < T;
    const int midx = sl ? __ldg(map + (size_t)(base + tl) * k + jl) : 0;
    const float gl = sl ? (gates ? __ldg(gates + (size_t)(base + tl) * k + jl) : 1.0f) : 0.f;
    const int eidx = (sl && want_dl) ? __ldg(expert_idx + (size_t)(base + tl) * k + jl) : -1;
    uint4 d[TPW][VEC];
#pragma unroll
    for (int r = 0; r < TPW; ++r)
      if (base + r < T) {
        const uint4* ds = dy + (size_t)(base + r) * RV;
#pragma unroll
        for (int u = 0; u < VEC; ++u) d[r][u] = __ldg(ds + lane + 32 * u);
      }
    float lv[TPW][EQ];
    if (want_dl) {
#pragma unroll
      for (int r = 0; r < TPW; ++r)
#pragma unroll
        for (int q = 0; q < EQ; ++q) {
          const int e = lane + 32 * q;
          lv[r][q] = (q < EQn && e < E && base + r < T) ? __ldg(logits + (size_t)(base + r) * E + e) : -FLT_MAX;
        }
    }
    float dg_lane = 0.f;  // lane l holds dgates of its slot
    for (int j = 0; j < k; ++j) {
      uint4 yv[TPW][VEC];
      int m[TPW];
      float g[TPW];
#pragma unroll
      for (int r = 0; r < TPW; ++r) {
        m[r] = __shfl_sync(0xffffffffu, midx, r * k + j);
        g[r] = __shfl_sync(0xffffffffu, gl, r * k + j);
        if (want_dg && base + r < T && m[r] >= 0) {
          const uint4* ys = y_rows + (size_t)m[r] * RV;
#pragma unroll
          for (int u = 0; u < VEC; ++u) yv[r][u] = __ldg(ys + lane + 32 * u);
        } else {
#pragma unroll
          for (int u = 0; u < VEC; ++u) yv[r][u] = make_uint4(0u, 0u, 0u, 0u);
        }
      }
#pragma unroll
      for (int r = 0; r < TPW; ++r) {
        if (base + r >= T) continue;
        uint4* o = dy_rows + (size_t)m[r] * RV;
        float dot = 0.f;
#pragma unroll
        for (int u = 0; u < VEC; ++u) {
          float f[8];
          bf16x8_to_f32(d[r][u], f);
          if (want_dg) {
            float fy[8];
            bf16x8_to_f32(yv[r][u], fy);
#pragma unroll
            for (int q = 0; q < 8; ++q) dot = fmaf(fy[q], f[q], dot);
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) f[q] *= g[r];
          if (m[r] >= 0) o[lane + 32 * u] = f32_to_bf16x8(f);  // dropped slot: no row, dgate 0
        }
        if (want_dg) {
#pragma unroll
          for (int o2 = 16; o2 > 0; o2 >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o2);
          if (lane == r * k + j) dg_lane = dot;
        }
      }
    }
    if (want_dg && sl) dgates[(size_t)(base + tl) * k + jl] = dg_lane;
    if (want_dl) {
#pragma unroll
      for (int r = 0; r < TPW; ++r) {
        if (base + r >= T) continue;  // warp-uniform
        float mx = -FLT_MAX;
#pragma unroll
        for (int q = 0; q < EQ; ++q) mx = fmaxf(mx, lv[r][q]);
#pragma unroll
        for (int o2 = 16; o2 > 0; o2 >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o2));
        float ssum = 0.f, pv[EQ], dpl[EQ];
#pragma unroll
        for (int q = 0; q < EQ; ++q) {
          pv[q] = (q < EQn && lane + 32 * q < E) ? __expf(lv[r][q] - mx) : 0.f;
          ssum += pv[q];
          dpl[q] = 0.f;
        }
#pragma unroll
        for (int o2 = 16; o2 > 0; o2 >>= 1) ssum += __shfl_xor_sync(0xffffffffu, ssum, o2);
        const float inv = 1.f / ssum;
        // renormalised gates g_j = p_j / S (NEXT-4): the gradient reaching p_j is
        // (dg_j - sum_i dg_i g_i) / S
        float rs = 1.f, gd = 0.f;
        if (renorm) {
          float sp = 0.f, gp = 0.f;
          for (int j = 0; j < k; ++j) {
            const int ejj = __shfl_sync(0xffffffffu, eidx, r * k + j);
            const float dgj = __shfl_sync(0xffffffffu, dg_lane, r * k + j);
#pragma unroll
            for (int q = 0; q < EQ; ++q)
              if (lane + 32 * q == ejj) {
                sp += pv[q] * inv;
                gp += pv[q] * inv * dgj;
              }
          }
#pragma unroll
          for (int o2 = 16; o2 > 0; o2 >>= 1) {
            sp += __shfl_xor_sync(0xffffffffu, sp, o2);
            gp += __shfl_xor_sync(0xffffffffu, gp, o2);
          }
          rs = 1.f / sp;
          gd = gp * rs;
        }
        float pdp = 0.f;
        for (int j = 0; j < k; ++j) {  // warp-uniform
          const int ejj = __shfl_sync(0xffffffffu, eidx, r * k + j);
          float dgj = __shfl_sync(0xffffffffu, dg_lane, r * k + j);
          if (renorm) dgj = (dgj - gd) * rs;
#pragma unroll
          for (int q = 0; q < EQ; ++q)
            if (lane + 32 * q == ejj) {
              dpl[q] += dgj;
              pdp += pv[q] * inv * dgj;
            }
        }
        if (aux_c) {  // + the auxiliary loss's d/dp (every expert)
#pragma unroll
          for (int q = 0; q < EQ; ++q) {
            const int e = lane + 32 * q;
            if (q < EQn && e < E) {
              const float c = __ldg(aux_c + e);
              dpl[q] += c;
              pdp += pv[q] * inv * c;
            }
          }
        }
#pragma unroll
        for (int o2 = 16; o2 > 0; o2 >>= 1) pdp += __shfl_xor_sync(0xffffffffu, pdp, o2);
#pragma unroll
        for (int q = 0; q < EQ; ++q) {
          const int e = lane + 32 * q;
          if (q < EQn && e < E) {
            const float dl = pv[q] * inv * (dpl[q] - pdp);
            if (dlogits_bf16)
              dlogits_bf16[(size_t)(base + r) * E + e] = __float2bfloat16_rn(dl);
            else
              dlogits_f32[(size_t)(base + r) * E + e] = dl;
          }
        }
      }
    }
  }
  if (counts) zero_pad_rows<VEC>(dy_rows, counts, padded_bins, E, bs);
}

template <int VEC>
__global__ void __launch_bounds__(256) zero_pad_kernel(uint4* __restrict__ dst, const int32_t* __restrict__ counts,
                                                       const int32_t* __restrict__ padded_bins, int E, int bs) {
  pdl_trigger();
  pdl_wait();  // counts / padded_bins come from the topology kernel before it
  zero_pad_rows<VEC>(dst, counts, padded_bins, E, bs);
}

static int row_grid() { return moe_device_sm_count() * 8; }
// One wave of the kernel's resident CTAs (the row kernels are grid-stride
// loops: a second, partial wave of CTAs only adds a launch tail; e.g. the
// padded gather holds 5 CTAs per SM at 48 registers, not 8). MOE_ROW_GRID=8:
// the fixed 8 CTAs per SM.
template <typename K>
static int row_grid_for(K* kern) {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("MOE_ROW_GRID");
    env = e ? atoi(e) : 0;
  }
  if (env > 0) return moe_device_sm_count() * env;
  static int per_sm = 0;  // per kernel instantiation (the occupancy depends on the kernel only)
  if (per_sm == 0) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, 32 * kWarpsPerCta, 0) != cudaSuccess || n < 1) {
      cudaGetLastError();
      n = 8;
    }
    per_sm = n < 8 ? n : 8;
  }
  return moe_device_sm_count() * per_sm;
}

static moe_status check_rows(const moe_config* cfg, const moe_topology_t* topo, const char* name) {
  MOE_TRY(moe_check_config(cfg));
  MOE_TRY(check_topo(topo));
  if (cfg->hidden % 256 || cfg->hidden > 2048)
    return set_error(MOE_EUNSUPPORTED, "%s: hidden=%lld must be a multiple of 256 and <= 2048", name,
                     (long long)cfg->hidden);
  return MOE_OK;
}

#define MOE_VEC_CASE(V, NAME, KERNEL, ...) \
  case V: MOE_LAUNCH(NAME, KERNEL<V>, dim3(row_grid_for(KERNEL<V>)), dim3(32 * kWarpsPerCta), 0, s, __VA_ARGS__); break;
#define MOE_VEC_DISPATCH(VEC_EXPR, NAME, KERNEL, ...)  \
  switch (VEC_EXPR) {                                  \
    MOE_VEC_CASE(1, NAME, KERNEL, __VA_ARGS__)         \
    MOE_VEC_CASE(2, NAME, KERNEL, __VA_ARGS__)         \
    MOE_VEC_CASE(3, NAME, KERNEL, __VA_ARGS__)         \
    MOE_VEC_CASE(4, NAME, KERNEL, __VA_ARGS__)         \
    MOE_VEC_CASE(5, NAME, KERNEL, __VA_ARGS__)         \
    MOE_VEC_CASE(6, NAME, KERNEL, __VA_ARGS__)         \
    MOE_VEC_CASE(7, NAME, KERNEL, __VA_ARGS__)         \
    default: MOE_LAUNCH(NAME, KERNEL<8>, dim3(row_grid_for(KERNEL<8>)), dim3(32 * kWarpsPerCta), 0, s, __VA_ARGS__); break; \
  }

struct SbwdArgs {
  const uint4* dy;
  const uint4* y_rows;
  const int32_t* map;
  const float* gates;
  uint4* dy_rows;
  float* dgates;
  int T, k;
  const float* logits;
  const int32_t* expert_idx;
  int E;
  __nv_bfloat16* dl16;
  float* dl32;
  const int32_t* counts;
  const int32_t* pbins;
  int bs;
  int renorm;
  const float* aux_c;
};

template <int V, int TPW>
static moe_status sbwd_launch(const SbwdArgs& a, cudaStream_t s) {
  if (a.E <= 64)
    MOE_LAUNCH("scatter_bwd", (scatter_bwd_kernel<V, TPW, 2>), dim3(row_grid_for(scatter_bwd_kernel<V, TPW, 2>)),
               dim3(32 * kWarpsPerCta), 0, s, a.dy,
               a.y_rows, a.map, a.gates, a.dy_rows, a.dgates, a.T, a.k, a.logits, a.expert_idx, a.E, a.dl16, a.dl32,
               a.counts, a.pbins, a.bs, a.renorm, a.aux_c);
  else
    MOE_LAUNCH("scatter_bwd", (scatter_bwd_kernel<V, TPW, 8>), dim3(row_grid_for(scatter_bwd_kernel<V, TPW, 8>)),
               dim3(32 * kWarpsPerCta), 0, s, a.dy,
               a.y_rows, a.map, a.gates, a.dy_rows, a.dgates, a.T, a.k, a.logits, a.expert_idx, a.E, a.dl16, a.dl32,
               a.counts, a.pbins, a.bs, a.renorm, a.aux_c);
  return MOE_OK;
}

moe_status scatter_bwd_fused(const moe_config* cfg, const void* dy, const void* y_rows, const int32_t* map,
                             const float* gates, void* dy_rows, float* dgates, const float* logits,
                             const int32_t* expert_idx, __nv_bfloat16* dlogits_bf16, float* dlogits_f32,
                             const moe_topology_t* pad_topo, cudaStream_t s, const float* aux_c) {
  const int vec = (int)(cfg->hidden / 256);
  SbwdArgs a{reinterpret_cast<const uint4*>(dy), reinterpret_cast<const uint4*>(y_rows), map, gates,
             reinterpret_cast<uint4*>(dy_rows), dgates, (int)cfg->tokens, (int)cfg->top_k, logits, expert_idx,
             (int)cfg->num_experts, dlogits_bf16, dlogits_f32, pad_topo ? pad_topo->counts : nullptr,
             pad_topo ? pad_topo->padded_bins : nullptr, (int)cfg->block_size, cfg->renormalize, aux_c};
  // one token per warp: measured faster than 2-4 tokens per warp (whose register
  // footprint halves the occupancy) at MoE-XS
  switch (vec) {
    case 1: return sbwd_launch<1, 1>(a, s);
    case 2: return sbwd_launch<2, 1>(a, s);
    case 3: return sbwd_launch<3, 1>(a, s);
    case 4: return sbwd_launch<4, 1>(a, s);
    case 5: return sbwd_launch<5, 1>(a, s);
    case 6: return sbwd_launch<6, 1>(a, s);
    case 7: return sbwd_launch<7, 1>(a, s);
    default: return sbwd_launch<8, 1>(a, s);
  }
}

}  // namespace moe

using namespace moe;

extern "C" {

moe_status moe_gather(const moe_config* cfg, const void* x, const moe_topology_t* topo, void* x_g, void* stream) {
  MOE_TRY(check_rows(cfg, topo, "moe_gather"));
  MOE_CHECK_ARG(x && x_g, "moe_gather: NULL pointer");
  cudaStream_t s = as_stream(stream);
  const int R = (int)(cfg->tokens * cfg->top_k);
  MOE_VEC_DISPATCH((int)(cfg->hidden / 256), "moe_gather", scatter_rows_kernel, reinterpret_cast<const uint4*>(x), topo->pos,
                   reinterpret_cast<uint4*>(x_g), R, (int)cfg->top_k, topo->counts, topo->padded_bins,
                   (int)cfg->num_experts, (int)cfg->block_size);
  return MOE_OK;
}

moe_status moe_scatter(const moe_config* cfg, const void* y_g, const moe_topology_t* topo, const float* gates,
                       void* y, void* stream) {
  MOE_TRY(check_rows(cfg, topo, "moe_scatter"));
  MOE_CHECK_ARG(y_g && y, "moe_scatter: NULL pointer");
  cudaStream_t s = as_stream(stream);
  MOE_VEC_DISPATCH((int)(cfg->hidden / 256), "moe_scatter", combine_kernel, reinterpret_cast<const uint4*>(y_g), topo->pos, gates,
                   reinterpret_cast<uint4*>(y), (int)cfg->tokens, (int)cfg->top_k);
  return MOE_OK;
}

moe_status moe_scatter_bwd(const moe_config* cfg, const void* dy, const void* y_g, const moe_topology_t* topo,
                           const float* gates, void* dy_g, float* dgates, void* stream) {
  MOE_TRY(check_rows(cfg, topo, "moe_scatter_bwd"));
  MOE_CHECK_ARG(dy && dy_g && (y_g || !dgates), "moe_scatter_bwd: NULL pointer");
  return scatter_bwd_fused(cfg, dy, y_g, topo->pos, gates, dy_g, dgates, nullptr, nullptr, nullptr, nullptr, topo,
                           as_stream(stream));
}

moe_status moe_gather_bwd(const moe_config* cfg, const void* dx_g, const moe_topology_t* topo, void* dx,
                          void* stream) {
  MOE_TRY(check_rows(cfg, topo, "moe_gather_bwd"));
  MOE_CHECK_ARG(dx_g && dx, "moe_gather_bwd: NULL pointer");
  cudaStream_t s = as_stream(stream);
  MOE_VEC_DISPATCH((int)(cfg->hidden / 256), "moe_gather_bwd", combine_kernel, reinterpret_cast<const uint4*>(dx_g), topo->pos, nullptr,
                   reinterpret_cast<uint4*>(dx), (int)cfg->tokens, (int)cfg->top_k);
  return MOE_OK;
}

moe_status moe_sort_rows(const moe_config* cfg, const void* x, const moe_topology_t* topo, void* x_sorted,
                         void* stream) {
  MOE_TRY(check_rows(cfg, topo, "moe_sort_rows"));
  MOE_CHECK_ARG(x && x_sorted, "moe_sort_rows: NULL pointer");
  cudaStream_t s = as_stream(stream);
  const int R = (int)(cfg->tokens * cfg->top_k);
  MOE_VEC_DISPATCH((int)(cfg->hidden / 256), "moe_sort_rows", scatter_rows_kernel, reinterpret_cast<const uint4*>(x), topo->sorted_pos,
                   reinterpret_cast<uint4*>(x_sorted), R, (int)cfg->top_k, nullptr, nullptr, 0, 1);
  return MOE_OK;
}

moe_status moe_unsort_rows(const moe_config* cfg, const void* y_sorted, const moe_topology_t* topo,
                           const float* gates, void* y, void* stream) {
  MOE_TRY(check_rows(cfg, topo, "moe_unsort_rows"));
  MOE_CHECK_ARG(y_sorted && y, "moe_unsort_rows: NULL pointer");
  cudaStream_t s = as_stream(stream);
  MOE_VEC_DISPATCH((int)(cfg->hidden / 256), "moe_unsort_rows", combine_kernel, reinterpret_cast<const uint4*>(y_sorted),
                   topo->sorted_pos, gates, reinterpret_cast<uint4*>(y), (int)cfg->tokens, (int)cfg->top_k);
  return MOE_OK;
}

moe_status moe_unsort_rows_bwd(const moe_config* cfg, const void* dy, const void* y_sorted, const moe_topology_t* topo,
                               const float* gates, void* dy_sorted, float* dgates, void* stream) {
  MOE_TRY(check_rows(cfg, topo, "moe_unsort_rows_bwd"));
  MOE_CHECK_ARG(dy && dy_sorted && (y_sorted || !dgates), "moe_unsort_rows_bwd: NULL pointer");
  return scatter_bwd_fused(cfg, dy, y_sorted, topo->sorted_pos, gates, dy_sorted, dgates, nullptr, nullptr, nullptr,
                           nullptr, nullptr, as_stream(stream));
}

moe_status moe_sort_rows_bwd(const moe_config* cfg, const void* dx_sorted, const moe_topology_t* topo, void* dx,
                             void* stream) {
  return moe_unsort_rows(cfg, dx_sorted, topo, nullptr, dx, stream);
}

moe_status moe_zero_pad_rows(const moe_config* cfg, const moe_topology_t* topo, void* x_g, void* stream) {
  MOE_TRY(check_rows(cfg, topo, "moe_zero_pad_rows"));
  MOE_CHECK_ARG(x_g, "moe_zero_pad_rows: NULL x_g");
  cudaStream_t s = as_stream(stream);
  MOE_VEC_DISPATCH((int)(cfg->hidden / 256), "moe_zero_pad_rows", zero_pad_kernel, reinterpret_cast<uint4*>(x_g),
                   topo->counts, topo->padded_bins, (int)cfg->num_experts, (int)cfg->block_size);
  return MOE_OK;
}

}  // extern "C"
