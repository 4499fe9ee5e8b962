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
      if (base + r < R) {
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
        if (base + r < T) {
          const uint4* s = rows + (size_t)m * RV;
#pragma unroll
          for (int u = 0; u < VEC; ++u) v[r][u] = __ldg(s + lane + 32 * u);
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

// Per token t (one warp): dy_rows[map[i]] = g_i * dy[t]; dgates[i] = <y_rows[map[i]], dy[t]>,
// i = t*k + j. Optionally fused router backward (P:98 softmax chain rule):
// dlogits[t,:] = p * (dp - <p,dp>), p = softmax(logits[t,:]), dp[e] = sum_{j: idx_j = e} dgates_j.
template <int VEC>
__global__ void __launch_bounds__(256) scatter_bwd_kernel(
    const uint4* __restrict__ dy, const uint4* __restrict__ y_rows, const int32_t* __restrict__ map,
    const float* __restrict__ gates, uint4* __restrict__ dy_rows, float* __restrict__ dgates, int T, int k,
    const float* __restrict__ logits, const int32_t* __restrict__ expert_idx, int E,
    __nv_bfloat16* __restrict__ dlogits_bf16, float* __restrict__ dlogits_f32, const int32_t* __restrict__ counts,
    const int32_t* __restrict__ padded_bins, int bs) {
  pdl_trigger();
  pdl_wait();
  constexpr int RV = VEC * 32;
  const int lane = threadIdx.x & 31;
  const bool want_dg = dgates != nullptr;
  for (int t = warp_global(); t < T; t += warps_total()) {
    uint4 d[VEC];
    const uint4* ds = dy + (size_t)t * RV;
#pragma unroll
    for (int u = 0; u < VEC; ++u) d[u] = __ldg(ds + lane + 32 * u);
    float df[VEC][8];
#pragma unroll
    for (int u = 0; u < VEC; ++u) bf16x8_to_f32(d[u], df[u]);
    const int midx = lane < k ? __ldg(map + (size_t)t * k + lane) : 0;
    const float gl = lane < k ? (gates ? __ldg(gates + (size_t)t * k + lane) : 1.0f) : 0.f;
    float dg_lane = 0.f;  // lane j holds dgates[t, j]
    for (int j = 0; j < k; ++j) {
      const int m = __shfl_sync(0xffffffffu, midx, j);
      const float g = __shfl_sync(0xffffffffu, gl, j);
      uint4 yv[VEC];
      if (want_dg) {
        const uint4* ys = y_rows + (size_t)m * RV;
#pragma unroll
        for (int u = 0; u < VEC; ++u) yv[u] = __ldg(ys + lane + 32 * u);
      }
      uint4* o = dy_rows + (size_t)m * RV;
#pragma unroll
      for (int u = 0; u < VEC; ++u) {
        float f[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) f[q] = g * df[u][q];
        o[lane + 32 * u] = f32_to_bf16x8(f);
      }
      if (want_dg) {
        float dot = 0.f;
#pragma unroll
        for (int u = 0; u < VEC; ++u) {
          float fy[8];
          bf16x8_to_f32(yv[u], fy);
#pragma unroll
          for (int q = 0; q < 8; ++q) dot = fmaf(fy[q], df[u][q], dot);
        }
#pragma unroll
        for (int o2 = 16; o2 > 0; o2 >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o2);
        if (lane == j) dg_lane = dot;
      }
    }
    if (want_dg && lane < k) dgates[(size_t)t * k + lane] = dg_lane;
    if (logits && (dlogits_bf16 || dlogits_f32)) {  // E <= 256 (checked on the host)
      const float* row = logits + (size_t)t * E;
      float lv[8];
      float m = -FLT_MAX;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int e = lane + 32 * q;
        lv[q] = e < E ? row[e] : -FLT_MAX;
        m = fmaxf(m, lv[q]);
      }
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o2));
      float ssum = 0.f, pv[8], dpl[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        pv[q] = lane + 32 * q < E ? __expf(lv[q] - m) : 0.f;
        ssum += pv[q];
        dpl[q] = 0.f;
      }
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) ssum += __shfl_xor_sync(0xffffffffu, ssum, o2);
      const float inv = 1.f / ssum;
      const int ej = lane < k ? __ldg(expert_idx + (size_t)t * k + lane) : -1;
      float pdp = 0.f;
      for (int j = 0; j < k; ++j) {  // warp-uniform
        const int ejj = __shfl_sync(0xffffffffu, ej, j);
        const float dgj = __shfl_sync(0xffffffffu, dg_lane, j);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (lane + 32 * q == ejj) {
            dpl[q] += dgj;
            pdp += pv[q] * inv * dgj;
          }
      }
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) pdp += __shfl_xor_sync(0xffffffffu, pdp, o2);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int e = lane + 32 * q;
        if (e < E) {
          const float dl = pv[q] * inv * (dpl[q] - pdp);
          if (dlogits_bf16)
            dlogits_bf16[(size_t)t * E + e] = __float2bfloat16_rn(dl);
          else
            dlogits_f32[(size_t)t * E + e] = dl;
        }
      }
    }
  }
  if (counts) zero_pad_rows<VEC>(dy_rows, counts, padded_bins, E, bs);
}

static int row_grid() { return moe_device_sm_count() * 8; }

static moe_status check_rows(const moe_config* cfg, const moe_topology_t* topo, const char* name) {
  MOE_TRY(moe_check_config(cfg));
  MOE_TRY(check_topo(topo));
  if (cfg->hidden % 256 || cfg->hidden > 2048)
    return set_error(MOE_EUNSUPPORTED, "%s: hidden=%lld must be a multiple of 256 and <= 2048", name,
                     (long long)cfg->hidden);
  return MOE_OK;
}

#define MOE_VEC_CASE(V, NAME, KERNEL, ...) \
  case V: MOE_LAUNCH(NAME, KERNEL<V>, dim3(row_grid()), dim3(32 * kWarpsPerCta), 0, s, __VA_ARGS__); break;
#define MOE_VEC_DISPATCH(VEC_EXPR, NAME, KERNEL, ...)  \
  switch (VEC_EXPR) {                                  \
    MOE_VEC_CASE(1, NAME, KERNEL, __VA_ARGS__)         \
    MOE_VEC_CASE(2, NAME, KERNEL, __VA_ARGS__)         \
    MOE_VEC_CASE(3, NAME, KERNEL, __VA_ARGS__)         \
    MOE_VEC_CASE(4, NAME, KERNEL, __VA_ARGS__)         \
    MOE_VEC_CASE(5, NAME, KERNEL, __VA_ARGS__)         \
    MOE_VEC_CASE(6, NAME, KERNEL, __VA_ARGS__)         \
    MOE_VEC_CASE(7, NAME, KERNEL, __VA_ARGS__)         \
    default: MOE_LAUNCH(NAME, KERNEL<8>, dim3(row_grid()), dim3(32 * kWarpsPerCta), 0, s, __VA_ARGS__); break; \
  }

moe_status scatter_bwd_fused(const moe_config* cfg, const void* dy, const void* y_rows, const int32_t* map,
                             const float* gates, void* dy_rows, float* dgates, const float* logits,
                             const int32_t* expert_idx, __nv_bfloat16* dlogits_bf16, float* dlogits_f32,
                             const moe_topology_t* pad_topo, cudaStream_t s) {
  const int vec = (int)(cfg->hidden / 256);
  const int T = (int)cfg->tokens, k = (int)cfg->top_k, E = (int)cfg->num_experts, bs = (int)cfg->block_size;
  const int32_t* counts = pad_topo ? pad_topo->counts : nullptr;
  const int32_t* pbins = pad_topo ? pad_topo->padded_bins : nullptr;
  MOE_VEC_DISPATCH(vec, "scatter_bwd", scatter_bwd_kernel, reinterpret_cast<const uint4*>(dy), reinterpret_cast<const uint4*>(y_rows),
                   map, gates, reinterpret_cast<uint4*>(dy_rows), dgates, T, k, logits, expert_idx, E, dlogits_bf16,
                   dlogits_f32, counts, pbins, bs);
  return MOE_OK;
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

}  // extern "C"
