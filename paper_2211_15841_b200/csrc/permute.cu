// permute.cu — padded permutation kernels ("we pad each group of tokens
// with zeros to the nearest multiple of 128 and fuse this operation into
// custom permutation kernels"), the weighted un-permutation (P:279-280,
// §2.4) and their backward passes, plus the unpadded expert-order
// permutation used for expert-parallel dispatch.
//
// All kernels are HBM-bandwidth bound row copies: one warp per output row,
// 16-byte vector loads/stores, loads of a row issued before its stores,
// grid-stride over rows with the device-side row count (no host sync).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"

namespace moe {

constexpr int kWarpsPerCta = 8;
constexpr int kMaxVec = 8;  // h <= 8 * 32 * 8 = 2048 elements per lane pass

struct RowCtx {
  const int32_t* counts;
  const int32_t* bins;
  const int32_t* padded_bins;
  const int32_t* sorted_idx;
  const int32_t* col_indices;
  const int32_t* sizes;
  int F, bs;
};

// Flat id (t*k+j) stored in padded row p, or -1 for a pad row.
__device__ __forceinline__ int padded_row_source(const RowCtx& c, int p) {
  const int r = p / c.bs;
  const int e = __ldg(c.col_indices + (size_t)r * c.F) / c.F;
  const int cnt = __ldg(c.counts + e);
  const int pc = ((cnt + c.bs - 1) / c.bs) * c.bs;
  const int rank = p - (__ldg(c.padded_bins + e) - pc);
  if (rank >= cnt) return -1;
  return __ldg(c.sorted_idx + __ldg(c.bins + e) - cnt + rank);
}

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

// x_g[p] = x[src(p)/k] or 0   (output-driven: every row of x_g written once)
__global__ void gather_kernel(const uint4* __restrict__ x, uint4* __restrict__ xg, RowCtx c, int k, int vec) {
  const int Tp = c.sizes[0];
  const int lane = threadIdx.x & 31;
  for (int p = blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5); p < Tp; p += gridDim.x * kWarpsPerCta) {
    const int i = padded_row_source(c, p);
    uint4 v[kMaxVec];
    if (i >= 0) {
      const uint4* src = x + (size_t)(i / k) * vec;
#pragma unroll
      for (int u = 0; u < kMaxVec; ++u)
        if (lane + 32 * u < vec) v[u] = __ldg(src + lane + 32 * u);
    } else {
#pragma unroll
      for (int u = 0; u < kMaxVec; ++u) v[u] = make_uint4(0, 0, 0, 0);
    }
    uint4* dst = xg + (size_t)p * vec;
#pragma unroll
    for (int u = 0; u < kMaxVec; ++u)
      if (lane + 32 * u < vec) dst[lane + 32 * u] = v[u];
  }
}

// y[t] = sum_j g[t,j] * rows[map[t*k+j]]  (fp32 accumulate, ascending j)
__global__ void combine_kernel(const uint4* __restrict__ rows, const int32_t* __restrict__ map,
                               const float* __restrict__ gates, uint4* __restrict__ y, int T, int k, int vec) {
  const int lane = threadIdx.x & 31;
  for (int t = blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5); t < T; t += gridDim.x * kWarpsPerCta) {
    float acc[kMaxVec][8];
#pragma unroll
    for (int u = 0; u < kMaxVec; ++u)
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[u][q] = 0.f;
    for (int j = 0; j < k; ++j) {
      const int i = t * k + j;
      const float g = gates ? __ldg(gates + i) : 1.0f;
      const uint4* src = rows + (size_t)__ldg(map + i) * vec;
#pragma unroll
      for (int u = 0; u < kMaxVec; ++u) {
        if (lane + 32 * u < vec) {
          float f[8];
          bf16x8_to_f32(__ldg(src + lane + 32 * u), f);
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[u][q] = fmaf(g, f[q], acc[u][q]);
        }
      }
    }
    uint4* dst = y + (size_t)t * vec;
#pragma unroll
    for (int u = 0; u < kMaxVec; ++u)
      if (lane + 32 * u < vec) dst[lane + 32 * u] = f32_to_bf16x8(acc[u]);
  }
}

// dy_g[p] = g * dy[t] (0 for pad rows); dgates[i] = <y_g[p], dy[t]>.
// Output-driven over padded rows when `padded`, else over sorted rows u < R.
__global__ void scatter_bwd_kernel(const uint4* __restrict__ dy, const uint4* __restrict__ yg, RowCtx c,
                                   const float* __restrict__ gates, uint4* __restrict__ dyg, float* __restrict__ dgates,
                                   int k, int vec, int padded, int R) {
  const int lane = threadIdx.x & 31;
  const int nrows = padded ? c.sizes[0] : R;
  for (int p = blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5); p < nrows; p += gridDim.x * kWarpsPerCta) {
    const int i = padded ? padded_row_source(c, p) : __ldg(c.sorted_idx + p);
    uint4* dst = dyg + (size_t)p * vec;
    if (i < 0) {
#pragma unroll
      for (int u = 0; u < kMaxVec; ++u)
        if (lane + 32 * u < vec) dst[lane + 32 * u] = make_uint4(0, 0, 0, 0);
      continue;
    }
    const float g = gates ? __ldg(gates + i) : 1.0f;
    const uint4* d = dy + (size_t)(i / k) * vec;
    const uint4* yr = yg + (size_t)p * vec;
    uint4 dv[kMaxVec], yv[kMaxVec];
#pragma unroll
    for (int u = 0; u < kMaxVec; ++u)
      if (lane + 32 * u < vec) {
        dv[u] = __ldg(d + lane + 32 * u);
        if (dgates) yv[u] = __ldg(yr + lane + 32 * u);
      }
    float dot = 0.f;
#pragma unroll
    for (int u = 0; u < kMaxVec; ++u) {
      if (lane + 32 * u < vec) {
        float fd[8];
        bf16x8_to_f32(dv[u], fd);
        if (dgates) {
          float fy[8];
          bf16x8_to_f32(yv[u], fy);
#pragma unroll
          for (int q = 0; q < 8; ++q) dot = fmaf(fy[q], fd[q], dot);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) fd[q] *= g;
        dst[lane + 32 * u] = f32_to_bf16x8(fd);
      }
    }
    if (dgates) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
      if (lane == 0) dgates[i] = dot;
    }
  }
}

// dst[u] = src[sorted_idx[u] / k], u < R   (unpadded expert-order permutation)
__global__ void sort_rows_kernel(const uint4* __restrict__ x, const int32_t* __restrict__ sorted_idx,
                                 uint4* __restrict__ out, int R, int k, int vec) {
  const int lane = threadIdx.x & 31;
  for (int u0 = blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5); u0 < R; u0 += gridDim.x * kWarpsPerCta) {
    const uint4* src = x + (size_t)(__ldg(sorted_idx + u0) / k) * vec;
    uint4 v[kMaxVec];
#pragma unroll
    for (int u = 0; u < kMaxVec; ++u)
      if (lane + 32 * u < vec) v[u] = __ldg(src + lane + 32 * u);
    uint4* dst = out + (size_t)u0 * vec;
#pragma unroll
    for (int u = 0; u < kMaxVec; ++u)
      if (lane + 32 * u < vec) dst[lane + 32 * u] = v[u];
  }
}

static int row_grid(int64_t rows) {
  int64_t g = ceil_div(rows > 0 ? rows : 1, kWarpsPerCta);
  const int64_t cap = (int64_t)moe_device_sm_count() * 16;
  return (int)(g < cap ? g : cap);
}

static RowCtx row_ctx(const moe_config* cfg, const moe_topology_t* t) {
  RowCtx c;
  c.counts = t->counts;
  c.bins = t->bins;
  c.padded_bins = t->padded_bins;
  c.sorted_idx = t->sorted_idx;
  c.col_indices = t->col_indices;
  c.sizes = t->sizes;
  c.F = (int)(cfg->ffn_hidden / cfg->block_size);
  c.bs = (int)cfg->block_size;
  return c;
}

static moe_status check_rows(const moe_config* cfg, const moe_topology_t* topo, const char* name) {
  MOE_TRY(moe_check_config(cfg));
  MOE_TRY(check_topo(topo));
  if (cfg->hidden % 8 || cfg->hidden > 8 * 32 * kMaxVec)
    return set_error(MOE_EUNSUPPORTED, "%s: hidden=%lld must be a multiple of 8 and <= %d", name,
                     (long long)cfg->hidden, 8 * 32 * kMaxVec);
  return MOE_OK;
}

}  // namespace moe

using namespace moe;

extern "C" {

moe_status moe_gather(const moe_config* cfg, const void* x, const moe_topology_t* topo, void* x_g, void* stream) {
  MOE_TRY(check_rows(cfg, topo, "moe_gather"));
  MOE_CHECK_ARG(x && x_g, "moe_gather: NULL pointer");
  const int vec = (int)(cfg->hidden / 8);
  gather_kernel<<<row_grid(moe_max_padded_rows(cfg)), 32 * kWarpsPerCta, 0, as_stream(stream)>>>(
      reinterpret_cast<const uint4*>(x), reinterpret_cast<uint4*>(x_g), row_ctx(cfg, topo), (int)cfg->top_k, vec);
  MOE_CHECK_LAUNCH("moe_gather");
  return MOE_OK;
}

moe_status moe_scatter(const moe_config* cfg, const void* y_g, const moe_topology_t* topo, const float* gates,
                       void* y, void* stream) {
  MOE_TRY(check_rows(cfg, topo, "moe_scatter"));
  MOE_CHECK_ARG(y_g && y, "moe_scatter: NULL pointer");
  const int T = (int)cfg->tokens;
  combine_kernel<<<row_grid(T), 32 * kWarpsPerCta, 0, as_stream(stream)>>>(
      reinterpret_cast<const uint4*>(y_g), topo->pos, gates, reinterpret_cast<uint4*>(y), T, (int)cfg->top_k,
      (int)(cfg->hidden / 8));
  MOE_CHECK_LAUNCH("moe_scatter");
  return MOE_OK;
}

moe_status moe_scatter_bwd(const moe_config* cfg, const void* dy, const void* y_g, const moe_topology_t* topo,
                           const float* gates, void* dy_g, float* dgates, void* stream) {
  MOE_TRY(check_rows(cfg, topo, "moe_scatter_bwd"));
  MOE_CHECK_ARG(dy && dy_g && (y_g || !dgates), "moe_scatter_bwd: NULL pointer");
  scatter_bwd_kernel<<<row_grid(moe_max_padded_rows(cfg)), 32 * kWarpsPerCta, 0, as_stream(stream)>>>(
      reinterpret_cast<const uint4*>(dy), reinterpret_cast<const uint4*>(y_g), row_ctx(cfg, topo), gates,
      reinterpret_cast<uint4*>(dy_g), dgates, (int)cfg->top_k, (int)(cfg->hidden / 8), 1, 0);
  MOE_CHECK_LAUNCH("moe_scatter_bwd");
  return MOE_OK;
}

moe_status moe_gather_bwd(const moe_config* cfg, const void* dx_g, const moe_topology_t* topo, void* dx,
                          void* stream) {
  MOE_TRY(check_rows(cfg, topo, "moe_gather_bwd"));
  MOE_CHECK_ARG(dx_g && dx, "moe_gather_bwd: NULL pointer");
  const int T = (int)cfg->tokens;
  combine_kernel<<<row_grid(T), 32 * kWarpsPerCta, 0, as_stream(stream)>>>(
      reinterpret_cast<const uint4*>(dx_g), topo->pos, nullptr, reinterpret_cast<uint4*>(dx), T, (int)cfg->top_k,
      (int)(cfg->hidden / 8));
  MOE_CHECK_LAUNCH("moe_gather_bwd");
  return MOE_OK;
}

moe_status moe_sort_rows(const moe_config* cfg, const void* x, const moe_topology_t* topo, void* x_sorted,
                         void* stream) {
  MOE_TRY(check_rows(cfg, topo, "moe_sort_rows"));
  MOE_CHECK_ARG(x && x_sorted, "moe_sort_rows: NULL pointer");
  const int R = (int)(cfg->tokens * cfg->top_k);
  sort_rows_kernel<<<row_grid(R), 32 * kWarpsPerCta, 0, as_stream(stream)>>>(
      reinterpret_cast<const uint4*>(x), topo->sorted_idx, reinterpret_cast<uint4*>(x_sorted), R, (int)cfg->top_k,
      (int)(cfg->hidden / 8));
  MOE_CHECK_LAUNCH("moe_sort_rows");
  return MOE_OK;
}

moe_status moe_unsort_rows(const moe_config* cfg, const void* y_sorted, const moe_topology_t* topo,
                           const float* gates, void* y, void* stream) {
  MOE_TRY(check_rows(cfg, topo, "moe_unsort_rows"));
  MOE_CHECK_ARG(y_sorted && y, "moe_unsort_rows: NULL pointer");
  const int T = (int)cfg->tokens;
  combine_kernel<<<row_grid(T), 32 * kWarpsPerCta, 0, as_stream(stream)>>>(
      reinterpret_cast<const uint4*>(y_sorted), topo->sorted_pos, gates, reinterpret_cast<uint4*>(y), T,
      (int)cfg->top_k, (int)(cfg->hidden / 8));
  MOE_CHECK_LAUNCH("moe_unsort_rows");
  return MOE_OK;
}

moe_status moe_unsort_rows_bwd(const moe_config* cfg, const void* dy, const void* y_sorted, const moe_topology_t* topo,
                               const float* gates, void* dy_sorted, float* dgates, void* stream) {
  MOE_TRY(check_rows(cfg, topo, "moe_unsort_rows_bwd"));
  MOE_CHECK_ARG(dy && dy_sorted && (y_sorted || !dgates), "moe_unsort_rows_bwd: NULL pointer");
  const int R = (int)(cfg->tokens * cfg->top_k);
  scatter_bwd_kernel<<<row_grid(R), 32 * kWarpsPerCta, 0, as_stream(stream)>>>(
      reinterpret_cast<const uint4*>(dy), reinterpret_cast<const uint4*>(y_sorted), row_ctx(cfg, topo), gates,
      reinterpret_cast<uint4*>(dy_sorted), dgates, (int)cfg->top_k, (int)(cfg->hidden / 8), 0, R);
  MOE_CHECK_LAUNCH("moe_unsort_rows_bwd");
  return MOE_OK;
}

moe_status moe_sort_rows_bwd(const moe_config* cfg, const void* dx_sorted, const moe_topology_t* topo, void* dx,
                             void* stream) {
  return moe_unsort_rows(cfg, dx_sorted, topo, nullptr, dx, stream);
}

}  // extern "C"
