// router.cu — learned router (§2.1): logits = x . Wr, softmax,
// greedy top-k; and its backward pass (softmax chain rule).
//
// v1 SIMT implementation (fp32 FMA on CUDA cores, bf16 operands staged in
// shared memory). The router is ~4% of the strict layer roofline (SURVEY.md
// §8(a) a1/b7); DESIGN.md §5 tracks moving it onto tcgen05.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <float.h>

#include "bsgemm.cuh"
#include "common.cuh"
#include "permute.cuh"
#include "tma.cuh"
#include "gemm_util.cuh"

namespace moe {

constexpr int RT_TOK = 64;   // tokens per CTA
constexpr int RT_EXP = 64;   // experts per CTA
constexpr int RT_K = 32;     // contraction chunk

// logits[t, e] = sum_i x[t,i] * wr[i,e]; 256 threads, each 4 tokens x 4 experts.
__global__ void __launch_bounds__(256) router_logits_kernel(const __nv_bfloat16* __restrict__ x,
                                                             const __nv_bfloat16* __restrict__ wr,
                                                             float* __restrict__ logits, int T, int h, int E) {
  pdl_trigger();
  pdl_wait();
  __shared__ float sx[RT_K][RT_TOK + 1];
  __shared__ float sw[RT_K][RT_EXP];
  const int t0 = blockIdx.x * RT_TOK, e0 = blockIdx.y * RT_EXP;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;  // experts tx*4.., tokens ty*4..
  float acc[4][4] = {};
  for (int k0 = 0; k0 < h; k0 += RT_K) {
    for (int i = threadIdx.x; i < RT_TOK * RT_K; i += 256) {
      const int tt = i / RT_K, kk = i % RT_K;
      const int t = t0 + tt;
      sx[kk][tt] = (t < T && k0 + kk < h) ? __bfloat162float(x[(size_t)t * h + k0 + kk]) : 0.f;
    }
    for (int i = threadIdx.x; i < RT_K * RT_EXP; i += 256) {
      const int kk = i / RT_EXP, ee = i % RT_EXP;
      const int e = e0 + ee;
      sw[kk][ee] = (e < E && k0 + kk < h) ? __bfloat162float(wr[(size_t)(k0 + kk) * E + e]) : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < RT_K; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sx[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = sw[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int t = t0 + ty * 4 + i;
    if (t >= T) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int e = e0 + tx * 4 + j;
      if (e < E) logits[(size_t)t * E + e] = acc[i][j];
    }
  }
}

// One warp per token: top-k of the fp32 logits (descending, ties -> lower e)
// then gates = softmax probabilities of the chosen experts.
constexpr int kMaxTopK = 32;
__global__ void topk_kernel(const float* __restrict__ logits, int32_t* __restrict__ idx, float* __restrict__ gates,
                            int T, int E, int k, int renorm) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (t >= T) return;
  const float* row = logits + (size_t)t * E;
  // softmax denominator with the row max (fixed ascending-e per-lane order, then tree)
  float m = -FLT_MAX;
  for (int e = lane; e < E; e += 32) m = fmaxf(m, row[e]);
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float ssum = 0.f;
  for (int e = lane; e < E; e += 32) ssum += expf(row[e] - m);
  for (int o = 16; o > 0; o >>= 1) ssum += __shfl_xor_sync(0xffffffffu, ssum, o);
  // k rounds of arg-max excluding already chosen experts
  unsigned chosen = 0;  // per-lane bitmask of chosen experts e = lane + 32*b (E <= 1024)
  for (int j = 0; j < k; ++j) {
    float bv = -FLT_MAX;
    int be = 0x7fffffff;
    for (int b = 0, e = lane; e < E; ++b, e += 32) {
      const bool taken = (chosen >> b) & 1u;
      const float v = row[e];
      if (!taken && (v > bv || (v == bv && e < be))) {
        bv = v;
        be = e;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oe = __shfl_xor_sync(0xffffffffu, be, o);
      if (ov > bv || (ov == bv && oe < be)) {
        bv = ov;
        be = oe;
      }
    }
    if ((be & 31) == lane) chosen |= 1u << (be >> 5);
    if (lane == 0) {
      idx[(size_t)t * k + j] = be;
      gates[(size_t)t * k + j] = expf(bv - m) / ssum;
    }
  }
  if (renorm && lane == 0) {  // NEXT-4: the k gates divided by their sum
    float gs = 0.f;
    for (int j = 0; j < k; ++j) gs += gates[(size_t)t * k + j];
    for (int j = 0; j < k; ++j) gates[(size_t)t * k + j] /= gs;
  }
}

// dlogits[t,:] = p * (dp - <p, dp>) with p = softmax(logits[t,:]), dp sparse from dgates.
// With renorm (gates g_j = p_j / S, S = sum of the chosen p): the gradient
// reaching p_j is (dg_j - sum_i dg_i g_i) / S.
// aux_c (optional, [E]): the auxiliary loss's d/dp, added to every expert's dp.
__global__ void router_dlogits_kernel(const float* __restrict__ logits, const int32_t* __restrict__ idx,
                                      const float* __restrict__ dgates, float* __restrict__ dlogits,
                                      __nv_bfloat16* __restrict__ dlogits_bf16, int T, int E, int k, int renorm,
                                      const float* __restrict__ aux_c) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (t >= T) return;
  const float* row = logits + (size_t)t * E;
  float m = -FLT_MAX;
  for (int e = lane; e < E; e += 32) m = fmaxf(m, row[e]);
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float ssum = 0.f;
  for (int e = lane; e < E; e += 32) ssum += expf(row[e] - m);
  for (int o = 16; o > 0; o >>= 1) ssum += __shfl_xor_sync(0xffffffffu, ssum, o);
  const float inv = 1.f / ssum;
  float rs = 1.f, gd = 0.f;  // renorm: 1/S and sum_i dg_i g_i
  if (renorm) {
    float S = 0.f;
    for (int j = 0; j < k; ++j) S += expf(row[idx[(size_t)t * k + j]] - m) * inv;
    rs = 1.f / S;
    for (int j = 0; j < k; ++j) gd += dgates[(size_t)t * k + j] * expf(row[idx[(size_t)t * k + j]] - m) * inv * rs;
  }
  auto dgp = [&](int j) { return renorm ? (dgates[(size_t)t * k + j] - gd) * rs : dgates[(size_t)t * k + j]; };
  // <p, dp> = sum_j p[idx_j] * dp_j
  float pdp = 0.f;
  for (int j = 0; j < k; ++j) {
    const int e = idx[(size_t)t * k + j];
    pdp += expf(row[e] - m) * inv * dgp(j);
  }
  if (aux_c) {  // + <p, c>
    float pa = 0.f;
    for (int e = lane; e < E; e += 32) pa += expf(row[e] - m) * inv * __ldg(aux_c + e);
    for (int o = 16; o > 0; o >>= 1) pa += __shfl_xor_sync(0xffffffffu, pa, o);
    pdp += pa;
  }
  for (int e = lane; e < E; e += 32) {
    float dp = aux_c ? __ldg(aux_c + e) : 0.f;
    for (int j = 0; j < k; ++j)
      if (idx[(size_t)t * k + j] == e) dp += dgp(j);
    const float p = expf(row[e] - m) * inv;
    if (dlogits_bf16)
      dlogits_bf16[(size_t)t * E + e] = __float2bfloat16_rn(p * (dp - pdp));
    else
      dlogits[(size_t)t * E + e] = p * (dp - pdp);
  }
}

// Partial dWr over a token range: part[q][i][e] = sum_{t in range q} x[t,i] dlogits[t,e].
// grid (parts, ceil(h/32)), 256 threads: 32 rows i x 64 experts per CTA slice.
__global__ void __launch_bounds__(256) router_dwr_part_kernel(const __nv_bfloat16* __restrict__ x,
                                                               const float* __restrict__ dlogits,
                                                               float* __restrict__ part, int T, int h, int E,
                                                               int tok_per_part) {
  pdl_trigger();
  pdl_wait();
  __shared__ float sx[32][33];
  __shared__ float sd[32][64];
  const int q = blockIdx.x, i0 = blockIdx.y * 32;
  const int tb = q * tok_per_part, te = min(T, tb + tok_per_part);
  for (int e0 = 0; e0 < E; e0 += 64) {
    const int ti = threadIdx.x / 8;        // row i within slice (0..31)
    const int tj = (threadIdx.x % 8) * 8;  // 8 experts
    float acc[8] = {};
    for (int t0 = tb; t0 < te; t0 += 32) {
      for (int u = threadIdx.x; u < 32 * 32; u += 256) {
        const int tt = u / 32, ii = u % 32;
        const int t = t0 + tt, i = i0 + ii;
        sx[tt][ii] = (t < te && i < h) ? __bfloat162float(x[(size_t)t * h + i]) : 0.f;
      }
      for (int u = threadIdx.x; u < 32 * 64; u += 256) {
        const int tt = u / 64, ee = u % 64;
        const int t = t0 + tt, e = e0 + ee;
        sd[tt][ee] = (t < te && e < E) ? dlogits[(size_t)t * E + e] : 0.f;
      }
      __syncthreads();
#pragma unroll 4
      for (int tt = 0; tt < 32; ++tt) {
        const float a = sx[tt][ti];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = fmaf(a, sd[tt][tj + j], acc[j]);
      }
      __syncthreads();
    }
    const int i = i0 + ti;
    if (i < h)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int e = e0 + tj + j;
        if (e < E) part[((size_t)q * h + i) * E + e] = acc[j];
      }
  }
}

__global__ void router_dwr_reduce_kernel(const float* __restrict__ part, float* __restrict__ dwr, int parts, int n) {
  pdl_trigger();
  pdl_wait();
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= n) return;
  float s = 0.f;
  for (int q = 0; q < parts; ++q) s += part[(size_t)q * n + o];
  dwr[o] = s;
}

// dx[t, i] += sum_e dlogits[t,e] * wr[i,e]; one warp per token, wr^T slices cached in smem.
__global__ void __launch_bounds__(256) router_dx_kernel(const float* __restrict__ dlogits,
                                                         const __nv_bfloat16* __restrict__ wr,
                                                         __nv_bfloat16* __restrict__ dx, int T, int h, int E) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float s_dl[];  // [8 warps][E]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int t = blockIdx.x * 8 + warp;
  if (t < T)
    for (int e = lane; e < E; e += 32) s_dl[warp * E + e] = dlogits[(size_t)t * E + e];
  __syncwarp();
  if (t >= T) return;
  for (int i = lane; i < h; i += 32) {
    const __nv_bfloat16* w = wr + (size_t)i * E;
    float s = 0.f;
    for (int e = 0; e < E; ++e) s = fmaf(s_dl[warp * E + e], __bfloat162float(w[e]), s);
    const size_t o = (size_t)t * h + i;
    dx[o] = __float2bfloat16_rn(__bfloat162float(dx[o]) + s);
  }
}

}  // namespace moe

namespace moe {

// dWr = x^T . dlogits on tcgen05 (M = h, N = E, K = T split over `parts`
// token ranges into fp32 partials, then a fixed-order reduction).
moe_status router_dwr_tc(const moe_config* cfg, const void* x, const __nv_bfloat16* dlogits, float* dwr, void* ws,
                         cudaStream_t s) {
  const int T = (int)cfg->tokens, h = (int)cfg->hidden, E = (int)cfg->num_experts;
  const int parts = router_bwd_parts(cfg);
  float* part = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + ws_layout(cfg).dwr_part);
  GemmLaunch L{};
  L.name = "router dWr";
  L.mode = DENSE;
  L.bn = E;
  L.a_mn = true;
  L.b_mn = true;
  L.p.m_tiles = (int)ceil_div(h, 128);
  L.p.n_tiles = 1;
  L.p.splits = parts;
  L.p.k_iters_total = (int)ceil_div(T, BK);
  L.p.kiters_split = (int)ceil_div(L.p.k_iters_total, parts);
  L.p.epi = EPI_F32;
  L.p.rows_valid = h;
  L.p.out_f32 = part;
  L.p.ld_f32 = E;
  L.p.split_stride = (long long)h * E;
  L.max_tiles = parts * L.p.m_tiles;
  MOE_TRY(make_tmap_bf16_mn(&L.ta, x, h, T, h, 2, "router dWr x^T"));
  MOE_TRY(make_tmap_bf16_mn(&L.tb, dlogits, E, T, E, L.bn / 64, "router dWr dlogits"));
  L.tc = L.td = L.ta;
  MOE_TRY(gemm_launch(L, s));
  MOE_LAUNCH("router_dwr_reduce", router_dwr_reduce_kernel, dim3((int)ceil_div((int64_t)h * E, 256)), dim3(256), 0, s, part, dwr, parts, h * E);
  return MOE_OK;
}

// dx = dlogits . Wr^T + addend on tcgen05 (M = T, N = h, K = E); the addend is
// the row t of `addend` or, with addend_map, sum_j addend[addend_map[t*k+j]]
// (the padded-gather backward fused into the epilogue).
moe_status router_dx_tc(const moe_config* cfg, const __nv_bfloat16* dlogits, const void* wr, void* dx,
                        const void* addend, const int32_t* addend_map, int addend_k, long long ld_add,
                        cudaStream_t s) {
  const int T = (int)cfg->tokens, h = (int)cfg->hidden, E = (int)cfg->num_experts;
  GemmLaunch D{};
  D.name = "router dx";
  D.mode = DENSE;
  D.bn = 128;  // two 32-column chunks per epilogue warp: its gathered addend rows are prefetched in registers
  D.a_mn = false;
  D.b_mn = false;
  D.p.m_tiles = (int)ceil_div(T, 128);
  D.p.n_tiles = h / D.bn;
  D.p.splits = 1;
  D.p.k_iters_total = D.p.kiters_split = E / BK;
  D.p.epi = EPI_ADD_ROWS;
  D.p.rows_valid = T;
  D.p.addend = reinterpret_cast<const __nv_bfloat16*>(addend);
  D.p.ld_add = ld_add;
  D.p.addend_map = addend_map;
  D.p.addend_k = addend_k;
  D.max_tiles = D.p.m_tiles * D.p.n_tiles;
  MOE_TRY(make_tmap_bf16(&D.ta, dlogits, E, T, E, BK, 128, "router dx dlogits", KSW));
  MOE_TRY(make_tmap_bf16(&D.tb, wr, E, h, E, BK, D.bn, "router dx wr", KSW));
  MOE_TRY(make_tmap_epi(&D.tc, dx, h, T, h, "router dx out"));
  set_epi_out(D.p, 0, dx, T, h);
  D.td = D.tc;
  return gemm_launch(D, s);
}

}  // namespace moe

using namespace moe;

extern "C" {

moe_status moe_topk(const moe_config* cfg, const float* logits, int32_t* expert_idx, float* gates, void* stream) {
  MOE_TRY(moe_check_config(cfg));
  MOE_CHECK_ARG(logits && expert_idx && gates, "moe_topk: NULL pointer");
  if (cfg->top_k > kMaxTopK) return set_error(MOE_EUNSUPPORTED, "top_k=%lld > %d", (long long)cfg->top_k, kMaxTopK);
  const int T = (int)cfg->tokens;
  MOE_LAUNCH("moe_topk", topk_kernel, dim3((int)ceil_div(T, 8)), dim3(256), 0, as_stream(stream), logits, expert_idx, gates, T, (int)cfg->num_experts, (int)cfg->top_k, cfg->renormalize);
  return MOE_OK;
}

// logits = x . Wr on tcgen05 (M = tokens, N = E, K = h) with the greedy top-k
// + softmax gate epilogue fused (one thread per token row); with topo, the
// topology is built in the same (cooperative) launch.
static moe_status router_tc_launch(const moe_config* cfg, const void* x, const void* wr, float* logits,
                                   int32_t* expert_idx, float* gates, void* ws, const moe_topology_t* topo,
                                   void* stream) {
  const int T = (int)cfg->tokens, h = (int)cfg->hidden, E = (int)cfg->num_experts;
  GemmLaunch L{};
  L.name = topo ? "moe_router_topology" : "moe_router";
  L.mode = DENSE;
  L.bn = E;
  L.a_mn = false;
  L.b_mn = true;
  L.p.m_tiles = (int)ceil_div(T, 128);
  L.p.n_tiles = 1;
  L.p.splits = 1;
  L.p.k_iters_total = L.p.kiters_split = (int)ceil_div(h, BK);
  L.p.epi = EPI_ROUTER;
  L.p.rows_valid = T;
  L.p.logits = logits;
  L.p.idx = expert_idx;
  L.p.gates = gates;
  L.p.E = E;
  L.p.topk = (int)cfg->top_k;
  L.p.renorm = cfg->renormalize;
  // per-tile expert histograms for the topology (moe_topology_from_router, or fused below)
  L.p.hist_out = ws ? reinterpret_cast<int32_t*>(reinterpret_cast<char*>(ws) + ws_layout(cfg).router_hist) : nullptr;
  if (topo) {
    L.p.topo_fused = 1;
    L.p.topo = *topo;
    L.p.topo_bs = (int)cfg->block_size;
    L.p.topo_F = (int)(cfg->ffn_hidden / cfg->block_size);
    L.p.topo_capacity = (int)cfg->capacity;
  }
  L.max_tiles = L.p.m_tiles;
  MOE_TRY(make_tmap_bf16(&L.ta, x, h, T, h, BK, 128, "moe_router x", KSW));
  MOE_TRY(make_tmap_bf16_mn(&L.tb, wr, E, h, E, L.bn / 64, "moe_router wr"));
  MOE_TRY(make_tmap_f32(&L.tc, logits, E, T, E, "moe_router logits"));
  L.td = L.tc;
  return gemm_launch(L, as_stream(stream));
}

moe_status moe_router(const moe_config* cfg, const void* x, const void* wr, float* logits, int32_t* expert_idx,
                      float* gates, void* ws, void* stream) {
  MOE_TRY(moe_check_config(cfg));
  MOE_CHECK_ARG(x && wr && logits && expert_idx && gates, "moe_router: NULL pointer");
  const int T = (int)cfg->tokens, h = (int)cfg->hidden, E = (int)cfg->num_experts;
  if (router_on_tensor_cores(cfg)) return router_tc_launch(cfg, x, wr, logits, expert_idx, gates, ws, nullptr, stream);
  dim3 grid((unsigned)ceil_div(T, RT_TOK), (unsigned)ceil_div(E, RT_EXP));
  MOE_LAUNCH("router_logits", router_logits_kernel, dim3(grid), dim3(256), 0, as_stream(stream), reinterpret_cast<const __nv_bfloat16*>(x), reinterpret_cast<const __nv_bfloat16*>(wr), logits, T, h, E);
  return moe_topk(cfg, logits, expert_idx, gates, stream);
}

// Whether moe_router_topology builds the topology inside the router launch
// (MOE_ROUTER_TOPO_FUSED=1, read per call; default off): the tensor-core
// router, 128*k assignments per router tile within one CTA's threads (k <= 2).
// Measured at MoE-XS: 36.0 us fused against 28.7 us for the router plus the
// one-launch topology (the grid barrier and every CTA rescanning the
// histograms cost more than the launch they save).
static bool router_topo_fusable(const moe_config* cfg) {
  const char* e = getenv("MOE_ROUTER_TOPO_FUSED");
  return e && e[0] == '1' && router_on_tensor_cores(cfg) && cfg->top_k <= 2;
}

moe_status moe_router_topology(const moe_config* cfg, const void* x, const void* wr, float* logits,
                               int32_t* expert_idx, float* gates, const moe_topology_t* topo, void* ws, void* stream) {
  MOE_TRY(moe_check_config(cfg));
  MOE_TRY(check_topo(topo));
  MOE_CHECK_ARG(x && wr && logits && expert_idx && gates && ws, "moe_router_topology: NULL pointer");
  if (router_topo_fusable(cfg)) return router_tc_launch(cfg, x, wr, logits, expert_idx, gates, ws, topo, stream);
  MOE_TRY(moe_router(cfg, x, wr, logits, expert_idx, gates, ws, stream));
  return moe_topology_from_router(cfg, expert_idx, topo, ws, stream);
}

moe_status moe_router_bwd(const moe_config* cfg, const void* x, const void* wr, const float* logits,
                          const int32_t* expert_idx, const float* dgates, float* dwr, void* dx, void* ws,
                          void* stream) {
  MOE_TRY(moe_check_config(cfg));
  MOE_CHECK_ARG(x && wr && logits && expert_idx && dgates && dwr && dx && ws, "moe_router_bwd: NULL pointer");
  const int T = (int)cfg->tokens, h = (int)cfg->hidden, E = (int)cfg->num_experts, k = (int)cfg->top_k;
  const WsLayout WL = ws_layout(cfg);
  float* dlogits = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + WL.dlogits);
  float* part = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + WL.dwr_part);
  const float* aux_c =
      cfg->aux_loss_coeff > 0.f ? reinterpret_cast<const float*>(reinterpret_cast<char*>(ws) + WL.aux) + 1 : nullptr;
  cudaStream_t s = as_stream(stream);
  const int parts = router_bwd_parts(cfg);
  if (router_on_tensor_cores(cfg)) {
    __nv_bfloat16* dl16 = reinterpret_cast<__nv_bfloat16*>(dlogits);
    MOE_LAUNCH("router_dlogits", router_dlogits_kernel, dim3((int)ceil_div(T, 8)), dim3(256), 0, s, logits, expert_idx, dgates, nullptr, dl16, T, E, k,
               cfg->renormalize, aux_c);
    MOE_TRY(router_dwr_tc(cfg, x, dl16, dwr, ws, s));
    return router_dx_tc(cfg, dl16, wr, dx, dx, nullptr, 1, h, s);  // dx += dlogits . Wr^T (in place)
  }
  MOE_LAUNCH("router_dlogits", router_dlogits_kernel, dim3((int)ceil_div(T, 8)), dim3(256), 0, s, logits, expert_idx, dgates, dlogits, nullptr, T, E, k,
             cfg->renormalize, aux_c);
  const int tpp = (int)ceil_div(T, parts);
  MOE_LAUNCH("router_dwr_part", router_dwr_part_kernel, dim3(dim3(parts, (unsigned)ceil_div(h, 32))), dim3(256), 0, s, reinterpret_cast<const __nv_bfloat16*>(x), dlogits, part, T, h, E, tpp);
  MOE_LAUNCH("router_dwr_reduce", router_dwr_reduce_kernel, dim3((int)ceil_div((int64_t)h * E, 256)), dim3(256), 0, s, part, dwr, parts, h * E);
  const size_t smem = 8 * E * sizeof(float);
  if (smem > 48 * 1024) return set_error(MOE_EUNSUPPORTED, "router_bwd: num_experts too large");
  MOE_LAUNCH("router_dx", router_dx_kernel, dim3((int)ceil_div(T, 8)), dim3(256), smem, s, dlogits, reinterpret_cast<const __nv_bfloat16*>(wr), reinterpret_cast<__nv_bfloat16*>(dx), T, h, E);
  return MOE_OK;
}

}  // extern "C"

extern "C" {

moe_status moe_scatter_bwd_router(const moe_config* cfg, const void* dy, const void* y_g, const moe_topology_t* topo,
                                  const float* gates, const float* logits, const int32_t* expert_idx, void* dy_g,
                                  float* dgates, void* dlogits_bf16, void* stream) {
  MOE_TRY(moe_check_config(cfg));
  MOE_TRY(check_topo(topo));
  MOE_CHECK_ARG(dy && y_g && gates && logits && expert_idx && dy_g && dgates && dlogits_bf16,
                "moe_scatter_bwd_router: NULL pointer");
  if (!router_on_tensor_cores(cfg))
    return set_error(MOE_EUNSUPPORTED, "moe_scatter_bwd_router: needs E %% 64 == 0, E <= 256, top_k <= 8");
  return scatter_bwd_fused(cfg, dy, y_g, topo->pos, gates, dy_g, dgates, logits, expert_idx,
                           reinterpret_cast<__nv_bfloat16*>(dlogits_bf16), nullptr, topo, as_stream(stream));
}

}  // extern "C"

namespace moe {
// moe_scatter_bwd_router + the auxiliary loss's gradient (the layer's form)
moe_status scatter_bwd_router_aux(const moe_config* cfg, const void* dy, const void* y_g, const moe_topology_t* topo,
                                  const float* gates, const float* logits, const int32_t* expert_idx, void* dy_g,
                                  float* dgates, void* dlogits_bf16, const float* aux_c, cudaStream_t s) {
  return scatter_bwd_fused(cfg, dy, y_g, topo->pos, gates, dy_g, dgates, logits, expert_idx,
                           reinterpret_cast<__nv_bfloat16*>(dlogits_bf16), nullptr, topo, s, aux_c);
}

// Auxiliary load-balancing loss. Partials: CTA q owns tokens
// [q*T/P, (q+1)*T/P); each warp accumulates softmax probabilities of its tokens
// per expert in registers-backed shared rows, reduced in warp order.
__global__ void __launch_bounds__(256) aux_partial_kernel(const float* __restrict__ logits,
                                                          const int32_t* __restrict__ idx, int T, int E, int k,
                                                          float* __restrict__ part_p, int* __restrict__ part_c) {
  pdl_trigger();
  pdl_wait();  // logits / idx come from the router before it
  extern __shared__ float s_acc[];  // [8 warps][E] probabilities, then int [E] top-1 counts
  int* s_cnt = reinterpret_cast<int*>(s_acc + 8 * E);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 8 * E; i += blockDim.x) s_acc[i] = 0.f;
  for (int i = threadIdx.x; i < E; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  const int t0 = (int)((long long)blockIdx.x * T / gridDim.x), t1 = (int)((long long)(blockIdx.x + 1) * T / gridDim.x);
  for (int t = t0 + warp; t < t1; t += 8) {
    const float* row = logits + (size_t)t * E;
    float m = -FLT_MAX;
    for (int e = lane; e < E; e += 32) m = fmaxf(m, row[e]);
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float ssum = 0.f;
    for (int e = lane; e < E; e += 32) ssum += expf(row[e] - m);
    for (int o = 16; o > 0; o >>= 1) ssum += __shfl_xor_sync(0xffffffffu, ssum, o);
    const float inv = 1.f / ssum;
    for (int e = lane; e < E; e += 32) s_acc[warp * E + e] += expf(row[e] - m) * inv;
    if (lane == 0) atomicAdd(&s_cnt[idx[(size_t)t * k]], 1);  // integer: order-free
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    float a = 0.f;
    for (int w = 0; w < 8; ++w) a += s_acc[w * E + e];
    part_p[(size_t)blockIdx.x * E + e] = a;
    part_c[(size_t)blockIdx.x * E + e] = s_cnt[e];
  }
}

__global__ void __launch_bounds__(256) aux_final_kernel(const float* __restrict__ part_p,
                                                        const int* __restrict__ part_c, int parts, int T, int E,
                                                        float coeff, float* __restrict__ aux) {
  pdl_trigger();
  pdl_wait();  // the partials of aux_partial_kernel
  __shared__ float s_red[256];
  float acc = 0.f;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    float P = 0.f;
    long long c = 0;
    for (int q = 0; q < parts; ++q) {
      P += part_p[(size_t)q * E + e];
      c += part_c[(size_t)q * E + e];
    }
    const float f = (float)c / (float)T;
    aux[1 + e] = coeff * (float)E * f / (float)T;  // d loss / d p[t, e]
    acc += f * (P / (float)T);
  }
  s_red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {  // fixed-shape tree: deterministic
    if ((int)threadIdx.x < o) s_red[threadIdx.x] += s_red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) aux[0] = coeff * (float)E * s_red[0];
}

// dlogits[t, :] += p * (c - <p, c>) in place (bf16), c = the aux coefficients
__global__ void aux_dlogits_kernel(const float* __restrict__ logits, const float* __restrict__ aux_c,
                                   __nv_bfloat16* __restrict__ dlogits, int T, int E) {
  pdl_trigger();
  pdl_wait();  // dlogits from the scatter backward, aux_c from aux_final_kernel
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (t >= T) return;
  const float* row = logits + (size_t)t * E;
  float m = -FLT_MAX;
  for (int e = lane; e < E; e += 32) m = fmaxf(m, row[e]);
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float ssum = 0.f, pc = 0.f;
  for (int e = lane; e < E; e += 32) {
    const float q = expf(row[e] - m);
    ssum += q;
    pc += q * __ldg(aux_c + e);
  }
  for (int o = 16; o > 0; o >>= 1) {
    ssum += __shfl_xor_sync(0xffffffffu, ssum, o);
    pc += __shfl_xor_sync(0xffffffffu, pc, o);
  }
  const float inv = 1.f / ssum;
  pc *= inv;
  for (int e = lane; e < E; e += 32) {
    __nv_bfloat16* d = dlogits + (size_t)t * E + e;
    const float pe = expf(row[e] - m) * inv;
    *d = __float2bfloat16_rn(__bfloat162float(*d) + pe * (__ldg(aux_c + e) - pc));
  }
}
}  // namespace moe

extern "C" {

moe_status moe_load_balance_loss(const moe_config* cfg, const float* logits, const int32_t* expert_idx, void* ws,
                                 void* stream) {
  MOE_TRY(moe_check_config(cfg));
  MOE_CHECK_ARG(logits && expert_idx && ws, "moe_load_balance_loss: NULL pointer");
  const int T = (int)cfg->tokens, E = (int)cfg->num_experts, k = (int)cfg->top_k;
  const WsLayout WL = ws_layout(cfg);
  char* base = reinterpret_cast<char*>(ws) + WL.aux;
  float* aux = reinterpret_cast<float*>(base);
  float* part_p = aux + 1 + E;
  int* part_c = reinterpret_cast<int*>(part_p + (size_t)kAuxParts * E);
  const size_t smem = (size_t)8 * E * sizeof(float) + (size_t)E * sizeof(int);
  if (smem > 48 * 1024) return set_error(MOE_EUNSUPPORTED, "moe_load_balance_loss: num_experts=%d too large", E);
  cudaStream_t s = as_stream(stream);
  MOE_LAUNCH("aux_partial", aux_partial_kernel, dim3(kAuxParts), dim3(256), smem, s, logits, expert_idx, T, E, k, part_p,
             part_c);
  MOE_LAUNCH("aux_final", aux_final_kernel, dim3(1), dim3(256), 0, s, part_p, part_c, kAuxParts, T, E,
             cfg->aux_loss_coeff, aux);
  return MOE_OK;
}

moe_status moe_router_dwr(const moe_config* cfg, const void* x, const void* dlogits_bf16, float* dwr, void* ws,
                          void* stream) {
  MOE_TRY(moe_check_config(cfg));
  MOE_CHECK_ARG(x && dlogits_bf16 && dwr && ws, "moe_router_dwr: NULL pointer");
  if (!router_on_tensor_cores(cfg))
    return set_error(MOE_EUNSUPPORTED, "moe_router_dwr: needs E %% 64 == 0, E <= 256, top_k <= 8");
  return router_dwr_tc(cfg, x, reinterpret_cast<const __nv_bfloat16*>(dlogits_bf16), dwr, ws, as_stream(stream));
}

moe_status moe_router_dx(const moe_config* cfg, const void* dlogits_bf16, const void* wr, const void* dx_g,
                         const moe_topology_t* topo, void* dx, void* stream) {
  MOE_TRY(moe_check_config(cfg));
  MOE_TRY(check_topo(topo));
  MOE_CHECK_ARG(dlogits_bf16 && wr && dx_g && dx, "moe_router_dx: NULL pointer");
  if (!router_on_tensor_cores(cfg))
    return set_error(MOE_EUNSUPPORTED, "moe_router_dx: needs E %% 64 == 0, E <= 256, top_k <= 8");
  return router_dx_tc(cfg, reinterpret_cast<const __nv_bfloat16*>(dlogits_bf16), wr, dx, dx_g, topo->pos,
                      (int)cfg->top_k, cfg->hidden, as_stream(stream));
}

}  // extern "C"

extern "C" {

moe_status moe_unsort_rows_bwd_router(const moe_config* cfg, const void* dy, const void* y_sorted,
                                      const moe_topology_t* topo, const float* gates, const float* logits,
                                      const int32_t* expert_idx, void* dy_sorted, float* dgates,
                                      void* dlogits_bf16, void* stream) {
  MOE_TRY(moe_check_config(cfg));
  MOE_TRY(check_topo(topo));
  MOE_CHECK_ARG(dy && y_sorted && gates && logits && expert_idx && dy_sorted && dgates && dlogits_bf16,
                "moe_unsort_rows_bwd_router: NULL pointer");
  if (!router_on_tensor_cores(cfg))
    return set_error(MOE_EUNSUPPORTED, "moe_unsort_rows_bwd_router: needs E %% 64 == 0, E <= 256, top_k <= 8");
  // unpadded expert-order rows: sorted_pos map, no pad rows to zero
  return scatter_bwd_fused(cfg, dy, y_sorted, topo->sorted_pos, gates, dy_sorted, dgates, logits, expert_idx,
                           reinterpret_cast<__nv_bfloat16*>(dlogits_bf16), nullptr, nullptr, as_stream(stream));
}

moe_status moe_sort_rows_bwd_router(const moe_config* cfg, const void* dx_sorted, const moe_topology_t* topo,
                                    const void* dlogits_bf16, const void* wr, void* dx, void* stream) {
  MOE_TRY(moe_check_config(cfg));
  MOE_TRY(check_topo(topo));
  MOE_CHECK_ARG(dx_sorted && dlogits_bf16 && wr && dx, "moe_sort_rows_bwd_router: NULL pointer");
  if (!router_on_tensor_cores(cfg))
    return set_error(MOE_EUNSUPPORTED, "moe_sort_rows_bwd_router: needs E %% 64 == 0, E <= 256, top_k <= 8");
  // the dx GEMM's epilogue gathers the k rows itself (a coalesced re-sort followed by the GEMM with
  // contiguous addend rows measured slower at one-rank EP C1: 0.738-0.747 vs 0.725 ms/step)
  return router_dx_tc(cfg, reinterpret_cast<const __nv_bfloat16*>(dlogits_bf16), wr, dx, dx_sorted, topo->sorted_pos,
                      (int)cfg->top_k, cfg->hidden, as_stream(stream));
}

}  // extern "C"

extern "C" moe_status moe_add_aux_dlogits(const moe_config* cfg, const float* logits, void* dlogits_bf16, const void* ws,
                                          void* stream) {
  MOE_TRY(moe_check_config(cfg));
  MOE_CHECK_ARG(logits && dlogits_bf16 && ws, "moe_add_aux_dlogits: NULL pointer");
  if (!(cfg->aux_loss_coeff > 0.f)) return MOE_OK;
  const WsLayout WL = ws_layout(cfg);
  const float* aux_c = reinterpret_cast<const float*>(reinterpret_cast<const char*>(ws) + WL.aux) + 1;
  const int T = (int)cfg->tokens;
  MOE_LAUNCH("aux_dlogits", aux_dlogits_kernel, dim3((unsigned)ceil_div(T, 8)), dim3(256), 0, as_stream(stream),
             logits, aux_c, reinterpret_cast<__nv_bfloat16*>(dlogits_bf16), T, (int)cfg->num_experts);
  return MOE_OK;
}
