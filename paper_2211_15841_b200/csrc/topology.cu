// topology.cu — moe_topology: the permutation plan and the hybrid
// blocked-CSR-COO topology with transpose indices, built on the device in one
// stream-ordered pass with no host synchronisation (Fig. 5
// make_topology; "we create the metadata for the block-sparse matrix
// using a custom CUDA kernel ... construct the transposed metadata at this
// time"; P:242 COO row indices; P:290 transpose indices).
//
// Two launches:
//  1. topo_hist:       per-chunk expert histograms (shared-memory integer
//                      atomics: order-independent, so deterministic).
//  2. topo_scan_emit:  every CTA rescans the chunk histograms in shared memory
//                      (counts, bins, padded_bins, pair_bins; CTA 0 publishes
//                      them with {Tp, nnz}, t_col_offsets, row_offsets[end]),
//                      then (a) ranks assignments stably within their expert
//                      (warp match_any + per-warp prefix) -> sorted_idx, pos,
//                      sorted_pos, or (b) emits the BCSR, COO and transpose
//                      entries, one thread per nonzero block, in closed form.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "topo_body.cuh"

namespace moe {

__global__ void topo_hist_kernel(const int32_t* __restrict__ idx, int R, int E, int32_t* __restrict__ chunk_counts) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ int32_t s_cnt[];
  for (int e = threadIdx.x; e < E; e += blockDim.x) s_cnt[e] = 0;
  __syncthreads();
  const int i = blockIdx.x * kTopoChunk + threadIdx.x;
  if (i < R) atomicAdd(&s_cnt[idx[i]], 1);
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) chunk_counts[(size_t)blockIdx.x * E + e] = s_cnt[e];
}

// Scan + emit in one launch (topo_scan_emit_kernel: CTAs [0, n_rank) rank,
// the others emit; topo_scan_emit_body is shared with the router kernel's
// fused topology, whose every CTA ranks and emits after a grid barrier).
__global__ void __launch_bounds__(1024) topo_scan_emit_kernel(const int32_t* __restrict__ idx, int R, int E, int bs,
                                                               int F, int n_chunks,
                                                               const int32_t* __restrict__ chunk_counts,
                                                               moe_topology_t topo, int capacity, int n_rows,
                                                               int row_chunk, int rows_per_cta) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ int32_t s_dyn[];
  const bool ranking = (int)blockIdx.x < n_chunks;
  TopoTask tk;
  tk.rank_first = ranking ? (int)blockIdx.x : n_chunks;  // emit CTAs rank nothing
  tk.rank_stride = n_chunks;
  tk.emit_first = ranking ? -1 : (int)blockIdx.x - n_chunks;
  tk.emit_stride = (int)gridDim.x - n_chunks;
  tk.publish = blockIdx.x == 0;
  topo_scan_emit_body(idx, R, E, bs, F, n_chunks, chunk_counts, topo, capacity, n_rows, row_chunk, rows_per_cta, tk,
                      s_dyn);
}


// Expert-parallel receive ids (moe_ep_recv_ids): segments (source q, local
// expert l) in arrival order, segment length counts_all[q*E + e0 + l]; every
// CTA rescans the P*E_l segment lengths in shared memory (E_l*P = E entries at
// most), then writes ids grid-stride with a binary search over the prefix.
__global__ void ep_recv_ids_kernel(const int32_t* __restrict__ counts_all, int P, int E, int e0, int El,
                                   int32_t* __restrict__ ids, long long max_rows) {
  pdl_trigger();
  pdl_wait();  // the gathered counts come from earlier kernels / copies
  extern __shared__ int32_t s_pre[];  // [P*El + 1] exclusive prefix
  const int nseg = P * El;
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int g = 0; g < nseg; ++g) {
      s_pre[g] = acc;
      acc += __ldg(counts_all + (size_t)(g / El) * E + e0 + g % El);
    }
    s_pre[nseg] = acc;
  }
  __syncthreads();
  const long long total = min((long long)s_pre[nseg], max_rows);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    int lo = 0, hi = nseg - 1;   // last segment with s_pre[g] <= i
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_pre[mid] <= i) lo = mid; else hi = mid - 1;
    }
    ids[i] = lo % El;
  }
}

}  // namespace moe

using namespace moe;

extern "C" moe_status moe_topology(const moe_config* cfg, const int32_t* expert_idx, const moe_topology_t* topo,
                                   void* ws, void* stream) {
  // the topology alone is generic in the block size (NEXT-3, "smaller tile
  // dimensions"): bs = 32 or 64 as well as 128; the products need bs = 128
  if (cfg && (cfg->block_size == 32 || cfg->block_size == 64)) {
    moe_config c128 = *cfg;
    c128.block_size = 128;
    MOE_CHECK_ARG(cfg->ffn_hidden % cfg->block_size == 0, "moe_topology: ffn_hidden %% block_size != 0");
    if (cfg->ffn_hidden % 128 == 0) MOE_TRY(moe_check_config(&c128));
  } else {
    MOE_TRY(moe_check_config(cfg));
  }
  MOE_TRY(check_topo(topo));
  MOE_CHECK_ARG(expert_idx && ws, "moe_topology: NULL expert_idx or workspace");
  const int R = (int)(cfg->tokens * cfg->top_k);
  const int E = (int)cfg->num_experts, bs = (int)cfg->block_size, F = (int)(cfg->ffn_hidden / cfg->block_size);
  const int n_chunks = (int)ceil_div(R, kTopoChunk);
  const WsLayout L = ws_layout(cfg);
  int32_t* chunk_counts = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(ws) + L.topo_chunk_counts);
  cudaStream_t s = as_stream(stream);
  MOE_LAUNCH("topo_hist", topo_hist_kernel, dim3(n_chunks), dim3(kTopoChunk), E * sizeof(int32_t), s, expert_idx, R, E,
             chunk_counts);
  const int emit_smem = topo_body_smem_ints(E, 1024) * (int)sizeof(int32_t);
  static unsigned long long smem_mask = 0;
  static int smem_set = 0;
  if (emit_smem > 48 * 1024) set_smem_attr_once(topo_scan_emit_kernel, emit_smem, smem_mask, smem_set);
  const int64_t max_nnz = moe_max_nnz_blocks(cfg);
  const int blk_ctas = (int)ceil_div(max_nnz, 1024);
  MOE_LAUNCH("topo_scan_emit", topo_scan_emit_kernel, dim3(n_chunks + blk_ctas), dim3(1024), emit_smem, s, expert_idx, R,
             E, bs, F, n_chunks, chunk_counts, *topo, (int)cfg->capacity, n_chunks, kTopoChunk, 1);
  return MOE_OK;
}

namespace moe {

moe_status topology_from_hist(const moe_config* cfg, const int32_t* expert_idx, const int32_t* hist, int n_rows,
                              int row_chunk, const moe_topology_t* topo, cudaStream_t s) {
  const int E = (int)cfg->num_experts, bs = (int)cfg->block_size, F = (int)(cfg->ffn_hidden / cfg->block_size);
  const int R = (int)(cfg->tokens * cfg->top_k);
  MOE_CHECK_ARG(row_chunk >= 1 && row_chunk <= 1024, "topology_from_hist: row_chunk=%d", row_chunk);
  const int rows_per_cta = 1024 / row_chunk;
  const int n_rank = (n_rows + rows_per_cta - 1) / rows_per_cta;
  const int emit_smem = topo_body_smem_ints(E, 1024) * (int)sizeof(int32_t);
  static unsigned long long smem_mask = 0;
  static int smem_set = 0;
  if (emit_smem > 48 * 1024) set_smem_attr_once(topo_scan_emit_kernel, emit_smem, smem_mask, smem_set);
  const int blk_ctas = (int)ceil_div(moe_max_nnz_blocks(cfg), 1024);
  MOE_LAUNCH("topo_scan_emit", topo_scan_emit_kernel, dim3(n_rank + blk_ctas), dim3(1024), emit_smem, s, expert_idx, R,
             E, bs, F, n_rank, hist, *topo, (int)cfg->capacity, n_rows, row_chunk, rows_per_cta);
  return MOE_OK;
}

}  // namespace moe

extern "C" moe_status moe_topology_from_router(const moe_config* cfg, const int32_t* expert_idx,
                                               const moe_topology_t* topo, void* ws, void* stream) {
  MOE_TRY(moe_check_config(cfg));
  MOE_TRY(check_topo(topo));
  MOE_CHECK_ARG(expert_idx && ws, "moe_topology_from_router: NULL pointer");
  if (!router_on_tensor_cores(cfg)) return moe_topology(cfg, expert_idx, topo, ws, stream);
  const int32_t* hist = reinterpret_cast<const int32_t*>(reinterpret_cast<char*>(ws) + ws_layout(cfg).router_hist);
  return topology_from_hist(cfg, expert_idx, hist, (int)((cfg->tokens + 127) / 128), (int)(128 * cfg->top_k), topo,
                            as_stream(stream));
}

extern "C" moe_status moe_ep_recv_ids(const int32_t* counts_all, int nranks, int num_experts, int e0, int local_experts,
                                      int32_t* ids, int64_t max_rows, void* stream) {
  MOE_CHECK_ARG(counts_all && ids, "moe_ep_recv_ids: NULL pointer");
  MOE_CHECK_ARG(nranks >= 1 && local_experts >= 1 && e0 >= 0 && e0 + local_experts <= num_experts && max_rows >= 0,
                "moe_ep_recv_ids: bad ranks/experts (P=%d E=%d e0=%d E_l=%d)", nranks, num_experts, e0, local_experts);
  const int nseg = nranks * local_experts;
  MOE_CHECK_ARG(nseg + 1 <= 12 * 1024, "moe_ep_recv_ids: %d segments exceed the shared-memory scan", nseg);
  if (max_rows == 0) return MOE_OK;
  const int ctas = (int)std::min<int64_t>(ceil_div(max_rows, 256), 4 * 148);
  MOE_LAUNCH("ep_recv_ids", ep_recv_ids_kernel, dim3(ctas), dim3(256), (nseg + 1) * sizeof(int32_t),
             as_stream(stream), counts_all, nranks, num_experts, e0, local_experts, ids, (long long)max_rows);
  return MOE_OK;
}

extern "C" moe_status moe_topology_counts(const moe_config* cfg, const int32_t* counts_per_source, int nsources,
                                          const moe_topology_t* topo, void* stream) {
  MOE_TRY(moe_check_config(cfg));
  MOE_TRY(check_topo(topo));
  MOE_CHECK_ARG(counts_per_source && nsources >= 1, "moe_topology_counts: NULL counts or nsources < 1");
  const int E = (int)cfg->num_experts, bs = (int)cfg->block_size, F = (int)(cfg->ffn_hidden / cfg->block_size);
  const int emit_smem = topo_body_smem_ints(E, 1024) * (int)sizeof(int32_t);
  static unsigned long long smem_mask = 0;
  static int smem_set = 0;
  if (emit_smem > 48 * 1024) set_smem_attr_once(topo_scan_emit_kernel, emit_smem, smem_mask, smem_set);
  const int64_t max_nnz = moe_max_nnz_blocks(cfg);
  const int blk_ctas = (int)ceil_div(max_nnz, 1024);
  // the per-source histograms play the per-chunk ones; no assignment is ranked (R = 0)
  MOE_LAUNCH("topo_scan_emit", topo_scan_emit_kernel, dim3(nsources + blk_ctas), dim3(1024), emit_smem,
             as_stream(stream), (const int32_t*)nullptr, 0, E, bs, F, nsources, counts_per_source, *topo, 0, nsources, 1, 1);
  return MOE_OK;
}
