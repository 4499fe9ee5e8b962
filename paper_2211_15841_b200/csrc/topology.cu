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

// Scan + emit in one launch. Every CTA first recomputes, from the per-chunk
// histograms (G x E ints, L2-resident), the per-expert totals, the chunk
// prefix it needs and the E-long scans (bins, padded_bins, pair_bins) in
// shared memory; CTA 0 also publishes the global arrays. Then blocks
// [0, n_chunks) rank assignments stably (warp match_any + per-warp prefix) ->
// sorted_idx, pos, sorted_pos, and the remaining blocks emit the BCSR, COO and
// transpose entries, one thread per nonzero block, in closed form.
__global__ void __launch_bounds__(1024) topo_scan_emit_kernel(const int32_t* __restrict__ idx, int R, int E, int bs,
                                                               int F, int n_chunks,
                                                               const int32_t* __restrict__ chunk_counts,
                                                               moe_topology_t topo, int capacity, int n_rows,
                                                               int row_chunk, int rows_per_cta) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ int32_t s_dyn[];           // [32 warps][E] per-warp counts (ranking CTAs)
  __shared__ int32_t s_cnt[1024], s_start[1024], s_pstart[1024], s_pair[1024], s_base[1024];
  __shared__ int32_t s_tot[3];
  // n_chunks ranking CTAs; CTA b ranks assignments [b * span, (b+1) * span),
  // span = rows_per_cta * row_chunk <= 1024, i.e. histogram rows
  // [b * rows_per_cta, (b+1) * rows_per_cta) of chunk_counts [n_rows][E]
  // (row_chunk assignments per row: kTopoChunk from topo_hist, 128 tokens x k
  // from the router epilogue)
  const bool ranking = (int)blockIdx.x < n_chunks;
  const int span = rows_per_cta * row_chunk;
  const int warp_id = threadIdx.x >> 5, lane_id = threadIdx.x & 31;
  // (1) per-expert totals and (ranking CTAs) the exclusive base of the CTA's
  //     first row: the threads split into S = 1024 / E row slices x E experts
  //     (coalesced over e), each summing its slice's rows with independent
  //     loads; partial sums reduced over the slices in shared memory
  {
    const int S = 1024 / E;
    const int first = ranking ? (int)blockIdx.x * rows_per_cta : 0;
    const int t = threadIdx.x;
    if (t < S * E) {
      const int sl = t / E, e = t - sl * E;
      const int r0 = (int)((long long)n_rows * sl / S), r1 = (int)((long long)n_rows * (sl + 1) / S);
      int32_t tot = 0, pre = 0;
#pragma unroll 8
      for (int c = r0; c < r1; ++c) {
        const int32_t v = __ldg(chunk_counts + (size_t)c * E + e);
        tot += v;
        pre += c < first ? v : 0;
      }
      s_start[t] = tot;
      s_pstart[t] = pre;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      int32_t tot = 0, pre = 0;
      for (int sl = 0; sl < S; ++sl) {
        tot += s_start[sl * E + e];
        pre += s_pstart[sl * E + e];
      }
      s_base[e] = pre;
      s_cnt[e] = capacity > 0 ? min(tot, capacity) : tot;    // kept assignments (token dropping)
    }
  }
  __syncthreads();
  // (2) exclusive scans over experts (unpadded, padded group starts P:297, row
  //     pairs) by warp 0: lane l owns experts [l*per, (l+1)*per)
  if (warp_id == 0) {
    const int per = (E + 31) / 32;
    const int e0 = min(E, lane_id * per), e1 = min(E, e0 + per);
    int32_t a0 = 0, a1 = 0, a2 = 0;
    for (int e = e0; e < e1; ++e) {
      const int32_t c = s_cnt[e], pc = ((c + bs - 1) / bs) * bs;
      a0 += c;
      a1 += pc;
      a2 += (pc / bs + 1) / 2;
    }
    int32_t i0 = a0, i1 = a1, i2 = a2;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y0 = __shfl_up_sync(0xffffffffu, i0, o), y1 = __shfl_up_sync(0xffffffffu, i1, o),
                    y2 = __shfl_up_sync(0xffffffffu, i2, o);
      if (lane_id >= o) {
        i0 += y0;
        i1 += y1;
        i2 += y2;
      }
    }
    int32_t r0 = i0 - a0, r1 = i1 - a1, r2 = i2 - a2;
    for (int e = e0; e < e1; ++e) {
      const int32_t c = s_cnt[e], pc = ((c + bs - 1) / bs) * bs;
      s_start[e] = r0;
      s_pstart[e] = r1;
      s_pair[e] = r2;
      r0 += c;
      r1 += pc;
      r2 += (pc / bs + 1) / 2;
    }
    if (lane_id == 31) {
      s_tot[0] = i0;
      s_tot[1] = i1;
      s_tot[2] = i2;
    }
  }
  __syncthreads();
  const int Tp = s_tot[1];
  const int nnz = (Tp / bs) * F;
  if (blockIdx.x == 0) {
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      const int32_t c = s_cnt[e], pc = ((c + bs - 1) / bs) * bs;
      topo.counts[e] = c;
      topo.bins[e] = s_start[e] + c;
      topo.padded_bins[e] = s_pstart[e] + pc;
      topo.pair_bins[e] = s_pair[e] + (pc / bs + 1) / 2;
    }
    // transposed offsets of expert e's F block-columns: F*start/bs + j*pc/bs
    for (int q = threadIdx.x; q < E * F; q += blockDim.x) {
      const int e = q / F, j = q - e * F;
      const int32_t pc = ((s_cnt[e] + bs - 1) / bs) * bs;
      topo.t_col_offsets[q] = F * (s_pstart[e] / bs) + j * (pc / bs);
    }
    if (threadIdx.x == 0) {
      topo.t_col_offsets[E * F] = nnz;
      topo.row_offsets[Tp / bs] = nnz;
      topo.sizes[0] = Tp;
      topo.sizes[1] = nnz;
      topo.sizes[2] = s_tot[2];
    }
  }
  if (ranking) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 32 * E; i += blockDim.x) s_dyn[i] = 0;
    __syncthreads();
    const int i = blockIdx.x * span + threadIdx.x;
    const bool valid = (int)threadIdx.x < span && i < R;
    const int e = valid ? __ldg(idx + i) : E + lane;  // unique sentinel for inactive lanes
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    const unsigned lt = (1u << lane) - 1u;
    const int rank_w = __popc(peers & lt);
    if (valid && rank_w == 0) s_dyn[warp * E + e] = __popc(peers);
    __syncthreads();
    for (int x = threadIdx.x; x < E; x += blockDim.x) {
      int32_t run = 0;
      for (int w = 0; w < 32; ++w) {
        int32_t v = s_dyn[w * E + x];
        s_dyn[w * E + x] = run;
        run += v;
      }
    }
    __syncthreads();
    if (valid) {
      const int rank = s_base[e] + s_dyn[warp * E + e] + rank_w;  // within expert e, by flat id
      if (capacity > 0 && rank >= capacity) {  // dropped (keep-earliest)
        topo.sorted_pos[i] = -1;
        topo.pos[i] = -1;
        return;
      }
      const int u = s_start[e] + rank;
      const int p = s_pstart[e] + rank;
      topo.sorted_idx[u] = i;
      topo.sorted_pos[i] = u;
      topo.pos[i] = p;
      topo.row_src[p] = i;
    }
  } else {
    const int s = (blockIdx.x - n_chunks) * blockDim.x + threadIdx.x;
    if (s >= nnz) return;
    const int r = s / F, j = s - r * F;
    // expert of block-row r: last e with padded start <= r*bs (empty experts have no rows)
    int lo = 0, hi = E - 1;
    const int row0 = r * bs;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_pstart[mid] <= row0) lo = mid; else hi = mid - 1;
    }
    // (an empty expert e < E-1 starts where e+1 starts, so the last start <= row0
    // belongs to the non-empty owner of the row)
    const int e = lo;
    const int r0 = s_pstart[e] / bs;
    topo.row_indices[s] = r;
    topo.col_indices[s] = e * F + j;
    const int32_t pc = ((s_cnt[e] + bs - 1) / bs) * bs;
    if (j == 0) {
      topo.row_offsets[r] = s;
      // the unpadded layout (P:297 partial blocks at the fringe, R23): dense rows of block-row r
      const int i = r - r0;
      topo.brow_start[r] = s_start[e] + bs * i;
      topo.brow_rows[r] = min(bs, s_cnt[e] - bs * i);
    }
    // pad rows of this block-row (the tail of expert e's group) hold no
    // assignment: the row's F threads write them strided
    const int pad0 = s_pstart[e] + s_cnt[e];
    for (int q = max(row0, pad0) + j; q < row0 + bs && q < s_pstart[e] + pc; q += F) topo.row_src[q] = -1;
    const int qpos = F * (s_pstart[e] / bs) + j * (pc / bs) + (r - r0);
    topo.t_block_offsets[qpos] = s;
    topo.t_row_indices[qpos] = r;
  }
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
  MOE_TRY(moe_check_config(cfg));
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
  const int emit_smem = 32 * E * (int)sizeof(int32_t);
  static unsigned long long smem_mask = 0;
  static int smem_set = 0;
  if (emit_smem > 48 * 1024 - 21 * 1024) set_smem_attr_once(topo_scan_emit_kernel, emit_smem, smem_mask, smem_set);
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
  const int emit_smem = 32 * E * (int)sizeof(int32_t);
  static unsigned long long smem_mask = 0;
  static int smem_set = 0;
  if (emit_smem > 48 * 1024 - 21 * 1024) set_smem_attr_once(topo_scan_emit_kernel, emit_smem, smem_mask, smem_set);
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
  const int emit_smem = 32 * E * (int)sizeof(int32_t);
  static unsigned long long smem_mask = 0;
  static int smem_set = 0;
  if (emit_smem > 48 * 1024 - 21 * 1024) set_smem_attr_once(topo_scan_emit_kernel, emit_smem, smem_mask, smem_set);
  const int64_t max_nnz = moe_max_nnz_blocks(cfg);
  const int blk_ctas = (int)ceil_div(max_nnz, 1024);
  // the per-source histograms play the per-chunk ones; no assignment is ranked (R = 0)
  MOE_LAUNCH("topo_scan_emit", topo_scan_emit_kernel, dim3(nsources + blk_ctas), dim3(1024), emit_smem,
             as_stream(stream), (const int32_t*)nullptr, 0, E, bs, F, nsources, counts_per_source, *topo, 0, nsources, 1, 1);
  return MOE_OK;
}
