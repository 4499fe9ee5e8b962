// topology.cu — moe_topology: the permutation plan and the hybrid
// blocked-CSR-COO topology with transpose indices, built on the device in one
// stream-ordered pass with no host synchronisation (Fig. 5
// make_topology; "we create the metadata for the block-sparse matrix
// using a custom CUDA kernel ... construct the transposed metadata at this
// time"; P:242 COO row indices; P:290 transpose indices).
//
// Three launches:
//  1. topo_hist:   per-chunk expert histograms (shared-memory integer atomics:
//                  order-independent, so deterministic).
//  2. topo_scan:   one CTA: per-expert exclusive scan over chunks, counts, bins,
//                  padded_bins, {Tp, nnz}, t_col_offsets, row_offsets[end].
//  3. topo_emit:   (a) stable rank of every assignment within its expert
//                  (warp match_any + per-warp prefix) -> sorted_idx, pos,
//                  sorted_pos; (b) one thread per nonzero block emits the BCSR,
//                  COO and transpose entries in closed form.
#include <cuda_runtime.h>

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

// Block-wide exclusive scan helper over `n` ints in shared memory (n <= 4096),
// single CTA of 1024 threads, sequential per-thread segments + warp scan.
__device__ void block_exclusive_scan(int32_t* data, int n, int32_t* s_tmp, int32_t* total_out) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int per = (n + nt - 1) / nt;
  const int b = tid * per, e = min(n, b + per);
  int32_t local = 0;
  for (int i = b; i < e; ++i) local += data[i];
  // warp inclusive scan
  const int lane = tid & 31, w = tid >> 5;
  int32_t v = local;
  for (int o = 1; o < 32; o <<= 1) {
    int32_t y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  if (lane == 31) s_tmp[w] = v;
  __syncthreads();
  if (w == 0) {
    int32_t x = lane < (nt >> 5) ? s_tmp[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      int32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    s_tmp[lane] = x;  // inclusive per-warp totals
  }
  __syncthreads();
  int32_t run = (w > 0 ? s_tmp[w - 1] : 0) + v - local;  // exclusive start of this thread's segment
  for (int i = b; i < e; ++i) {
    int32_t d = data[i];
    data[i] = run;
    run += d;
  }
  if (total_out && tid == nt - 1) *total_out = run;
  __syncthreads();
}

__global__ void __launch_bounds__(1024) topo_scan_kernel(int32_t* __restrict__ chunk_counts, int n_chunks, int E,
                                                          int bs, int F, moe_topology_t topo) {
  pdl_trigger();
  pdl_wait();
  __shared__ int32_t s_counts[1024];
  __shared__ int32_t s_pad[1024];
  __shared__ int32_t s_tmp[32];
  __shared__ int32_t s_pairs[1024];
  __shared__ int32_t s_tot[3];
  // (1) per-expert exclusive scan over chunks (chunk_counts becomes chunk base rank)
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int32_t run = 0;
    for (int c0 = 0; c0 < n_chunks; c0 += 16) {
      int32_t v[16];  // batch the loads so they are in flight together
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = c0 + u < n_chunks ? chunk_counts[(size_t)(c0 + u) * E + e] : 0;
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        if (c0 + u < n_chunks) chunk_counts[(size_t)(c0 + u) * E + e] = run;
        run += v[u];
      }
    }
    s_counts[e] = run;
    s_pad[e] = ((run + bs - 1) / bs) * bs;
    s_pairs[e] = (s_pad[e] / bs + 1) / 2;  // same-expert block-row pairs
    topo.counts[e] = run;
  }
  __syncthreads();
  // (2) bins / padded_bins = inclusive cumsums (P:297 padding to a multiple of bs)
  block_exclusive_scan(s_counts, E, s_tmp, &s_tot[0]);
  block_exclusive_scan(s_pad, E, s_tmp, &s_tot[1]);
  block_exclusive_scan(s_pairs, E, s_tmp, &s_tot[2]);
  const int Tp = s_tot[1];
  const int nnz = (Tp / bs) * F;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int32_t c = topo.counts[e];
    const int32_t pc = ((c + bs - 1) / bs) * bs;
    topo.bins[e] = s_counts[e] + c;
    topo.padded_bins[e] = s_pad[e] + pc;
    topo.pair_bins[e] = s_pairs[e] + (pc / bs + 1) / 2;
    // transposed offsets of expert e's F block-columns: F*start/bs + j*pc/bs
    for (int j = 0; j < F; ++j) topo.t_col_offsets[e * F + j] = F * (s_pad[e] / bs) + j * (pc / bs);
  }
  if (threadIdx.x == 0) {
    topo.t_col_offsets[E * F] = nnz;
    topo.row_offsets[Tp / bs] = nnz;
    topo.sizes[0] = Tp;
    topo.sizes[1] = nnz;
    topo.sizes[2] = s_tot[2];
  }
}

// Part (a): blocks [0, n_chunks) rank assignments; part (b): remaining blocks
// emit the topology, one thread per potential nonzero block.
__global__ void __launch_bounds__(1024) topo_emit_kernel(const int32_t* __restrict__ idx, int R, int E, int bs, int F,
                                                          int n_chunks, const int32_t* __restrict__ chunk_base,
                                                          moe_topology_t topo) {
  pdl_trigger();
  pdl_wait();
  if ((int)blockIdx.x < n_chunks) {
    extern __shared__ int32_t s_w[];  // [32 warps][E] counts -> exclusive prefix over warps
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 32 * E; i += blockDim.x) s_w[i] = 0;
    __syncthreads();
    const int i = blockIdx.x * kTopoChunk + threadIdx.x;
    const bool valid = i < R;
    const int e = valid ? idx[i] : E + lane;  // unique sentinel for inactive lanes
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    const unsigned lt = (1u << lane) - 1u;
    const int rank_w = __popc(peers & lt);
    if (valid && rank_w == 0) s_w[warp * E + e] = __popc(peers);
    __syncthreads();
    for (int x = threadIdx.x; x < E; x += blockDim.x) {
      int32_t run = 0;
      for (int w = 0; w < 32; ++w) {
        int32_t v = s_w[w * E + x];
        s_w[w * E + x] = run;
        run += v;
      }
    }
    __syncthreads();
    if (valid) {
      const int rank = chunk_base[(size_t)blockIdx.x * E + e] + s_w[warp * E + e] + rank_w;
      const int c = topo.counts[e];
      const int pc = ((c + bs - 1) / bs) * bs;
      const int u = topo.bins[e] - c + rank;
      const int p = topo.padded_bins[e] - pc + rank;
      topo.sorted_idx[u] = i;
      topo.sorted_pos[i] = u;
      topo.pos[i] = p;
    }
  } else {
    const int s = (blockIdx.x - n_chunks) * blockDim.x + threadIdx.x;
    const int nnz = topo.sizes[1];
    if (s >= nnz) return;
    const int r = s / F, j = s - r * F;
    // expert of block-row r: first e with padded_bins[e] > r*bs
    int lo = 0, hi = E - 1;
    const int row0 = r * bs;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (topo.padded_bins[mid] > row0) hi = mid; else lo = mid + 1;
    }
    const int e = lo;
    const int pc = topo.padded_bins[e] - (e > 0 ? topo.padded_bins[e - 1] : 0);
    const int r0 = (topo.padded_bins[e] - pc) / bs;
    topo.row_indices[s] = r;
    topo.col_indices[s] = e * F + j;
    if (j == 0) topo.row_offsets[r] = s;
    const int qpos = topo.t_col_offsets[e * F + j] + (r - r0);
    topo.t_block_offsets[qpos] = s;
    topo.t_row_indices[qpos] = r;
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
  MOE_LAUNCH("topo_hist", topo_hist_kernel, dim3(n_chunks), dim3(kTopoChunk), E * sizeof(int32_t), s, expert_idx, R, E, chunk_counts);
  MOE_LAUNCH("topo_scan", topo_scan_kernel, dim3(1), dim3(1024), 0, s, chunk_counts, n_chunks, E, bs, F, *topo);
  const int emit_smem = 32 * E * (int)sizeof(int32_t);
  static int smem_set = 0;
  if (emit_smem > 48 * 1024 && smem_set < emit_smem) {
    cudaFuncSetAttribute(topo_emit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, emit_smem);
    smem_set = emit_smem;
  }
  const int64_t max_nnz = moe_max_nnz_blocks(cfg);
  const int blk_ctas = (int)ceil_div(max_nnz, 1024);
  MOE_LAUNCH("topo_emit", topo_emit_kernel, dim3(n_chunks + blk_ctas), dim3(1024), emit_smem, s, expert_idx, R, E, bs, F, n_chunks, chunk_counts, *topo);
  return MOE_OK;
}
