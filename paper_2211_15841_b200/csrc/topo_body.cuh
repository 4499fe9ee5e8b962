// topo_body.cuh — the scan + emit of the topology (Fig. 5
// make_topology; P:235-242 hybrid blocked-CSR-COO; P:290 transpose indices;
// P:297 padding; "we create the metadata for the block-sparse matrix
// using a custom CUDA kernel ... construct the transposed metadata at this
// time") as a CTA-level device function over any block size, shared by the
// standalone topo_scan_emit_kernel (topology.cu) and the tensor-core router
// kernel's fused topology (bsgemm.cu), which runs it on every CTA after a grid
// barrier.
//
// Inputs: expert ids idx [R] (flat id i = t*k + j) and per-row expert
// histograms chunk_counts [n_rows][E], row q counting the assignments
// [q*row_chunk, (q+1)*row_chunk). Ranking group g (rows [g*rows_per_cta,
// (g+1)*rows_per_cta), span = rows_per_cta*row_chunk <= blockDim assignments)
// ranks its assignments stably within their expert; emitting covers the
// nonzero blocks s grid-stride. Every CTA recomputes the per-expert totals and
// scans in shared memory; the `publish` CTA writes the E-long arrays.
// Deterministic: integer atomics are not used; order-independent counts only.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/moe.h"

namespace moe {

struct TopoTask {
  int rank_first, rank_stride;  // ranking groups g = rank_first, +rank_stride, ... (< n_rank)
  int emit_first, emit_stride;  // emit chunks of blockDim blocks: c = emit_first, +emit_stride (-1: none)
  bool publish;                 // this CTA writes counts / bins / padded_bins / pair_bins / t_col_offsets / sizes
};

// Shared-memory scratch (int32): 5 * max(E, blockDim) + 4 + (blockDim / 32) * E.
__host__ __device__ inline int topo_body_smem_ints(int E, int nthreads) {
  const int m = E > nthreads ? E : nthreads;
  return 5 * m + 4 + (nthreads / 32) * E;
}

// Requires E <= blockDim.x (the router path: E <= 256 < 352 threads; the
// standalone kernel: 1024 threads, E <= 1024).
__device__ inline void topo_scan_emit_body(const int32_t* __restrict__ idx, int R, int E, int bs, int F, int n_rank,
                                           const int32_t* __restrict__ chunk_counts, const moe_topology_t& topo,
                                           int capacity, int n_rows, int row_chunk, int rows_per_cta,
                                           const TopoTask& tk, int32_t* sm) {
  const int nt = blockDim.x, nw = nt / 32;
  const int m = E > nt ? E : nt;
  int32_t* s_cnt = sm;
  int32_t* s_start = sm + m;
  int32_t* s_pstart = sm + 2 * m;
  int32_t* s_pair = sm + 3 * m;
  int32_t* s_base = sm + 4 * m;
  int32_t* s_tot = sm + 5 * m;
  int32_t* s_dyn = s_tot + 4;  // [nw][E] per-warp counts of a ranking group
  const int span = rows_per_cta * row_chunk;
  const int warp_id = threadIdx.x >> 5, lane_id = threadIdx.x & 31;
  // (1) per-expert totals: the threads split into S = nt / E row slices x E
  //     experts (coalesced over e), each summing its slice with independent loads.
  //     A CTA ranking exactly one group also sums the rows before its group in
  //     the same pass (its per-expert base, s_base), instead of a second pass.
  const bool one_group = tk.rank_first < n_rank && tk.rank_first + tk.rank_stride >= n_rank;
  const int first0 = one_group ? tk.rank_first * rows_per_cta : 0;
  {
    const int S = nt / E;
    const int t = threadIdx.x;
    if (t < S * E) {
      const int sl = t / E, e = t - sl * E;
      const int r0 = (int)((long long)n_rows * sl / S), r1 = (int)((long long)n_rows * (sl + 1) / S);
      int32_t tot = 0, pre = 0;
#pragma unroll 8
      for (int c = r0; c < r1; ++c) {
        const int32_t v = __ldg(chunk_counts + (size_t)c * E + e);
        tot += v;
        pre += c < first0 ? v : 0;
      }
      s_start[t] = tot;
      s_pstart[t] = pre;  // scratch until the scans
    }
    __syncthreads();
    for (int e = threadIdx.x; e < E; e += nt) {
      int32_t tot = 0, pre = 0;
      for (int sl = 0; sl < S; ++sl) {
        tot += s_start[sl * E + e];
        pre += s_pstart[sl * E + e];
      }
      s_cnt[e] = capacity > 0 ? min(tot, capacity) : tot;  // kept assignments (token dropping)
      s_base[e] = pre;
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
  if (tk.publish) {
    for (int e = threadIdx.x; e < E; e += nt) {
      const int32_t c = s_cnt[e], pc = ((c + bs - 1) / bs) * bs;
      topo.counts[e] = c;
      topo.bins[e] = s_start[e] + c;
      topo.padded_bins[e] = s_pstart[e] + pc;
      topo.pair_bins[e] = s_pair[e] + (pc / bs + 1) / 2;
    }
    // transposed offsets of expert e's F block-columns: F*start/bs + j*pc/bs
    for (int q = threadIdx.x; q < E * F; q += nt) {
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
  // (3) ranking groups: stable rank within the expert (warp match_any +
  //     per-warp prefix) -> sorted_idx, pos, sorted_pos, row_src
  __syncthreads();  // the publish above has read s_pair, reused as scratch below
  for (int g = tk.rank_first; g < n_rank; g += tk.rank_stride) {
    // this group's exclusive base per expert: rows [0, g*rows_per_cta) (already
    // summed in pass (1) when the CTA ranks one group)
    const int first = g * rows_per_cta;
    if (!one_group) {
      const int S = nt / E;
      const int t = threadIdx.x;
      if (t < S * E) {
        const int sl = t / E, e = t - sl * E;
        const int r0 = (int)((long long)first * sl / S), r1 = (int)((long long)first * (sl + 1) / S);
        int32_t pre = 0;
#pragma unroll 8
        for (int c = r0; c < r1; ++c) pre += __ldg(chunk_counts + (size_t)c * E + e);
        s_pair[m - 1 - t] = pre;  // s_pair's tail as scratch (the pair scan is no longer needed)
      }
      __syncthreads();
      for (int e = threadIdx.x; e < E; e += nt) {
        int32_t pre = 0;
        for (int sl = 0; sl < S; ++sl) pre += s_pair[m - 1 - (sl * E + e)];
        s_base[e] = pre;
      }
    }
    for (int i = threadIdx.x; i < nw * E; i += nt) s_dyn[i] = 0;
    __syncthreads();
    const int i = g * span + threadIdx.x;
    const bool valid = (int)threadIdx.x < span && i < R;
    const int e = valid ? __ldg(idx + i) : E + lane_id;  // unique sentinel for inactive lanes
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    const unsigned lt = (1u << lane_id) - 1u;
    const int rank_w = __popc(peers & lt);
    if (valid && rank_w == 0) s_dyn[warp_id * E + e] = __popc(peers);
    __syncthreads();
    for (int x = threadIdx.x; x < E; x += nt) {
      int32_t run = 0;
      for (int w = 0; w < nw; ++w) {
        int32_t v = s_dyn[w * E + x];
        s_dyn[w * E + x] = run;
        run += v;
      }
    }
    __syncthreads();
    if (valid) {
      const int rank = s_base[e] + s_dyn[warp_id * E + e] + rank_w;  // within expert e, by flat id
      if (capacity > 0 && rank >= capacity) {  // dropped (keep-earliest)
        topo.sorted_pos[i] = -1;
        topo.pos[i] = -1;
      } else {
        const int u = s_start[e] + rank;
        const int p = s_pstart[e] + rank;
        topo.sorted_idx[u] = i;
        topo.sorted_pos[i] = u;
        topo.pos[i] = p;
        topo.row_src[p] = i;
      }
    }
    __syncthreads();  // s_dyn / s_base reused by the next group
  }
  // (4) BCSR, COO and transpose entries, one thread per nonzero block, closed form
  if (tk.emit_first < 0) return;
  for (int s = tk.emit_first * nt + (int)threadIdx.x; s < nnz; s += tk.emit_stride * nt) {
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
      const int ii = r - r0;
      topo.brow_start[r] = s_start[e] + bs * ii;
      topo.brow_rows[r] = min(bs, s_cnt[e] - bs * ii);
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

}  // namespace moe
