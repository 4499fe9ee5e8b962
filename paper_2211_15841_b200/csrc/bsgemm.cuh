// bsgemm.cuh — launch interface of the tcgen05 GEMM engine (bsgemm.cu), shared
// by the block-sparse products and the router's dense GEMMs.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/moe.h"

namespace moe {

enum GemmMode { SDD = 0, DSD_ROW = 1, DS_COL = 2, DDS_COL = 3, DDS_ROW = 4, DENSE = 5 };
enum EpiKind { EPI_STORE = 0, EPI_ACT_FWD = 1, EPI_ACT_BWD = 2, EPI_ROUTER = 3, EPI_F32 = 4, EPI_ADD_ROWS = 5 };

struct GemmParams {
  // sparse topology (device)
  const int32_t* sizes;  // {Tp, nnz}
  const int32_t* row_offsets;
  const int32_t* col_indices;
  const int32_t* row_indices;
  const int32_t* t_col_offsets;
  const int32_t* t_block_offsets;
  const int32_t* t_row_indices;
  const int32_t* pair_bins;    // [E] inclusive cumsum of same-expert block-row pairs
  const int32_t* padded_bins;  // [E]
  const int32_t* counts;       // [E] assignments (kept) per expert
  int n_block_cols;  // E*F
  int F;             // block-columns per expert
  int dense_tiles;   // output tiles along the dense dimension
  int k_dense;       // SDD contraction length
  // DENSE mode: tiles = splits x m_tiles x n_tiles, kiters_split K-steps of 64 per split
  int m_tiles, n_tiles, splits, kiters_split, k_iters_total;
  // epilogue
  int epi, act, has_pre;
  int aux_deriv;
  // branch-coded activation (DESIGN R24): EPI_ACT_FWD writes only the coded A
  // (no second output); EPI_ACT_BWD decodes act'(H) from the coded A source
  int act_code;
  int l2_c, l2_d;  // L2 priority of the tmap_c / tmap_d epilogue stores: 0 normal, 1 evict_last, 2 evict_first
  // DSD_ROW + scatter_y (top-1 only): y[t] = gate[t] * row p of the output, t = row_src[p]
  // (tile::scatter4 through tmap_d; pad rows dropped)
  int scatter_y, scatter_T, scatter_only;
  int extra_k;
  int gather_a, gather_k, gather_T;  // SDD / DDS_COL: A rows gathered from x [T, h] by row_src / k (OOB: zeros)  // DSD_ROW: dense K-steps appended per tile (A: tmap_e gathered by row_src, B: tmap_f)
  const int32_t* row_src;
  // unpadded dense layout (moe_config.unpadded, P:297 partial blocks at the fringe): dense rows of
  // block-row r start at brow_start[r], rows >= brow_rows[r] of its blocks are the fringe
  int unpadded;
  const int32_t* brow_start;
  const int32_t* brow_rows;
  const int32_t* sorted_idx;  // dense row u -> flat id (the token for top-1)
  const float* scatter_gates;  // EPI_ACT_FWD: the aux output is act'(H), not H; EPI_ACT_BWD: the source holds act'(H)
  int rows_valid;  // rows of the output that exist (DENSE: M)
  // EPI_ROUTER
  float* logits;
  int32_t* idx;
  float* gates;
  int E, topk;
  int renorm;  // gates divided by the sum of the token's k gates
  int32_t* hist_out;  // optional: per-tile expert histogram [m_tiles][E] of the selected experts (topology input)
  // EPI_ROUTER with topo_fused: after a grid barrier (cooperative launch) every CTA
  // builds the topology from hist_out (topo_body.cuh): router + top-k + topology in one launch
  int topo_fused, topo_bs, topo_F, topo_capacity;
  moe_topology_t topo;
  // EPI_F32
  float* out_f32;
  long long ld_f32, split_stride;
  // EPI_ADD_ROWS: out = acc + addend[row], or with addend_map:
  // out = acc + sum_{j < addend_k} addend[addend_map[row * addend_k + j]]
  const __nv_bfloat16* addend;
  long long ld_add;
  const int32_t* addend_map;
  int addend_k;
  // direct epilogue stores (MOE_EPI_DIRECT=1; default: TMA stores):
  // bf16 outputs of tmap_c / tmap_d written with coalesced st.global from a
  // per-warp shared-memory transpose; rows >= rows_c / rows_d are clipped as
  // the TMA store would clip them
  __nv_bfloat16* out_c;
  __nv_bfloat16* out_d;
  long long ldc, ldd, rows_c, rows_d;
  int direct;
  const unsigned long long* row_dst;  // DSD_ROW: output row p goes to address row_dst[p] (0: dropped)
  int kskip;     // DS_COL / DDS_COL: skip the second K-step of a column's last block-row when it holds <= 64 rows
  int h_direct;                    // CTA-pair SDD^T: act'(H) read by the epilogue lanes, not by TMA
  const __nv_bfloat16* h_src;      // ... from here ([nnz*128, 128] bf16)
  int tall;      // CTA-pair forward SDD: 64 x 64 (8 KB) store boxes staged by pairs of epilogue warps
  int sdd_half;
  int epi_alt;   // CTA-pair forward SDD (4 KB boxes): two epilogue warp groups drain alternate tiles  // CTA-pair SDD / SDD^T: an expert's lone last block-row runs as an M = 128 pair tile
  int wide;  // CTA-pair forward SDD: tmap_c / tmap_d have 64 x 32 boxes, 128 B swizzle (make_tmap_epi_wide)
  unsigned long long* trace;  // MOE_GEMM_TRACE: per-CTA per-tile timestamps (see gemm_trace_*)
  int mcast;    // DSD_ROW in 2-CTA clusters: the two column tiles of a block-row share A (each CTA
                // loads 64 of its 128 rows, multicast to both; MOE_DSD_MCAST)
  int reverse;  // walk the tiles last-to-first (reuse what the previous kernel left in L2)
  int dbg;  // experiment knobs (MOE_GEMM_DBG): 1 = no epilogue work, 2 = no MMA, 4 = no activation
           // math, 8 = no TMA loads, 64 = epilogue decoupled from the accumulator (timing only)
};

// Router backward on tcgen05 (router.cu): dWr = x^T . dlogits and
// dx = dlogits . Wr^T + addend (optionally gathered through addend_map).
moe_status router_dwr_tc(const moe_config* cfg, const void* x, const __nv_bfloat16* dlogits, float* dwr, void* ws,
                         cudaStream_t s);
moe_status scatter_bwd_router_aux(const moe_config* cfg, const void* dy, const void* y_g, const moe_topology_t* topo,
                                  const float* gates, const float* logits, const int32_t* expert_idx, void* dy_g,
                                  float* dgates, void* dlogits_bf16, const float* aux_c, cudaStream_t s);
moe_status router_dx_tc(const moe_config* cfg, const __nv_bfloat16* dlogits, const void* wr, void* dx,
                        const void* addend, const int32_t* addend_map, int addend_k, long long ld_add,
                        cudaStream_t s);

struct GemmLaunch {
  const char* name;
  int mode, bn;
  bool a_mn, b_mn, epi_h;
  int max_tiles;
  CUtensorMap ta, tb, tc, td, te, tf;
  GemmParams p;
};

moe_status gemm_launch(const GemmLaunch& L, cudaStream_t stream);
// Record a bf16 epilogue output (which 0: tmap_c, 1: tmap_d) for the direct-store epilogue.
inline void set_epi_out(GemmParams& p, int which, const void* ptr, long long rows, long long ld) {
  __nv_bfloat16* q = reinterpret_cast<__nv_bfloat16*>(const_cast<void*>(ptr));
  if (which == 0) {
    p.out_c = q;
    p.rows_c = rows;
    p.ldc = ld;
  } else {
    p.out_d = q;
    p.rows_d = rows;
    p.ldd = ld;
  }
}
// Persistent-grid size control for concurrent kernels (host, per thread):
// gemm_sm_budget() = SMs the next GEMM launches may use (default: all);
// set by moe_backward around the GEMMs that share the GPU with the router dWr.
int gemm_sm_budget();
void set_gemm_sm_budget(int sms);  // <= 0: all SMs
int gemm_dbg();
// Timeline tracing of the GEMM engine (debug only, env MOE_GEMM_TRACE=1):
// slot [launch][cta][tile][event], events: 0 producer first load, 1 MMA start,
// 2 MMA last commit, 3 epilogue got accumulator, 4 epilogue done.
constexpr int kTraceLaunches = 16, kTraceCtas = 160, kTraceTiles = 32, kTraceEvents = 14;
unsigned long long* gemm_trace_slot();

#ifdef __CUDACC__
__device__ __forceinline__ void trace_ev(const GemmParams& p, int tile_i, int ev) {
  if (p.trace && tile_i < kTraceTiles) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[((size_t)blockIdx.x * kTraceTiles + tile_i) * kTraceEvents + ev] = t;
  }
}

#endif
// CTA-pair (cta_group::2) variant for SDD / DSD_ROW / DS_COL / DDS_COL with
// 256 x 256 tiles (bsgemm2.cu); B boxes are 128 wide (each CTA's half).
moe_status gemm2_launch(const GemmLaunch& L, cudaStream_t stream);
bool gemm2_wide_h();   // the CTA-pair SDD^T takes 64 x 32 (4 KB) act'(H) / dH maps (else 32 x 32)
bool gemm2_h_coded();  // the CTA-pair SDD^T can decode the coded activation (R24)
bool gemm2_h_ring();   // the CTA-pair SDD^T runs the act'(H) ring epilogue (half pairs supported)
GemmParams gemm_params_topo(const moe_config* cfg, const moe_topology_t* topo);

}  // namespace moe
