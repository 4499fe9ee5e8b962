// bsgemm.cu — block-sparse SDD / DSD / DDS (and the router's dense GEMMs) on
// sm_100a tensor cores.
//
// The paper's products (§5.1; Triton notation P:177) over the
// hybrid blocked-CSR-COO topology with transpose indices
// (P:287-292). One persistent, warp-specialised kernel template serves all of
// them; the modes differ only in how a 128 x BN output tile enumerates its
// K-steps and where TMA fetches the two operand tiles from:
//
//   SDD     out blocks (r,c..c+BN/128)   K = dense dim; COO (row_indices, col_indices) lookup
//   DSD_ROW out [r-block, n-tile]         K walks the BCSR row r (row_offsets, col_indices)
//   DS_COL  out [c-block, n-tile]         K walks column c through the transpose index
//   DDS_COL out [m-tile, c..c+BN/128]     K walks column c through the transpose index
//   DDS_ROW out [m-tile, r-block]         K walks the BCSR row r
//   DENSE   out [m-tile, n-tile] (+split-K)  router logits, dWr, dx (router term)
//
// Transposition never moves values: a transposed sparse or dense operand is
// fed to tcgen05.mma as an MN-major instead of K-major shared-memory tile
// (descriptor bit), loaded by TMA from the same row-major storage.
// BN = 256 tiles pair two adjacent block-columns of the same expert (F even):
// they share their row set, so one walk of the transpose index serves both.
//
// Warp roles (1 CTA/SM): warps 0..NP-1 = TMA producers (stage s issued by warp
// s % NP), warp NP = TMEM allocator + single-thread MMA issuer, the next EPW
// warps = epilogue (two per TMEM lane quarter). Pipelines: STAGES-deep smem
// ring (full/empty mbarriers), double-buffered TMEM accumulator (tfull/tempty)
// so the epilogue of tile i overlaps the main loop of tile i+1. The epilogue
// stages bf16 results in 64B-swizzled shared memory and writes them with TMA
// bulk stores (or tile::scatter4 to token rows); the SDD forward writes act(H)
// and act'(H), the SDD^T epilogue prefetches the saved act'(H) by TMA. DSD_ROW
// tiles may append dense K-steps whose A rows are tile::gather4-ed (router dx).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <float.h>
#include <limits.h>
#include <stdio.h>
#include <stdlib.h>

#include <cooperative_groups.h>

#include "bsgemm.cuh"
#include "gemm_util.cuh"
#include "topo_body.cuh"
#include "common.cuh"
#include "sm100.cuh"
#include "tma.cuh"

#ifndef MOE_SDD_EPW
#define MOE_SDD_EPW 8
#endif
#ifndef MOE_GEMM_NP
#define MOE_GEMM_NP 2
#endif
#ifndef MOE_SDD_NBUF
#define MOE_SDD_NBUF 2
#endif

#ifndef MOE_DSD_EPW  // experiment: epilogue warps of the row-walk DSD (its scattered last-tile epilogue is exposed)
#define MOE_DSD_EPW 8
#endif
#ifndef MOE_DSD_NBUF
#define MOE_DSD_NBUF 2
#endif

#ifndef MOE_MAX_STAGES
#define MOE_MAX_STAGES 16
#endif

namespace moe {

using namespace sm100;

// Epilogue warps: 16 (four per TMEM lane quarter) for the wide block-sparse
// tiles, whose epilogues are store-latency bound; 8 elsewhere (router GEMMs,
// SDD^T whose H staging would not leave room for the operand ring).
__host__ __device__ constexpr int epi_warps(int mode, int bn, bool epi_h) {
  return (mode == SDD && bn == 256 && !epi_h) ? MOE_SDD_EPW : (mode == DSD_ROW && bn == 256) ? MOE_DSD_EPW : 8;
}
// Staging buffers per epilogue warp (stores in flight per warp).
__host__ __device__ constexpr int epi_bufs(int mode, int bn, bool epi_h) {
  return (mode == SDD && bn == 256 && !epi_h) ? MOE_SDD_NBUF : (mode == DSD_ROW && bn == 256) ? MOE_DSD_NBUF : 2;
}

// OCC = CTAs per SM: 1, or 2 for the router's forward GEMM under
// MOE_ROUTER_OCC=2 (its 128-row tiles are ~1.7 waves on one CTA per SM; two
// resident CTAs per SM take them in one wave, but with half the shared memory
// and 4 epilogue warps it measured slower). OCC 2 uses 4 epilogue warps.
template <int MODE, int BN, bool EPI_H, int OCC = 1>
struct Cfg {
  static constexpr int EPW = OCC == 2 ? 4 : epi_warps(MODE, BN, EPI_H);
  static constexpr int NP = MOE_GEMM_NP;           // TMA producer warps (stage s is issued by warp s % NP)
  static_assert(NP >= 1, "at least one producer warp");
  static constexpr int MMA_WARP = NP;
  static constexpr int EPI_WARP0 = NP + 1;
  static constexpr int THREADS = 32 * (NP + 1 + EPW);
  static constexpr int NBUF = epi_bufs(MODE, BN, EPI_H);
  static constexpr int EPI = EPW * NBUF * EPI_BUF;  // per-warp staging ring
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  // per-warp ring of prefetched act'(H) / coded-A chunks (SDD^T); two deep, so
  // that the coded-activation decode table (R24) fits beside three stages
  static constexpr int NH = 2;
  static constexpr int TAB = EPI_H ? ACT_CODE_BYTES : 0;
  // router epilogue exchange (+ the tile's expert histogram, E <= 256)
  static constexpr int XCH = MODE == DENSE ? 128 * (2 + 2 * kMaxRouterTopK) * 4 + 256 * 4 : 0;
  static constexpr int H_BYTES = EPI_H ? EPW * NH * EPI_BUF : 0;
  static constexpr int SMEM_CTA = OCC == 2 ? 113 * 1024 : SMEM_LIMIT;
  static constexpr int STAGES_RAW = (SMEM_CTA - SMEM_FIXED - EPI - H_BYTES - TAB - XCH) / STAGE;
  static constexpr int STAGES = STAGES_RAW > MOE_MAX_STAGES ? MOE_MAX_STAGES : STAGES_RAW;
  static constexpr int TMEM_COLS = 2 * BN <= 32 ? 32 : 2 * BN;
  static constexpr size_t SMEM = SMEM_FIXED + (size_t)STAGES * STAGE + EPI + H_BYTES + TAB + XCH;
  static_assert(STAGES >= 2, "not enough shared memory for two stages");
  static_assert(BN % 64 == 0 && BN <= 256, "BN must be 64, 128 or 256");
};

__device__ __forceinline__ int num_tiles(const GemmParams& p, int mode, int pair) {
  const int Tp = p.sizes ? p.sizes[0] : 0, nnz = p.sizes ? p.sizes[1] : 0;
  switch (mode) {
    case SDD: return nnz / pair;
    case DSD_ROW: return (Tp / BM) * p.dense_tiles;
    case DS_COL: return p.n_block_cols * p.dense_tiles;
    case DDS_COL: return (p.n_block_cols / pair) * p.dense_tiles;
    case DDS_ROW: return (Tp / BM) * p.dense_tiles;
    default: return p.splits * p.m_tiles * p.n_tiles;  // DENSE
  }
}

struct TileInfo {
  int kiters;
  int walk_begin;  // first storage index (row walk) or transpose position (column walk)
  int u, v;        // SDD: (block row, block col); DSD_ROW/DDS_ROW: (r, dense tile);
                   // DS_COL/DDS_COL: (block col, dense tile); DENSE: (m tile, n tile)
  int s;           // SDD: first block storage index; DENSE: split
  int drow;        // SDD / DSD_ROW: first dense row of block-row u (u*BM; brow_start[u] unpadded)
  int vr;          // SDD / DSD_ROW: rows of block-row u holding assignments (BM padded; brow_rows[u])
};

__device__ __forceinline__ TileInfo decode(const GemmParams& p, int mode, int pair, int tile) {
  TileInfo t;
  t.s = 0;
  t.walk_begin = 0;
  t.drow = 0;
  t.vr = BM;
  if (mode == SDD) {
    t.s = tile * pair;
    t.u = __ldg(p.row_indices + t.s);
    t.v = __ldg(p.col_indices + t.s);
    t.kiters = p.k_dense / BK;
    t.drow = p.unpadded ? __ldg(p.brow_start + t.u) : t.u * BM;
    if (p.unpadded) t.vr = __ldg(p.brow_rows + t.u);
  } else if (mode == DSD_ROW || mode == DDS_ROW) {
    t.u = tile / p.dense_tiles;
    t.v = tile % p.dense_tiles;
    t.drow = p.unpadded ? __ldg(p.brow_start + t.u) : t.u * BM;
    if (p.unpadded) t.vr = __ldg(p.brow_rows + t.u);
    const int b = __ldg(p.row_offsets + t.u), e = __ldg(p.row_offsets + t.u + 1);
    t.walk_begin = b;
    t.kiters = KPB * (e - b);
    t.s = t.kiters;  // sparse K-steps; DSD_ROW appends p.extra_k dense ones
    if (mode == DSD_ROW) t.kiters += p.extra_k;
  } else if (mode == DS_COL || mode == DDS_COL) {
    t.u = (tile / p.dense_tiles) * (mode == DDS_COL ? pair : 1);
    t.v = tile % p.dense_tiles;
    const int b = __ldg(p.t_col_offsets + t.u), e = __ldg(p.t_col_offsets + t.u + 1);
    t.walk_begin = b;
    t.kiters = KPB * (e - b);
    // the column's last block-row (its expert's fringe) holds <= 64 assignments:
    // its second K-step multiplies zero rows only (pad rows / zero sparse rows)
    // (the expert's count decides it: (count - 1) % 128 < 64; one load, off the index chain)
    if (KPB == 2 && p.kskip && e > b) {
      const int cnt = __ldg(p.counts + t.u / p.F);
      if (cnt > 0 && (cnt - 1) % BM < BM / 2) --t.kiters;
    }
  } else {  // DENSE: tile = (split * m_tiles + m) * n_tiles + n
    t.v = tile % p.n_tiles;
    const int rest = tile / p.n_tiles;
    t.u = rest % p.m_tiles;
    t.s = rest / p.m_tiles;
    const int k0 = t.s * p.kiters_split;
    const int left = p.k_iters_total - k0;
    t.kiters = left < p.kiters_split ? (left > 0 ? left : 0) : p.kiters_split;
  }
  return t;
}

// TMA coordinates (inner column, outer row) of the 64-column chunk `c` of the
// output tile, for the epilogue warp whose rows start at `row0` in the tile.
__device__ __forceinline__ void out_coords(const GemmParams& p, int mode, const TileInfo& t, int c, int row0,
                                           int BN, int& x, int& y) {
  const int col = c * EPI_COLS;
  switch (mode) {
    case SDD: {  // values as [nnz*128, 128]
      const int blk = t.s + col / 128;
      x = col % 128;
      y = blk * BM + row0;
      break;
    }
    case DSD_ROW: x = t.v * BN + col; y = t.drow + row0; break;
    case DS_COL: x = t.v * BN + col; y = t.u * BM + row0; break;
    case DDS_COL: x = t.u * 128 + col; y = t.v * BM + row0; break;
    case DDS_ROW: x = t.u * 128 + col; y = t.v * BM + row0; break;
    default: x = t.v * BN + col; y = t.u * BM + row0; break;  // DENSE
  }
}

// Issue the TMA boxes of K-step `kit` of tile t into the smem stage
// (completion on mbarrier fb). K-major operands are one 2-D box; MN-major
// operands are one 3-D box {64 elements, 64 K-rows, chunks} whose smem image is
// the [chunk][64 rows][128 B] layout of the MN-major UMMA descriptor (one TMA
// instruction per operand: the per-SM TMA issue rate, not bytes, limits small
// boxes; see scripts/micro/l2_tma_bw.cu).
// Loads of one operand side; a null map skips them (issue_stage's `part` mask).
__device__ __forceinline__ void ld2(void* dst, const CUtensorMap* m, uint64_t* fb, int c0, int c1) {
  if (m) tma_load_2d(dst, m, fb, c0, c1);
}
__device__ __forceinline__ void ld3(void* dst, const CUtensorMap* m, uint64_t* fb, int c0, int c1, int c2) {
  if (m) tma_load_3d(dst, m, fb, c0, c1, c2);
}
#define tma_load_2d ld2
#define tma_load_3d ld3
template <int MODE, bool A_MN, bool B_MN, int BN>
__device__ __forceinline__ void issue_stage(const CUtensorMap* ta, const CUtensorMap* tb, const GemmParams& p,
                                            const TileInfo& t, int kit, int sblk, int oblk, uint8_t* sa, uint8_t* sb,
                                            uint64_t* fb, int part = 3, int odrow = 0) {
  // odrow: first dense row of the walked block-row oblk (column walks: oblk*BM, brow_start[oblk] unpadded)
  const int kk = kit % KPB;
  if (!(part & 1)) ta = nullptr;  // A boxes skipped below
  if (!(part & 2)) tb = nullptr;
  if (MODE == SDD) {
    const int k0 = kit * BK;
    tma_load_2d(sa, ta, fb, k0, t.drow);
    if (B_MN)
      tma_load_3d(sb, tb, fb, 0, k0, t.v * 2);
    else
      tma_load_2d(sb, tb, fb, k0, t.v * 128);
  } else if (MODE == DSD_ROW) {
    tma_load_2d(sa, ta, fb, kk * BK, sblk * BM);
    if (B_MN)
      tma_load_3d(sb, tb, fb, 0, oblk * BM + kk * BK, t.v * (BN / 64));
    else
      tma_load_2d(sb, tb, fb, oblk * BM + kk * BK, t.v * BN);
  } else if (MODE == DS_COL) {
    tma_load_3d(sa, ta, fb, 0, sblk * BM + kk * BK, 0);
    if (B_MN)
      tma_load_3d(sb, tb, fb, 0, odrow + kk * BK, t.v * (BN / 64));
    else
      tma_load_2d(sb, tb, fb, odrow + kk * BK, t.v * BN);
  } else if (MODE == DDS_COL) {
    if (A_MN)
      tma_load_3d(sa, ta, fb, 0, odrow + kk * BK, t.v * 2);
    else
      tma_load_2d(sa, ta, fb, odrow + kk * BK, t.v * BM);
#pragma unroll
    for (int j = 0; j < BN / 128; ++j)  // blocks (r, c + j): storage sblk + j
      tma_load_3d(sb + j * (2 * BK * 128), tb, fb, 0, (sblk + j) * BM + kk * BK, 0);
  } else if (MODE == DDS_ROW) {
    if (A_MN)
      tma_load_3d(sa, ta, fb, 0, oblk * BM + kk * BK, t.v * 2);
    else
      tma_load_2d(sa, ta, fb, oblk * BM + kk * BK, t.v * BM);
    tma_load_2d(sb, tb, fb, kk * BK, sblk * BM);
  } else {  // DENSE
    const int k0 = (t.s * p.kiters_split + kit) * BK;
    if (A_MN)
      tma_load_3d(sa, ta, fb, 0, k0, t.u * 2);
    else
      tma_load_2d(sa, ta, fb, k0, t.u * BM);
    if (B_MN)
      tma_load_3d(sb, tb, fb, 0, k0, t.v * (BN / 64));
    else
      tma_load_2d(sb, tb, fb, k0, t.v * BN);
  }
}
#undef tma_load_2d
#undef tma_load_3d

template <int MODE, bool A_MN, bool B_MN, int BN, bool EPI_H, int OCC>
__global__ void __launch_bounds__(Cfg<MODE, BN, EPI_H, OCC>::THREADS, OCC)
    bsgemm_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                  const __grid_constant__ CUtensorMap tmap_c, const __grid_constant__ CUtensorMap tmap_d,
                  const __grid_constant__ CUtensorMap tmap_e, const __grid_constant__ CUtensorMap tmap_f,
                  const GemmParams p) {
  using C = Cfg<MODE, BN, EPI_H, OCC>;
  constexpr int STAGES = C::STAGES;
  constexpr int EPW = C::EPW;
  constexpr int NG = EPW / 4;  // epilogue warps per TMEM lane quarter
  constexpr int PAIR = (MODE == SDD || MODE == DDS_COL) ? BN / 128 : 1;
  constexpr int NCHUNK = BN / EPI_COLS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem_a + STAGES * A_BYTES;
  uint8_t* smem_epi = smem_b + STAGES * C::B_BYTES;
  uint8_t* smem_h = smem_epi + C::EPI;
  uint8_t* smem_tab = smem_h + C::H_BYTES;  // SDD^T: act'(H) decode table of the coded A (R24)
  uint8_t* smem_x = smem_tab + C::TAB;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_x + C::XCH);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* hbar = tempty + 2;  // [EPW][NH]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(hbar + C::NH * EPW);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], p.mcast ? 2 : 1);  // multicast A: both CTAs' MMAs free a stage
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], EPW);
    }
    for (int i = 0; i < C::NH * EPW; ++i) mbar_init(&hbar[i], 1);
    fence_barrier_init();
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
  }
  if (warp == C::MMA_WARP) tmem_alloc<C::TMEM_COLS>(tmem_holder);
  if (EPI_H && p.act_code) act_code_table_to_smem(smem_tab, g_act_code_tab);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  if (MODE == DSD_ROW && p.mcast) cluster_sync();  // the peer's barriers are initialised before its multicasts
  pdl_trigger();
  pdl_wait();  // operands and device-side sizes come from the previous kernels
  const int ntiles = num_tiles(p, MODE, PAIR);

  if (warp < C::NP) {
    // ===================== TMA producers (each warp walks; lane 0 issues its stages) =====================
    // One issuing thread sustains only a few TMA boxes in flight; NP warps
    // share the ring (stage s belongs to warp s % NP).
    int stage = 0;
    uint32_t phase = 0;
    int tile_i = 0;
    // SDD with gathered A (p.gather_a): the 128 token ids of a tile's rows come
    // from row_src (4 per lane), loaded one tile ahead into registers (the load
    // is only waited for at the next tile)
    auto tok_load = [&](int tl) -> int4 {
      if (tl >= ntiles) return make_int4(-1, -1, -1, -1);
      const int s0 = (p.reverse ? ntiles - 1 - tl : tl) * PAIR;
      return __ldg(reinterpret_cast<const int4*>(p.row_src + (size_t)(s0 / p.F) * BM) + lane);
    };
    int4 tok_next = make_int4(-1, -1, -1, -1);
    if (MODE == SDD && p.gather_a) tok_next = tok_load(blockIdx.x);
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tile_i) {
      const TileInfo t = decode(p, MODE, PAIR, p.reverse ? ntiles - 1 - tile : tile);
      if (lane == 0) trace_ev(p, tile_i, 0);
      int idx_a = 0, idx_b = 0, idx_c = 0;  // per-lane cached walk entries (32 sparse blocks at a time)
      int4 atok = make_int4(0, 0, 0, 0);
      if (MODE == SDD && p.gather_a) {
        const int4 r = tok_next;
        tok_next = tok_load(tile + gridDim.x);
        const int oob = p.gather_T, kq = p.gather_k;
        atok = make_int4(r.x >= 0 ? r.x / kq : oob, r.y >= 0 ? r.y / kq : oob, r.z >= 0 ? r.z / kq : oob,
                         r.w >= 0 ? r.w / kq : oob);
      }
      int4 gtok = make_int4(0, 0, 0, 0);
      if (MODE == DSD_ROW && p.extra_k) {  // tokens of the tile's rows 4*lane .. 4*lane+3
        const int oob = p.scatter_T;
        if (p.unpadded) {  // dense row drow + r holds flat id sorted_idx[drow + r] (= the token, top-1)
          const int r = 4 * lane;
          gtok = make_int4(r < t.vr ? __ldg(p.sorted_idx + t.drow + r) : oob,
                           r + 1 < t.vr ? __ldg(p.sorted_idx + t.drow + r + 1) : oob,
                           r + 2 < t.vr ? __ldg(p.sorted_idx + t.drow + r + 2) : oob,
                           r + 3 < t.vr ? __ldg(p.sorted_idx + t.drow + r + 3) : oob);
        } else {
          const int4 src = __ldg(reinterpret_cast<const int4*>(p.row_src + t.u * BM) + lane);
          gtok = make_int4(src.x >= 0 ? src.x : oob, src.y >= 0 ? src.y : oob, src.z >= 0 ? src.z : oob,
                           src.w >= 0 ? src.w : oob);
        }
      }
      for (int kit = 0; kit < t.kiters; ++kit) {
        const int blk = kit / KPB, kk = kit % KPB;
        if (MODE != SDD && MODE != DENSE && (blk & 31) == 0 && kk == 0 && (MODE != DSD_ROW || kit < t.s)) {
          const int q = t.walk_begin + blk + lane;
          if (q < t.walk_begin + (t.kiters + KPB - 1) / KPB) {  // (a skipped last half K-step still needs its block)
            if (MODE == DSD_ROW || MODE == DDS_ROW) {
              idx_a = q;
              idx_b = __ldg(p.col_indices + q);
            } else {
              idx_a = __ldg(p.t_block_offsets + q);
              idx_b = __ldg(p.t_row_indices + q);
              idx_c = p.unpadded ? __ldg(p.brow_start + idx_b) : idx_b * BM;
            }
          }
        }
        const int sblk = __shfl_sync(0xffffffffu, idx_a, blk & 31);
        const int oblk = __shfl_sync(0xffffffffu, idx_b, blk & 31);
        const int odrow = __shfl_sync(0xffffffffu, idx_c, blk & 31);
        const bool mine = stage % C::NP == warp;
        if (mine) mbar_wait_sleep(&empty[stage], phase ^ 1);
        if (mine && MODE == DSD_ROW && kit >= t.s) {
          // appended dense K-steps (dsdT + router dx): A = dlogits rows of the
          // tile's tokens, gathered 4 rows per lane (tile::gather4; pad rows are
          // out of range -> zeros), B = Wr^T
          const int ke = kit - t.s;
          if (lane == 0) mbar_arrive_expect_tx(&full[stage], C::STAGE);
          __syncwarp();
          tma_gather4(smem_a + stage * A_BYTES + lane * 512, &tmap_e, &full[stage], ke * BK, gtok.x, gtok.y, gtok.z,
                      gtok.w);
          if (lane == 0) tma_load_2d(smem_b + stage * C::B_BYTES, &tmap_f, &full[stage], ke * BK, t.v * BN);
        } else if (mine && MODE == SDD && p.gather_a) {
          // A rows gathered from x by token (tile::gather4, 4 rows per lane; pad rows -> zeros)
          if (lane == 0) mbar_arrive_expect_tx(&full[stage], C::STAGE);
          __syncwarp();
          tma_gather4(smem_a + stage * A_BYTES + lane * 4 * KSW, &tmap_a, &full[stage], kit * BK, atok.x, atok.y,
                      atok.z, atok.w);
          if (lane == 0)
            issue_stage<MODE, A_MN, B_MN, BN>(&tmap_a, &tmap_b, p, t, kit, sblk, oblk, smem_a + stage * A_BYTES,
                                              smem_b + stage * C::B_BYTES, &full[stage], 2);
        } else if (mine && lane == 0) {
          uint64_t* fb = &full[stage];
          if (p.dbg & 8) {
            mbar_arrive(fb);
          } else {
            mbar_arrive_expect_tx(fb, C::STAGE);
            if (MODE == DSD_ROW && p.mcast) {
              // the cluster's CTAs hold the two column tiles of one block-row: each
              // loads 64 of the A block's 128 rows into both (128 B swizzle atoms are 8 rows)
              const uint32_t r = cluster_ctarank();
              tma_load_2d_mcast(smem_a + stage * A_BYTES + r * (BM / 2) * KSW, &tmap_a, fb, (kit % KPB) * BK,
                                sblk * BM + (int)r * (BM / 2), 0x3);
              issue_stage<MODE, A_MN, B_MN, BN>(&tmap_a, &tmap_b, p, t, kit, sblk, oblk, smem_a + stage * A_BYTES,
                                                smem_b + stage * C::B_BYTES, fb, 2, odrow);
            } else {
              issue_stage<MODE, A_MN, B_MN, BN>(&tmap_a, &tmap_b, p, t, kit, sblk, oblk, smem_a + stage * A_BYTES,
                                                smem_b + stage * C::B_BYTES, fb, 3, odrow);
            }
          }
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == C::MMA_WARP) {
    // ===================== MMA issuer (one thread) =====================
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(BM, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int tile_i = -1;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const TileInfo t = decode(p, MODE, PAIR, p.reverse ? ntiles - 1 - tile : tile);
        ++tile_i;
        if (t.kiters == 0) continue;
        if (!(p.dbg & 64)) mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        trace_ev(p, tile_i, 1);
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kit = 0; kit < t.kiters; ++kit) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(smem_a + stage * A_BYTES);
          const uint32_t b_base = smem_u32(smem_b + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t adesc =
                A_MN ? make_sdesc(a_base + k * 2048, BK * 128, 1024) : make_sdesc(a_base + k * 32, 16, KSW * 8, KSW);
            const uint64_t bdesc =
                B_MN ? make_sdesc(b_base + k * 2048, BK * 128, 1024) : make_sdesc(b_base + k * 32, 16, KSW * 8, KSW);
            if (!(p.dbg & 2)) mma_bf16(d_tmem, adesc, bdesc, idesc, (kit | k) != 0);
          }
          if (MODE == DSD_ROW && p.mcast)
            mma_commit_mcast(&empty[stage], 0x3);  // the stage may be refilled by either CTA's multicast
          else
            mma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(&tfull[acc]);
        trace_ev(p, tile_i, 2);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // ===================== epilogue (warps 2 .. 2+EPW-1) =====================
    // Warp w reads TMEM lane quarter w % 4 (rows 32q..32q+31 of the tile) and
    // the 32-column chunks c = grp, grp + NG, ... (grp = (w - 2) / 4). The
    // TMEM load of the next chunk is in flight while the current one is
    // processed and stored.
    const int q = warp & 3;
    const int wq = warp - C::EPI_WARP0;
    const int grp = wq >> 2;
    const int row0 = q * 32;
    uint8_t* stg = smem_epi + wq * C::NBUF * EPI_BUF;
    uint8_t* hst = smem_h + wq * C::NH * EPI_BUF;
    uint64_t* hb = hbar + wq * C::NH;
    int sbuf = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    const bool bf16_out = p.epi == EPI_STORE || p.epi == EPI_ACT_FWD || p.epi == EPI_ACT_BWD || p.epi == EPI_ADD_ROWS;

    // L2 priority of the two epilogue outputs (GemmParams::l2_c / l2_d)
    const uint64_t pol_c = l2_policy(p.l2_c), pol_d = l2_policy(p.l2_d);
    // Direct stores: the warp's 32 x 32 bf16 chunk goes through its staging
    // buffer (conflict-free swizzled rows), is read back 4 lanes per 64-byte
    // row segment and written with coalesced 16-byte st.global (8 rows per
    // instruction): the epilogue does not queue behind the TMA unit, which
    // stays with the operand loads. `tok` maps staging row -> output row
    // (scatter to token rows; < 0 or >= rows: dropped).
    TileInfo cur_tile{};  // the tile being stored (row clipping of the unpadded layout)
    auto store_direct = [&](__nv_bfloat16* base, long long ld, long long nrows, const float* v, int x, int y,
                            int tok_of_lane) {
      uint8_t* buf = stg + sbuf * EPI_BUF;
      stage_row(buf, lane, v);
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = i * 8 + (lane >> 2), j = lane & 3;
        uint4 w;
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                     : "r"(smem_u32(buf) + r * 64 + swz64(j, r))
                     : "memory");
        const long long row = tok_of_lane == INT_MIN ? (long long)y + r : (long long)__shfl_sync(0xffffffffu, tok_of_lane, r);
        if (row >= 0 && row < nrows)
          *reinterpret_cast<uint4*>(base + row * ld + x + j * 8) = w;
      }
      sbuf = sbuf + 1 == C::NBUF ? 0 : sbuf + 1;  // the other buffer next: one __syncwarp per chunk
    };
    // moe_dsd_rows: this lane's output row goes to the address row_dst[y + lane]
    // (the EP combine fused into the DSD: a peer's return window; 0: pad row)
    auto store_rows_ptr = [&](const float* v, int x, int y) {
      uint8_t* buf = stg + sbuf * EPI_BUF;
      stage_row(buf, lane, v);
      const unsigned long long mine_p = __ldg(p.row_dst + y + lane);
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = i * 8 + (lane >> 2), j = lane & 3;
        uint4 w;
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                     : "r"(smem_u32(buf) + r * 64 + swz64(j, r))
                     : "memory");
        const unsigned long long rp = __shfl_sync(0xffffffffu, mine_p, r);
        if (rp) *reinterpret_cast<uint4*>(rp + 2ull * (unsigned long long)(x + j * 8)) = w;
      }
      sbuf = sbuf + 1 == C::NBUF ? 0 : sbuf + 1;
    };
    auto store_chunk = [&](const CUtensorMap* map, const float* v, int x, int y) {
      if (MODE == DSD_ROW && p.row_dst && map == &tmap_c) {
        store_rows_ptr(v, x, y);
        return;
      }
      if (MODE == DSD_ROW && p.unpadded && map == &tmap_c) {
        // the tile's block-row ends at the fringe (the rows below belong to the
        // next expert): warps with rows past it store row-clipped
        const TileInfo& tc = cur_tile;
        if (row0 + 32 > tc.vr) {
          store_direct(p.out_c, p.ldc, (long long)tc.drow + tc.vr, v, x, y, INT_MIN);
          return;
        }
      }
      if (p.direct) {
        if (map == &tmap_c)
          store_direct(p.out_c, p.ldc, p.rows_c, v, x, y, INT_MIN);
        else
          store_direct(p.out_d, p.ldd, p.rows_d, v, x, y, INT_MIN);
        return;
      }
      if (lane == 0) bulk_wait_read<C::NBUF - 1>();  // the store issued from this buffer NBUF stores ago has read it
      __syncwarp();
      stage_row(stg + sbuf * EPI_BUF, lane, v);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        const int kind = map == &tmap_c ? p.l2_c : p.l2_d;
        if (kind)
          tma_store_2d_hint(map, stg + sbuf * EPI_BUF, x, y, map == &tmap_c ? pol_c : pol_d);
        else
          tma_store_2d(map, stg + sbuf * EPI_BUF, x, y);
        bulk_commit();
      }
      sbuf = sbuf + 1 == C::NBUF ? 0 : sbuf + 1;
    };
    // the same for 16 bf16x2 words already packed (the coded A, R24)
    auto store_chunk_raw = [&](const CUtensorMap* map, const uint32_t* w, int x, int y) {
      if (lane == 0) bulk_wait_read<C::NBUF - 1>();
      __syncwarp();
      stage_row_raw(stg + sbuf * EPI_BUF, lane, w);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(map, stg + sbuf * EPI_BUF, x, y);
        bulk_commit();
      }
      sbuf = sbuf + 1 == C::NBUF ? 0 : sbuf + 1;
    };
    const uint32_t tab_smem = smem_u32(smem_tab);
    // SDD^T: this warp's act'(H) chunks form one sequence j = 0, 1, ... over
    // its tiles (tile blockIdx.x + (j / NPW) * gridDim.x, chunk grp + (j % NPW) * NG),
    // prefetched NH ahead into a ring, so the loads overlap the main loop.
    constexpr int NPW_ = NCHUNK / NG;
    const int my_tiles = ntiles > (int)blockIdx.x ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const int hseq_end = my_tiles * NPW_;
    int hseq = 0;  // next item to consume
    auto load_h = [&](int j) {
      if (j < hseq_end && lane == 0) {
        fence_proxy_async_smem();  // prior generic reads of this buffer before the async write
        const int tile_j = (int)blockIdx.x + (j / NPW_) * (int)gridDim.x;
        const TileInfo tj = decode(p, MODE, PAIR, p.reverse ? ntiles - 1 - tile_j : tile_j);
        int x, y;
        out_coords(p, MODE, tj, grp + (j % NPW_) * NG, row0, BN, x, y);
        const int b = j % C::NH;
        mbar_arrive_expect_tx(&hb[b], EPI_BUF);
        tma_load_2d(hst + b * EPI_BUF, &tmap_d, &hb[b], x, y);
      }
    };
    if (EPI_H && p.epi == EPI_ACT_BWD)
      for (int j = 0; j < C::NH; ++j) load_h(j);

    uint4 pre_next[MODE == DENSE ? NCHUNK / NG : 1][4];
    auto addend_prefetch = [&](int tl, uint4 (&dst)[MODE == DENSE ? NCHUNK / NG : 1][4]) {
      if (tl >= ntiles) return;
      const TileInfo tn = decode(p, MODE, PAIR, tl);
      const int trow = tn.u * BM + row0 + lane;
      if (trow >= p.rows_valid) return;
      const int m = p.addend_map ? __ldg(p.addend_map + (long long)trow * p.addend_k) : trow;
      const __nv_bfloat16* rowp = p.addend + (long long)m * p.ld_add + (long long)tn.v * BN;
#pragma unroll
      for (int i = 0; i < (MODE == DENSE ? NCHUNK / NG : 1); ++i) {
        const uint4* src = reinterpret_cast<const uint4*>(rowp + (grp + i * NG) * EPI_COLS);
#pragma unroll
        for (int q2 = 0; q2 < 4; ++q2) dst[i][q2] = m >= 0 ? __ldg(src + q2) : make_uint4(0u, 0u, 0u, 0u);
      }
    };
    int tile_i = -1;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const TileInfo t = decode(p, MODE, PAIR, p.reverse ? ntiles - 1 - tile : tile);
      cur_tile = t;
      ++tile_i;
      const bool has_acc = (p.dbg & 64) ? false : t.kiters > 0;
      // unpadded layout: this lane's row of an SDD tile is past the block-row's
      // assignments (the fringe): its values are written as exact zeros
      const bool fringe = MODE == SDD && p.unpadded && row0 + lane >= t.vr;
      // DENSE + EPI_ADD_ROWS: this lane's addend rows for all of its chunks are
      // in registers before the accumulator is waited for; the next tile's rows
      // are loaded now, so the gather latency overlaps this tile's epilogue.
      constexpr int NPW0 = NCHUNK / NG;
      uint4 pre[MODE == DENSE ? NPW0 : 1][4];
      int my_tok = 0x7fffffff;  // scatter target row (out of range: dropped)
      float my_gate = 0.f;
      if (MODE == DSD_ROW && p.scatter_y) {
        const int src = p.unpadded ? (row0 + lane < t.vr ? __ldg(p.sorted_idx + t.drow + row0 + lane) : -1)
                                   : __ldg(p.row_src + t.u * BM + row0 + lane);
        if (src >= 0) {
          my_tok = src;
          my_gate = p.scatter_gates ? __ldg(p.scatter_gates + src) : 1.f;
        }
      }
      if (MODE == DENSE && p.epi == EPI_ADD_ROWS) {
        if (tile_i == 0) addend_prefetch(tile, pre_next);
#pragma unroll
        for (int i = 0; i < (MODE == DENSE ? NPW0 : 1); ++i)
#pragma unroll
          for (int q2 = 0; q2 < 4; ++q2) pre[i][q2] = pre_next[i][q2];
        addend_prefetch(tile + (int)gridDim.x, pre_next);
      }
      if (has_acc) {
        mbar_wait_sleep(&tfull[acc], acc_phase);
        tc_fence_after();
      }
      if (wq == 0 && lane == 0) trace_ev(p, tile_i, 3);
      const uint32_t taddr = tmem_base + ((uint32_t)row0 << 16) + acc * BN;

      if (p.dbg & 1) {
        if (has_acc) {
          uint32_t r[32];
          tmem_ld32(taddr, r);
          tmem_ld_wait();
          if (r[0] == 0x7fffffffu && r[1] == 0x12345u) p.gates[0] = 1.f;
        }
      } else if (bf16_out) {
        // NPW chunks per warp, fully unrolled with ping-pong TMEM registers
        // (the next chunk's tcgen05.ld is in flight while this one is processed).
        constexpr int NPW = NCHUNK / NG;
        static_assert(NCHUNK % NG == 0, "chunks must divide evenly over the epilogue warps");
        // DENSE kernels keep registers for the prefetched addend rows instead
        constexpr bool PP = MODE != DENSE;
        uint32_t rr[PP ? 2 : 1][32];
        if (has_acc && PP) {
          tmem_ld32(taddr + grp * EPI_COLS, rr[0]);
          tmem_ld_wait();
        }
#pragma unroll
        for (int i = 0; i < NPW; ++i) {
          const int c = grp + i * NG;
          float v[32];
          if (has_acc) {
            if (!PP) {
              tmem_ld32(taddr + c * EPI_COLS, rr[0]);
              tmem_ld_wait();
            }
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(rr[PP ? (i & 1) : 0][e]);
            if (PP && i + 1 < NPW) tmem_ld32(taddr + (c + NG) * EPI_COLS, rr[PP ? ((i + 1) & 1) : 0]);  // next chunk, in flight
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = 0.f;
          }
          if (fringe) {
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = 0.f;
          }
          int x, y;
          out_coords(p, MODE, t, c, row0, BN, x, y);
          uint32_t wcode[16];
          bool coded_out = false;
          if (MODE == SDD && p.epi == EPI_ACT_FWD && p.act_code) {  // coded A only (R24)
            act_fwd_code32(p.act, v, wcode);
            coded_out = true;
          } else if (p.epi == EPI_ACT_FWD) {
            if (p.has_pre && p.aux_deriv) {  // save act'(H) beside act(H)
              float g[32];
              act_fwd_deriv32(p.act, v, g);
              if (fringe) {
#pragma unroll
                for (int e = 0; e < 32; ++e) g[e] = 0.f;
              }
              store_chunk(&tmap_d, g, x, y);
            } else {
              if (p.has_pre) store_chunk(&tmap_d, v, x, y);
              if (!(p.dbg & 4)) act_fwd32(p.act, v);
            }
          } else if (EPI_H && p.epi == EPI_ACT_BWD) {
            const int hb_i = hseq % C::NH;
            mbar_wait(&hb[hb_i], (uint32_t)(hseq / C::NH) & 1u);
            if (MODE == SDD && p.act_code) {  // the source is the coded A (R24): act'(H) by table lookup
              uint32_t wa[16];
              load_row_raw(hst + hb_i * EPI_BUF, lane, wa);
              act_code_mul32(p.act, v, wa, tab_smem);
            } else {
              float hf[32];
              load_row(hst + hb_i * EPI_BUF, lane, hf);
              if (p.aux_deriv) {  // the source already holds act'(H)
                mul32(v, hf);
              } else if (!(p.dbg & 4)) {
                act_grad_mul32(p.act, v, hf);
              }
            }
            __syncwarp();
            load_h(hseq + C::NH);  // refill the buffer just read
            ++hseq;
          } else if (MODE == DENSE && p.epi == EPI_ADD_ROWS) {
            // rows to add (router backward: dx += ...): the first term was
            // prefetched at the tile start; further top-k terms load here
            const int trow = t.u * BM + row0 + lane;
            if (trow < p.rows_valid) {
#pragma unroll
              for (int q2 = 0; q2 < 4; ++q2) {
                float af[8];
                unpack8(pre[i][q2], af);
#pragma unroll
                for (int e = 0; e < 8; ++e) v[8 * q2 + e] += af[e];
              }
              const long long col0 = (long long)t.v * BN + c * EPI_COLS;
              for (int j = 1; j < (p.addend_map ? p.addend_k : 1); ++j) {
                const int m = __ldg(p.addend_map + (long long)trow * p.addend_k + j);
                if (m < 0) continue;  // slot dropped by a capacity
                const uint4* src = reinterpret_cast<const uint4*>(p.addend + (long long)m * p.ld_add + col0);
#pragma unroll
                for (int q2 = 0; q2 < 4; ++q2) {
                  float af[8];
                  unpack8(__ldg(src + q2), af);
#pragma unroll
                  for (int e = 0; e < 8; ++e) v[8 * q2 + e] += af[e];
                }
              }
            }
          }
          if (coded_out)
            store_chunk_raw(&tmap_c, wcode, x, y);
          else if (!(MODE == DSD_ROW && p.scatter_only))
            store_chunk(&tmap_c, v, x, y);
          if (MODE == DSD_ROW && p.scatter_y && p.direct) {
            // the weighted un-permutation of the layer (top-1): the
            // gate-scaled rows go straight to y[token] (pad rows: dropped)
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] *= my_gate;
            store_direct(p.out_d, p.ldd, p.rows_d, v, x, 0, my_tok == 0x7fffffff ? -1 : my_tok);
          } else if (MODE == DSD_ROW && p.scatter_y) {
            // the weighted un-permutation of the layer (top-1): the
            // gate-scaled rows go straight to y[token] by tile::scatter4
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] *= my_gate;
            int tk[32];
#pragma unroll
            for (int u = 0; u < 32; ++u) tk[u] = __shfl_sync(0xffffffffu, my_tok, u);
            if (lane == 0) bulk_wait_read<C::NBUF - 1>();
            __syncwarp();
            stage_row(stg + sbuf * EPI_BUF, lane, v);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
#pragma unroll
              for (int g4 = 0; g4 < 8; ++g4)
                tma_scatter4(&tmap_d, stg + sbuf * EPI_BUF + g4 * 4 * 64, x, tk[4 * g4], tk[4 * g4 + 1],
                             tk[4 * g4 + 2], tk[4 * g4 + 3]);
              bulk_commit();
            }
            sbuf = sbuf + 1 == C::NBUF ? 0 : sbuf + 1;
          }
          if (PP && has_acc && i + 1 < NPW) tmem_ld_wait();
        }
      } else if (MODE == DENSE && p.epi == EPI_ROUTER) {
        // logits row of token t -> fp32 logits (TMA store), greedy top-k (ties ->
        // lower e), softmax gates. The two warps of a lane quarter split
        // the experts; each keeps an online (max, sum exp) and a local top-k,
        // group 1 hands its partials to group 0 through shared memory.
        constexpr int CG = BN / NG;  // experts per warp
        const int tok = t.u * BM + row0 + lane;
        const bool valid = tok < p.rows_valid;
        const int topk = p.topk;
        float bv[kMaxRouterTopK];
        int be[kMaxRouterTopK];
#pragma unroll
        for (int j = 0; j < kMaxRouterTopK; ++j) {
          bv[j] = -FLT_MAX;
          be[j] = 0x7fffffff;
        }
        float mx = -FLT_MAX, ssum = 0.f;
        // the tile's expert histogram (topology input): zeroed by the
        // 128 group-0 threads, each owning entries e = its index mod 128
        int32_t* s_hist = reinterpret_cast<int32_t*>(smem_x + 128 * (2 + 2 * kMaxRouterTopK) * 4);
        const int ht = q * 32 + lane;  // 0..127 over the group-0 warps
        if (p.hist_out && grp == 0) {
          for (int e = ht; e < p.E; e += 128) s_hist[e] = 0;
          asm volatile("bar.sync 5, 128;" ::: "memory");
        }
#pragma unroll 1
        for (int c = 0; c < CG / 32; ++c) {
          const int col0 = grp * CG + c * 32;
          uint32_t r[32];
          tmem_ld32(taddr + col0, r);
          tmem_ld_wait();
          // stage the 32 x 32 fp32 chunk (128B-swizzled rows) and TMA-store it
          if (lane == 0) bulk_wait_read<0>();
          __syncwarp();
          {
            const uint32_t row = smem_u32(stg) + lane * 128;
#pragma unroll
            for (int j = 0; j < 8; ++j)
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(row + ((j ^ (lane & 7)) << 4)),
                           "r"(r[4 * j]), "r"(r[4 * j + 1]), "r"(r[4 * j + 2]), "r"(r[4 * j + 3])
                           : "memory");
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmap_c, stg, col0, t.u * BM + row0);
            bulk_commit();
          }
          float cm = -FLT_MAX;
#pragma unroll
          for (int i = 0; i < 32; ++i) cm = fmaxf(cm, __uint_as_float(r[i]));
          float cs = 0.f;
#pragma unroll
          for (int i = 0; i < 32; ++i) cs += __expf(__uint_as_float(r[i]) - cm);
          const float nm = fmaxf(mx, cm);
          ssum = ssum * __expf(mx - nm) + cs * __expf(cm - nm);
          mx = nm;
          if (topk == 1) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float x = __uint_as_float(r[i]);
              if (x > bv[0]) {
                bv[0] = x;
                be[0] = col0 + i;
              }
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float x = __uint_as_float(r[i]);
              const int e = col0 + i;
              // stable insertion into the descending list (experts arrive in ascending e;
              // strict '>' keeps the lower e first on ties). Back to front, reading the
              // not-yet-updated predecessor.
#pragma unroll
              for (int j = kMaxRouterTopK - 1; j >= 0; --j) {
                if (j < topk && x > bv[j]) {
                  if (j > 0 && x > bv[j - 1]) {
                    bv[j] = bv[j - 1];
                    be[j] = be[j - 1];
                  } else {
                    bv[j] = x;
                    be[j] = e;
                  }
                }
              }
            }
          }
        }
        // group 1 -> group 0 through shared memory (per row: max, sum, k values, k experts)
        float* xr = reinterpret_cast<float*>(smem_x) + (row0 + lane) * (2 + 2 * kMaxRouterTopK);
        if (grp == 1) {
          xr[0] = mx;
          xr[1] = ssum;
#pragma unroll
          for (int j = 0; j < kMaxRouterTopK; ++j) {
            xr[2 + j] = bv[j];
            xr[2 + kMaxRouterTopK + j] = __int_as_float(be[j]);
          }
        }
        if (NG > 1) asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
        if (grp == 0) {
          const float m1 = NG > 1 ? xr[0] : -FLT_MAX, s1 = NG > 1 ? xr[1] : 0.f;
          const float M = fmaxf(mx, m1);
          const float S = ssum * __expf(mx - M) + s1 * __expf(m1 - M);
          // merge the two descending lists; on equal values list 0 (lower experts) first
          int i0 = 0, i1 = 0;
          float gsel[kMaxRouterTopK];
          float gsum = 0.f;
#pragma unroll
          for (int j = 0; j < kMaxRouterTopK; ++j) {
            if (j < topk) {
              float v0 = -FLT_MAX, v1 = -FLT_MAX;
              int e0 = 0x7fffffff, e1 = 0x7fffffff;
#pragma unroll
              for (int u = 0; u < kMaxRouterTopK; ++u) {
                if (u == i0) { v0 = bv[u]; e0 = be[u]; }
              }
              if (NG > 1 && i1 < kMaxRouterTopK) {
                v1 = xr[2 + i1];
                e1 = __float_as_int(xr[2 + kMaxRouterTopK + i1]);
              }
              const bool take1 = v1 > v0;
              const float v = take1 ? v1 : v0;
              const int e = take1 ? e1 : e0;
              i1 += take1 ? 1 : 0;
              i0 += take1 ? 0 : 1;
              gsel[j] = __expf(v - M) / S;
              gsum += gsel[j];
              if (valid) {
                p.idx[(long long)tok * topk + j] = e;
                if (p.hist_out) atomicAdd(&s_hist[e], 1);  // integer: order-independent
              }
            }
          }
          const float gscale = p.renorm ? 1.f / gsum : 1.f;  // NEXT-4 renormalisation over the k chosen
#pragma unroll
          for (int j = 0; j < kMaxRouterTopK; ++j)
            if (j < topk && valid) p.gates[(long long)tok * topk + j] = gsel[j] * gscale;
          if (p.hist_out) {
            asm volatile("bar.sync 5, 128;" ::: "memory");
            for (int e = ht; e < p.E; e += 128) p.hist_out[(long long)t.u * p.E + e] = s_hist[e];
          }
        }
        if (NG > 1) asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");  // xr reused by the next tile
      } else if (MODE == DENSE) {  // EPI_F32: fp32 partial tile (split-K)
        const int r = t.u * BM + row0 + lane;
        float* dst = p.out_f32 + (long long)t.s * p.split_stride + (long long)r * p.ld_f32 + t.v * BN;
#pragma unroll 1
        for (int c = grp; c < BN / 32; c += NG) {
          uint32_t rr[32];
          if (has_acc) {  // warp-uniform: every lane takes part in the collective TMEM load
            tmem_ld32(taddr + c * 32, rr);
            tmem_ld_wait();
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) rr[i] = 0u;
          }
          if (r < p.rows_valid) {
#pragma unroll
            for (int i = 0; i < 32; i += 4)
              *reinterpret_cast<float4*>(dst + c * 32 + i) =
                  make_float4(__uint_as_float(rr[i]), __uint_as_float(rr[i + 1]), __uint_as_float(rr[i + 2]),
                              __uint_as_float(rr[i + 3]));
          }
        }
      }
      if (has_acc) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
      if (wq == 0 && lane == 0) trace_ev(p, tile_i, 4);
    }
    if (lane == 0) bulk_wait<0>();
  }

  if (MODE == DENSE && p.topo_fused) {
    // router + top-k + topology in one launch ("custom CUDA kernel"): every
    // CTA's expert ids and tile histograms are in global memory after the grid
    // barrier; the operand ring (idle now) is the topology's scratch
    __syncthreads();
    cooperative_groups::this_grid().sync();
    const int k = p.topk, row_chunk = 128 * k;
    const int rows_per_cta = (int)blockDim.x / row_chunk;
    const int n_rows = p.m_tiles;
    TopoTask tk;
    tk.rank_first = blockIdx.x;
    tk.rank_stride = gridDim.x;
    tk.emit_first = blockIdx.x;
    tk.emit_stride = gridDim.x;
    tk.publish = blockIdx.x == 0;
    topo_scan_emit_body(p.idx, p.rows_valid * k, p.E, p.topo_bs, p.topo_F, (n_rows + rows_per_cta - 1) / rows_per_cta,
                        p.hist_out, p.topo, p.topo_capacity, n_rows, row_chunk, rows_per_cta, tk,
                        reinterpret_cast<int32_t*>(smem));
  }
  tc_fence_before();
  __syncthreads();
  if (MODE == DSD_ROW && p.mcast) cluster_sync();  // the peer's last commits / multicasts into this CTA are done
  if (warp == C::MMA_WARP) {
    tc_fence_after();
    tmem_dealloc<C::TMEM_COLS>(tmem_base);
  }
}

// ------------------------------------------------------------------ host side

static thread_local int t_sm_budget = 0;
void set_gemm_sm_budget(int sms) { t_sm_budget = sms; }
int gemm_sm_budget() {
  const int all = moe_device_sm_count();
  return (t_sm_budget > 0 && t_sm_budget < all) ? t_sm_budget : all;
}

// Experiment knobs for A/B timing (MOE_GEMM_DBG, see GemmParams::dbg); 0 in production.
int gemm_dbg() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MOE_GEMM_DBG");
    v = e ? atoi(e) : 0;
  }
  return v;
}

// Trace buffer: allocated on first use when MOE_GEMM_TRACE is set (debug only);
// successive launches take successive slots; moe_debug_trace_dump writes them out.
static unsigned long long* g_trace = nullptr;
static int g_trace_next = 0;
static const char* g_trace_names[kTraceLaunches];

unsigned long long* gemm_trace_slot() {
  static int on = -1;
  if (on < 0) on = getenv("MOE_GEMM_TRACE") != nullptr;
  if (!on || g_trace_next >= kTraceLaunches) return nullptr;
  const size_t per = (size_t)kTraceCtas * kTraceTiles * kTraceEvents;
  if (!g_trace) {
    if (cudaMalloc(&g_trace, per * kTraceLaunches * sizeof(unsigned long long)) != cudaSuccess) return nullptr;
    cudaMemset(g_trace, 0, per * kTraceLaunches * sizeof(unsigned long long));
  }
  return g_trace + per * g_trace_next++;
}

template <int MODE, bool A_MN, bool B_MN, int BN, bool EPI_H, int OCC = 1>
static moe_status launch_t(const GemmLaunch& L, cudaStream_t stream) {
  using C = Cfg<MODE, BN, EPI_H, OCC>;
  auto kern = bsgemm_kernel<MODE, A_MN, B_MN, BN, EPI_H, OCC>;
  {
    static unsigned long long smem_mask = 0;  // per device (the attribute is per device)
    static int smem_set = 0;
    cudaError_t e = set_smem_attr_once(kern, (int)C::SMEM, smem_mask, smem_set);
    if (e != cudaSuccess) return set_error(MOE_ECUDA, "%s: smem attribute: %s", L.name, cudaGetErrorString(e));
  }
  int grid = OCC * gemm_sm_budget();
  if (L.max_tiles < grid) grid = L.max_tiles;
  if (grid < 1) grid = 1;
  GemmParams p = L.p;
  p.dbg = MODE == DENSE ? 0 : gemm_dbg();  // experiment knobs act on the products only (routing stays valid)
  {
    // MOE_EPI_DIRECT=1: epilogue stores by st.global through a shared-memory
    // transpose instead of TMA (measured slower at MoE-XS: SDD 129 vs 111 us,
    // the others equal; kept for A/B experiments)
    static int direct = -1;
    if (direct < 0) {
      const char* e = getenv("MOE_EPI_DIRECT");
      direct = (e && e[0] == '1') ? 1 : 0;
    }
    p.direct = (direct && p.out_c) ? 1 : 0;
  }
  p.trace = gemm_trace_slot();
  {
    static int rev = -1;
    if (rev < 0) {
      // bit m reverses the tile order of mode m. Default: DSD_ROW (its S operand
      // was just written by the SDD / SDD^T before it; the tail is still in L2)
      // and the column walks DS^TD / DD^TS (-0.7 us each at MoE-XS)
      const char* e = getenv("MOE_GEMM_REVERSE");
      rev = e ? atoi(e) : (1 << DSD_ROW) | (1 << DS_COL) | (1 << DDS_COL);
    }
    if (((rev >> MODE) & 1) && !(MODE != SDD && p.gather_a)) p.reverse = 1;  // gathered DD^TS: forward order
  }
  cudaError_t le;
  if (MODE == DENSE && p.topo_fused) {  // grid barrier inside: cooperative launch (all CTAs co-resident)
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(C::THREADS);
    lc.dynamicSmemBytes = C::SMEM;
    lc.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    le = cudaLaunchKernelEx(&lc, kern, L.ta, L.tb, L.tc, L.td, L.te, L.tf, p);
  } else if (MODE == DSD_ROW && p.mcast) {  // 2-CTA clusters (an even grid: the clusters walk tile pairs)
    grid &= ~1;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(C::THREADS);
    lc.dynamicSmemBytes = C::SMEM;
    lc.stream = stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = pdl_enabled() ? 2 : 1;
    le = cudaLaunchKernelEx(&lc, kern, L.ta, L.tb, L.tc, L.td, L.te, L.tf, p);
  } else {
    le = launch_k(kern, dim3(grid), dim3(C::THREADS), C::SMEM, stream, L.ta, L.tb, L.tc, L.td, L.te, L.tf, p);
  }
  if (le != cudaSuccess) return set_error(MOE_ECUDA, "%s: %s", L.name, cudaGetErrorString(le));
  MOE_CHECK_LAUNCH(L.name);
  return MOE_OK;
}

static int router_occ() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MOE_ROUTER_OCC");  // 2: two CTAs per SM (measured slower: 21.3 vs 18.7 us at
    v = (e && e[0] == '2') ? 2 : 1;             // MoE-XS, 4 epilogue warps with register spills); default 1
  }
  return v;
}

#define MOE_GEMM_CASE(MODE, AMN, BMN, BN, H)                                                     \
  if (L.mode == MODE && L.a_mn == AMN && L.b_mn == BMN && L.bn == BN && L.epi_h == H)          \
    return launch_t<MODE, AMN, BMN, BN, H>(L, stream);

moe_status gemm_launch(const GemmLaunch& L, cudaStream_t stream) {
  // forward / backward products of the layer, 256-wide tiles
  MOE_GEMM_CASE(SDD, false, true, 256, false)     // SDD      X_g . W1
  MOE_GEMM_CASE(SDD, false, false, 256, true)     // SDD^T    dY_g . W2^T (+act')
  MOE_GEMM_CASE(SDD, false, false, 256, false)
  MOE_GEMM_CASE(DSD_ROW, false, true, 256, false)  // DSD      A . W2
  MOE_GEMM_CASE(DSD_ROW, false, false, 256, false) // DSD^T    dH . W1^T
  MOE_GEMM_CASE(DS_COL, true, true, 256, false)    // DS^TD    A^T . dY_g
  MOE_GEMM_CASE(DS_COL, true, false, 256, false)
  MOE_GEMM_CASE(DDS_COL, true, true, 256, false)   // DD^TS    X_g^T . dH
  MOE_GEMM_CASE(DDS_COL, false, true, 256, false)
  // 128-wide tiles (odd block-columns per expert, h % 256 != 0, DDS^T)
  MOE_GEMM_CASE(SDD, false, true, 128, false)
  MOE_GEMM_CASE(SDD, false, false, 128, true)
  MOE_GEMM_CASE(SDD, false, false, 128, false)
  MOE_GEMM_CASE(DSD_ROW, false, true, 128, false)
  MOE_GEMM_CASE(DSD_ROW, false, false, 128, false)
  MOE_GEMM_CASE(DS_COL, true, true, 128, false)
  MOE_GEMM_CASE(DS_COL, true, false, 128, false)
  MOE_GEMM_CASE(DDS_COL, true, true, 128, false)
  MOE_GEMM_CASE(DDS_COL, false, true, 128, false)
  MOE_GEMM_CASE(DDS_ROW, false, false, 128, false)
  MOE_GEMM_CASE(DDS_ROW, true, false, 128, false)
  // router
  // logits = x . Wr (+top-k epilogue); MOE_ROUTER_OCC=2: two CTAs per SM (experiment)
  if (L.mode == DENSE && !L.a_mn && L.b_mn && !L.epi_h && L.p.epi == EPI_ROUTER && router_occ() == 2) {
    if (L.bn == 64) return launch_t<DENSE, false, true, 64, false, 2>(L, stream);
    if (L.bn == 128) return launch_t<DENSE, false, true, 128, false, 2>(L, stream);
  }
  MOE_GEMM_CASE(DENSE, false, true, 64, false)
  MOE_GEMM_CASE(DENSE, false, true, 128, false)
  MOE_GEMM_CASE(DENSE, false, true, 256, false)
  MOE_GEMM_CASE(DENSE, true, true, 64, false)      // dWr partials = x^T . dlogits
  MOE_GEMM_CASE(DENSE, true, true, 128, false)
  MOE_GEMM_CASE(DENSE, true, true, 256, false)
  MOE_GEMM_CASE(DENSE, false, false, 256, false)   // dx += dlogits . Wr^T
  MOE_GEMM_CASE(DENSE, false, false, 128, false)
  return set_error(MOE_EUNSUPPORTED, "%s: no kernel instance for mode=%d a_mn=%d b_mn=%d bn=%d", L.name, L.mode,
                   (int)L.a_mn, (int)L.b_mn, L.bn);
}

GemmParams gemm_params_topo(const moe_config* cfg, const moe_topology_t* topo) {
  GemmParams p{};
  p.sizes = topo->sizes;
  p.row_offsets = topo->row_offsets;
  p.col_indices = topo->col_indices;
  p.row_indices = topo->row_indices;
  p.t_col_offsets = topo->t_col_offsets;
  p.t_block_offsets = topo->t_block_offsets;
  p.t_row_indices = topo->t_row_indices;
  p.pair_bins = topo->pair_bins;
  p.padded_bins = topo->padded_bins;
  p.counts = topo->counts;
  p.F = (int)(cfg->ffn_hidden / cfg->block_size);
  p.E = (int)cfg->num_experts;
  p.unpadded = cfg->unpadded;
  p.brow_start = topo->brow_start;
  p.brow_rows = topo->brow_rows;
  {
    // column walks skip the all-zero second K-step of a half-filled last
    // block-row (MOE_KSKIP=0: off)
    static int ks = -1;
    if (ks < 0) {
      const char* e = getenv("MOE_KSKIP");
      ks = (e && e[0] == '0') ? 0 : 1;
    }
    p.kskip = ks;
  }
  p.sorted_idx = topo->sorted_idx;
  p.n_block_cols = (int)(cfg->num_experts * cfg->ffn_hidden / cfg->block_size);
  p.k_dense = (int)cfg->hidden;
  p.epi = EPI_STORE;
  p.act = MOE_ACT_IDENTITY;
  return p;
}

// 256-wide tiles when every expert has an even number of block-columns and the
// hidden size is a multiple of 256; 128 otherwise.
static int pick_bn(const moe_config* cfg, bool pairs_columns) {
  const int64_t F = cfg->ffn_hidden / cfg->block_size;
  if (pairs_columns) return (F % 2 == 0) ? 256 : 128;
  static int force128 = -1;
  if (force128 < 0) force128 = getenv("MOE_DSD_BN128") != nullptr;  // experiment: 128-wide DSD tiles
  return (cfg->hidden % 256 == 0 && !force128) ? 256 : 128;
}

// Experiment switch MOE_GEMM_PAIR_ROWS: row-pair 2-SM tiles for DSD / DSD^T
// (measured slower at MoE-XS: half-empty pairs of odd-row experts).
static bool use_pair_rows() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MOE_GEMM_PAIR_ROWS");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// MOE_DSD_MCAST=1: the row-walk DSD runs in 2-CTA clusters whose CTAs hold the
// two column tiles of one block-row and share its A loads by TMA multicast.
static bool dsd_mcast() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MOE_DSD_MCAST");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// 2-SM (cta_group::2) 256 x 256 tiles: needs even F and h % 256 == 0.
// MOE_GEMM_PAIR=0 in the environment selects the 1-SM kernels (A/B testing).
// The CTA-pair forward SDD's epilogue stores 4 KB boxes (64 x 32, 128 B
// swizzle; 111 -> 104 us at MoE-XS); MOE_PAIR_WIDE=0: 2 KB boxes.
static bool pair_wide() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MOE_PAIR_WIDE");
    v = e && e[0] == '0' ? 0 : 1;
  }
  return v == 1;
}

static bool use_pair(const moe_config* cfg) {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("MOE_GEMM_PAIR");
    env = (e && e[0] == '0') ? 0 : 1;
  }
  const int64_t F = cfg->ffn_hidden / cfg->block_size;
  return env && F % 2 == 0 && cfg->hidden % 256 == 0;
}

}  // namespace moe

using namespace moe;

extern "C" {

/* Debug only: synchronise, write the recorded GEMM timelines (MOE_GEMM_TRACE)
 * as raw uint64 [launch][cta][tile][event] to `path`, reset. Returns launches. */
int moe_debug_trace_dump(const char* path) {
  if (!g_trace || !path) return 0;
  cudaDeviceSynchronize();
  const size_t per = (size_t)kTraceCtas * kTraceTiles * kTraceEvents;
  const size_t n = per * g_trace_next;
  unsigned long long* h = (unsigned long long*)malloc(n * sizeof(unsigned long long));
  if (!h) return -1;
  cudaMemcpy(h, g_trace, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  FILE* f = fopen(path, "wb");
  if (f) {
    fwrite(h, sizeof(unsigned long long), n, f);
    fclose(f);
  }
  free(h);
  const int launches = g_trace_next;
  g_trace_next = 0;
  cudaMemset(g_trace, 0, per * kTraceLaunches * sizeof(unsigned long long));
  return launches;
}

static moe_status sdd_launch(const moe_config* cfg, const void* a, const void* b, int trans_b,
                             const moe_topology_t* topo, int32_t act, const void* act_src, void* out_s, void* out_aux,
                             bool deriv, void* stream, const void* x_gather = nullptr, bool coded = false) {
  MOE_TRY(moe_check_config(cfg));
  MOE_TRY(check_topo(topo));
  MOE_CHECK_ARG(a && b && out_s, "moe_sdd: NULL operand");
  MOE_CHECK_ARG(act >= 0 && act <= 2, "moe_sdd: bad act %d", act);
  const int64_t nnz = moe_max_nnz_blocks(cfg);
  const int64_t rows = moe_max_padded_rows(cfg);
  const int64_t h = cfg->hidden, N = cfg->num_experts * cfg->ffn_hidden;
  GemmLaunch L{};
  L.name = trans_b ? "moe_sdd(T)" : "moe_sdd";
  L.mode = SDD;
  L.bn = pick_bn(cfg, true);
  L.a_mn = false;
  L.b_mn = !trans_b;
  L.p = gemm_params_topo(cfg, topo);
  L.p.act = act;
  L.p.epi = act_src ? EPI_ACT_BWD : ((act != MOE_ACT_IDENTITY || out_aux) ? EPI_ACT_FWD : EPI_STORE);
  L.p.has_pre = out_aux != nullptr;
  L.p.aux_deriv = deriv ? 1 : 0;
  L.p.act_code = coded && act != MOE_ACT_IDENTITY ? 1 : 0;
  if (L.p.act_code) {
    L.p.aux_deriv = 0;
    MOE_CHECK_ARG(!out_aux, "moe_sdd_act_coded: the coded form has no second output");
  }
  {
    // L2 priorities of the SDD outputs: act(H) (read next by the DSD) kept,
    // act'(H) (read only in the backward) streamed; SDD^T: dH kept.
    static int mode = -1;
    if (mode < 0) {
      const char* e = getenv("MOE_L2_HINTS");
      mode = e ? atoi(e) : 0;  // measured neutral at MoE-XS: opt-in
    }
    if (mode) {
      if (act_src) {
        L.p.l2_c = 1;
      } else {
        L.p.l2_c = 1;
        L.p.l2_d = 2;
      }
    }
  }
  L.epi_h = L.p.epi == EPI_ACT_BWD;
  // Row-pair 2-SM (cta_group::2) tiles: each SM streams half of the expert's
  // weight columns, so the operand traffic per output drops to 2/3 (MoE-XS:
  // SDD 109 -> 101 us, SDD^T 99.3 -> 97.6 with the in-place 4 KB act'(H)
  // ring) — when the experts average >= 3 block-rows: with fewer, the
  // half-empty pairs of odd-row experts cost more than the pairs save
  // (MoE-Medium T=8192: SDD 139.5 us 1-SM vs 143.4 pairs; top-2: SDD 189 vs
  // 199, SDD^T 191 vs 201). MOE_SDD_PAIR=0: 1-SM for both, =1: pairs for both.
  const char* pe = getenv("MOE_SDD_PAIR");  // read per call: the tests cover both forms in one process
  const int pair_env = pe && pe[0] ? (pe[0] == '1' ? 1 : 0) : -1;
  // (the A-row gather inside the loads, moe_sdd_gather, exists only in the 1-SM kernel)
  const bool deep = cfg->tokens * cfg->top_k >= 3LL * cfg->num_experts * BM;
  bool pair = use_pair(cfg) && !x_gather && (pair_env == 1 || (pair_env == -1 && deep));
  // the coded activation is wired into the CTA-pair kernel's 4 KB-box epilogues only
  if (pair && L.p.act_code && !(act_src ? gemm2_h_coded() : pair_wide())) pair = false;
  L.max_tiles = pair ? (int)((rows / BM / 2 + cfg->num_experts) * (L.p.F / 2)) : (int)(nnz / (L.bn / 128));
  if (x_gather) {  // A rows = x[row_src / k] by tile::gather4 (X_g never materialised)
    MOE_TRY(make_tmap_bf16(&L.ta, x_gather, h, cfg->tokens, h, BK, 1, "moe_sdd_gather x", KSW));
    L.p.gather_a = 1;
    L.p.gather_k = (int)cfg->top_k;
    L.p.gather_T = (int)cfg->tokens;
    L.p.row_src = topo->row_src;
  } else {
    MOE_TRY(make_tmap_bf16(&L.ta, a, h, rows, h, BK, 128, "moe_sdd a", KSW));
  }
  if (!trans_b)
    MOE_TRY(make_tmap_bf16_mn(&L.tb, b, N, h, N, pair ? 2 : L.bn / 64, "moe_sdd b"));
  else
    MOE_TRY(make_tmap_bf16(&L.tb, b, h, N, h, BK, pair ? 128 : L.bn, "moe_sdd b^T", KSW));
  const bool wide = pair && (act_src ? gemm2_wide_h() : pair_wide());
  L.p.wide = wide ? 1 : 0;
  {
    // an expert's lone last block-row as an M = 128 CTA-pair tile instead of a
    // half-empty 256-row pair (the 4 KB-box epilogues; MOE_SDD_HALF=0: off)
    static int half_env = -1;
    if (half_env < 0) {
      const char* e = getenv("MOE_SDD_HALF");
      half_env = (e && e[0] == '0') ? 0 : 1;
    }
    L.p.sdd_half = pair && half_env && (act_src ? gemm2_h_ring() : wide) ? 1 : 0;
    static int alt_env = -1;
    if (alt_env < 0) {
      const char* e = getenv("MOE_PAIR_EPI_ALT");
      alt_env = (e && e[0] == '1') ? 1 : 0;
    }
    L.p.epi_alt = pair && wide && !act_src && alt_env ? 1 : 0;
    static int tall_env = -1;
    if (tall_env < 0) {
      const char* e = getenv("MOE_PAIR_TALL");
      tall_env = (e && e[0] == '1') ? 1 : 0;
    }
    L.p.tall = pair && wide && !act_src && !L.p.act_code && !L.p.epi_alt && tall_env ? 1 : 0;
    static int hd_env = -1;
    if (hd_env < 0) {
      const char* e = getenv("MOE_SDDT_HDIRECT");
      hd_env = (e && e[0] == '1') ? 1 : 0;
    }
    L.p.h_direct = pair && act_src && !L.p.act_code && hd_env ? 1 : 0;
    L.p.h_src = reinterpret_cast<const __nv_bfloat16*>(act_src);
  }
  auto epi_map = L.p.tall ? make_tmap_epi_tall : wide ? make_tmap_epi_wide : make_tmap_epi;
  MOE_TRY(epi_map(&L.tc, out_s, 128, nnz * 128, 128, "moe_sdd out"));
  set_epi_out(L.p, 0, out_s, nnz * 128, 128);
  if (out_aux) MOE_TRY(epi_map(&L.td, out_aux, 128, nnz * 128, 128, "moe_sdd aux"));
  if (out_aux) set_epi_out(L.p, 1, out_aux, nnz * 128, 128);
  if (act_src) MOE_TRY(epi_map(&L.td, act_src, 128, nnz * 128, 128, "moe_sdd act src"));
  if (!out_aux && !act_src) L.td = L.tc;
  return pair ? gemm2_launch(L, as_stream(stream)) : gemm_launch(L, as_stream(stream));
}

moe_status moe_sdd(const moe_config* cfg, const void* a, const void* b, int trans_b, const moe_topology_t* topo,
                   int32_t act, const void* act_grad_src, void* out_s, void* out_pre, void* stream) {
  return sdd_launch(cfg, a, b, trans_b, topo, act, act_grad_src, out_s, out_pre, false, stream);
}

// The fused-gather products need the CTA-pair column kernels (even F, h % 256 == 0) and 64-wide K-steps.
static bool gather_fusable(const moe_config* cfg) {
  return use_pair(cfg) && BK == 64 && cfg->block_size == 128 && !cfg->unpadded;
}

// Whether the layer (moe_forward / moe_backward) gathers inside the products.
// Off by default: the 32 tile::gather4 requests per stage (one 128 B row each
// per 4-row op) are issue-rate bound — measured SDD 160 vs 100 + 14 us and
// DD^TS 269 vs 74 us at MoE-XS; MOE_GATHER_FUSED=1 enables it.
int moe_gather_is_fused(const moe_config* cfg) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("MOE_GATHER_FUSED");
    on = (e && e[0] == '1') ? 1 : 0;
  }
  return on && cfg && gather_fusable(cfg) ? 1 : 0;
}

moe_status moe_sdd_gather(const moe_config* cfg, const void* x, const void* w1, const moe_topology_t* topo,
                          int32_t act, void* out_s, void* out_deriv, void* x_g, void* stream) {
  MOE_CHECK_ARG(x && w1 && out_s, "moe_sdd_gather: NULL pointer");
  if (cfg && gather_fusable(cfg))
    return sdd_launch(cfg, x, w1, 0, topo, act, nullptr, out_s, out_deriv, true, stream, x);
  MOE_CHECK_ARG(x_g, "moe_sdd_gather: this config needs the x_g scratch (padded gather + SDD)");
  MOE_TRY(moe_gather(cfg, x, topo, x_g, stream));
  return sdd_launch(cfg, x_g, w1, 0, topo, act, nullptr, out_s, out_deriv, true, stream);
}

moe_status moe_sdd_act_coded(const moe_config* cfg, const void* a, const void* b, int trans_b,
                             const moe_topology_t* topo, int32_t act, const void* coded_src, void* out_s,
                             void* stream) {
  return sdd_launch(cfg, a, b, trans_b, topo, act, coded_src, out_s, nullptr, false, stream, nullptr, true);
}

moe_status moe_sdd_deriv(const moe_config* cfg, const void* a, const void* b, int trans_b,
                         const moe_topology_t* topo, int32_t act, const void* deriv_src, void* out_s,
                         void* out_deriv, void* stream) {
  MOE_CHECK_ARG(!(deriv_src && out_deriv), "moe_sdd_deriv: deriv_src and out_deriv are exclusive");
  return sdd_launch(cfg, a, b, trans_b, topo, act, deriv_src, out_s, out_deriv, true, stream);
}

// DSD launcher. With y: the output rows are also (or, with dl16, only) scattered
// to y[row_src[p]] by tile::scatter4, scaled by gates (NULL: 1). With dl16 and wr:
// each tile appends E/BK dense K-steps dl16[token rows] . wr^T (the router term
// of dx, P:98 chain rule) and writes only y.
static moe_status dsd_launch(const moe_config* cfg, const void* s, int trans_s, const void* b, int trans_b,
                             const moe_topology_t* topo, void* out, const float* gates, void* y, void* stream,
                             const void* dl16 = nullptr, const void* wr = nullptr,
                             const unsigned long long* row_dst = nullptr) {
  MOE_TRY(moe_check_config(cfg));
  MOE_TRY(check_topo(topo));
  MOE_CHECK_ARG(s && b && (out || row_dst), "moe_dsd: NULL operand");
  const int64_t rows = moe_max_padded_rows(cfg), nnz = moe_max_nnz_blocks(cfg);
  const int64_t h = cfg->hidden, N = cfg->num_experts * cfg->ffn_hidden;
  // (the row-pair DSD exists only for the padded layout; the row-address stores only in the 1-SM kernel)
  const bool pair = use_pair(cfg) && (trans_s || (use_pair_rows() && !cfg->unpadded && !row_dst));
  // dense rows the products read along K: with the unpadded layout the rows
  // past the last expert's fringe are out of range (TMA zero fill), so their
  // stale contents never meet the fringe's zero sparse rows
  const int64_t drows = cfg->unpadded ? cfg->tokens * cfg->top_k : rows;
  GemmLaunch L{};
  L.p = gemm_params_topo(cfg, topo);
  L.bn = pick_bn(cfg, false);
  L.p.dense_tiles = (int)(h / L.bn);
  L.b_mn = !trans_b;
  const int bbox = pair ? 128 : L.bn;
  if (!trans_s) {
    L.name = trans_b ? "moe_dsd(T)" : "moe_dsd";
    L.mode = DSD_ROW;
    L.a_mn = false;
    L.max_tiles = pair ? (int)((rows / BM / 2 + cfg->num_experts) * L.p.dense_tiles)
                       : (int)(rows / BM * L.p.dense_tiles);
    // 2-CTA clusters sharing A across the block-row's column tiles (pairs of them)
    L.p.mcast = (!pair && dsd_mcast() && L.p.dense_tiles % 2 == 0) ? 1 : 0;
    MOE_TRY(make_tmap_bf16(&L.ta, s, 128, nnz * 128, 128, BK, L.p.mcast ? 64 : 128, "moe_dsd s", KSW));
    if (!trans_b)
      MOE_TRY(make_tmap_bf16_mn(&L.tb, b, h, N, h, pair ? 2 : L.bn / 64, "moe_dsd b"));
    else
      MOE_TRY(make_tmap_bf16(&L.tb, b, N, h, N, BK, bbox, "moe_dsd b^T", KSW));
    if (row_dst) {  // rows stored by address (the map is never used for a store)
      L.p.row_dst = row_dst;
      MOE_TRY(make_tmap_epi(&L.tc, s, 128, nnz * 128, 128, "moe_dsd_rows (unused map)"));
    } else {
      MOE_TRY(make_tmap_epi(&L.tc, out, h, rows, h, "moe_dsd out"));
      set_epi_out(L.p, 0, out, rows, h);
    }
    if (y) {  // fused weighted un-permutation (top-1): rows scattered to y[token] by tile::scatter4
      MOE_TRY(make_tmap_bf16(&L.td, y, h, cfg->tokens, h, 32, 1, "moe_dsd_scatter y", 64));
      set_epi_out(L.p, 1, y, cfg->tokens, h);
      L.p.scatter_y = 1;
      L.p.scatter_T = (int)cfg->tokens;
      L.p.row_src = topo->row_src;
      L.p.scatter_gates = gates;
    }
    if (dl16 && wr) {  // + dlogits . Wr^T on the gathered token rows, only the scatter is written
      const int64_t E = cfg->num_experts;
      MOE_TRY(make_tmap_bf16(&L.te, dl16, E, cfg->tokens, E, 64, 1, "moe_dsd_dx dlogits", 128));
      MOE_TRY(make_tmap_bf16(&L.tf, wr, E, h, E, BK, L.bn, "moe_dsd_dx wr", KSW));
      L.p.extra_k = (int)(E / BK);
      L.p.scatter_only = 1;
    }
  } else {
    L.name = trans_b ? "moe_dsd(S^T,T)" : "moe_dsd(S^T)";
    L.mode = DS_COL;
    L.a_mn = true;
    L.max_tiles = (pair ? L.p.n_block_cols / 2 : L.p.n_block_cols) * L.p.dense_tiles;
    MOE_TRY(make_tmap_bf16_mn(&L.ta, s, 128, nnz * 128, 128, 2, "moe_dsd s^T"));
    if (!trans_b)
      MOE_TRY(make_tmap_bf16_mn(&L.tb, b, h, drows, h, pair ? 2 : L.bn / 64, "moe_dsd b"));
    else
      MOE_TRY(make_tmap_bf16(&L.tb, b, drows, h, rows, BK, bbox, "moe_dsd b^T", KSW));
    MOE_TRY(make_tmap_epi(&L.tc, out, h, N, h, "moe_dsd out"));
    set_epi_out(L.p, 0, out, N, h);
  }
  if (!L.p.scatter_y) L.td = L.tc;
  return pair ? gemm2_launch(L, as_stream(stream)) : gemm_launch(L, as_stream(stream));
}

moe_status moe_dsd(const moe_config* cfg, const void* s, int trans_s, const void* b, int trans_b,
                   const moe_topology_t* topo, void* out, void* stream) {
  return dsd_launch(cfg, s, trans_s, b, trans_b, topo, out, nullptr, nullptr, stream);
}

moe_status moe_dsd_rows(const moe_config* cfg, const void* s, const void* b, int trans_b,
                        const moe_topology_t* topo, const uint64_t* row_dst, void* stream) {
  MOE_CHECK_ARG(row_dst, "moe_dsd_rows: NULL row_dst");
  MOE_CHECK_ARG(cfg && !cfg->unpadded, "moe_dsd_rows: the padded layout only");
  return dsd_launch(cfg, s, 0, b, trans_b, topo, nullptr, nullptr, nullptr, stream, nullptr, nullptr,
                    reinterpret_cast<const unsigned long long*>(row_dst));
}

moe_status moe_dsd_dx(const moe_config* cfg, const void* dh, const void* w1, const moe_topology_t* topo,
                      const void* dlogits_bf16, const void* wr, void* dx, void* dx_g, void* stream) {
  MOE_CHECK_ARG(dh && w1 && dx, "moe_dsd_dx: NULL pointer");
  MOE_CHECK_ARG((dlogits_bf16 == nullptr) == (wr == nullptr), "moe_dsd_dx: dlogits and wr come together");
  const bool router_term = dlogits_bf16 != nullptr;
  if (cfg && cfg->top_k == 1 && cfg->capacity == 0 && cfg->block_size == 128 && cfg->hidden % 256 == 0 &&
      !use_pair_rows() && (!router_term || (cfg->num_experts % 64 == 0 && cfg->num_experts <= 256))) {
    if (router_term) return dsd_launch(cfg, dh, 0, w1, 1, topo, dx, nullptr, dx, stream, dlogits_bf16, wr);
    MOE_CHECK_ARG(dx_g, "moe_dsd_dx: the un-permutation-only form needs the dx_g buffer");
    return dsd_launch(cfg, dh, 0, w1, 1, topo, dx_g, nullptr, dx, stream);  // dX_g kept, rows also to dx
  }
  // general k: dX_g = dH . W1^T, then dx = sum_j dX_g[pos] (+ dlogits . Wr^T)
  MOE_CHECK_ARG(dx_g, "moe_dsd_dx: top_k > 1 needs the dx_g scratch buffer");
  MOE_TRY(moe_dsd(cfg, dh, 0, w1, 1, topo, dx_g, stream));
  if (cfg->unpadded)  // unpadded rows: the expert-order re-sort (+ the router term, tcgen05)
    return router_term ? moe_sort_rows_bwd_router(cfg, dx_g, topo, dlogits_bf16, wr, dx, stream)
                       : moe_sort_rows_bwd(cfg, dx_g, topo, dx, stream);
  if (!router_term) return moe_gather_bwd(cfg, dx_g, topo, dx, stream);
  static int gathered = -1;  // MOE_ROUTER_DX_GATHERED=1: the router-dx GEMM gathers the k rows itself
  if (gathered < 0) {
    const char* e = getenv("MOE_ROUTER_DX_GATHERED");
    gathered = e && e[0] == '1';
  }
  if (gathered) return moe_router_dx(cfg, dlogits_bf16, wr, dx_g, topo, dx, stream);
  // the k-row sum by the coalesced combine kernel, then dx += dlogits . Wr^T with
  // contiguous addend rows (in place)
  MOE_TRY(moe_gather_bwd(cfg, dx_g, topo, dx, stream));
  MOE_CHECK_ARG(router_on_tensor_cores(cfg), "moe_dsd_dx: the router term needs E %% 64 == 0, E <= 256, top_k <= 8");
  return router_dx_tc(cfg, reinterpret_cast<const __nv_bfloat16*>(dlogits_bf16), wr, dx, dx, nullptr, 1,
                      cfg->hidden, as_stream(stream));
}

moe_status moe_dsd_scatter(const moe_config* cfg, const void* s, const void* b, const moe_topology_t* topo,
                           const float* gates, void* y_g, void* y, void* stream) {
  MOE_CHECK_ARG(y, "moe_dsd_scatter: NULL y");  // gates may be NULL: unit weights (un-permutation only)
  // the fused form writes y only for tokens that own a padded row: dropless top-1 only
  if (cfg && cfg->top_k == 1 && cfg->capacity == 0 && cfg->block_size == 128 && !use_pair_rows())
    return dsd_launch(cfg, s, 0, b, 0, topo, y_g, gates, y, stream);
  MOE_TRY(moe_dsd(cfg, s, 0, b, 0, topo, y_g, stream));  // k > 1: slots are summed by the combine kernel
  if (cfg && cfg->unpadded) return moe_unsort_rows(cfg, y_g, topo, gates, y, stream);  // unpadded rows
  return moe_scatter(cfg, y_g, topo, gates, y, stream);
}

static moe_status dds_launch(const moe_config* cfg, const void* a, int trans_a, const void* s, int trans_s,
                             const moe_topology_t* topo, void* out, void* stream, const void* x_gather);

moe_status moe_dds(const moe_config* cfg, const void* a, int trans_a, const void* s, int trans_s,
                   const moe_topology_t* topo, void* out, void* stream) {
  return dds_launch(cfg, a, trans_a, s, trans_s, topo, out, stream, nullptr);
}

moe_status moe_dds_gather(const moe_config* cfg, const void* x, const void* dh, const moe_topology_t* topo, void* dw1,
                          void* x_g, void* stream) {
  MOE_CHECK_ARG(x && dh && dw1, "moe_dds_gather: NULL pointer");
  if (cfg && gather_fusable(cfg)) return dds_launch(cfg, x, 1, dh, 0, topo, dw1, stream, x);
  MOE_CHECK_ARG(x_g, "moe_dds_gather: this config needs the x_g scratch (padded gather + DD^TS)");
  MOE_TRY(moe_gather(cfg, x, topo, x_g, stream));
  return moe_dds(cfg, x_g, 1, dh, 0, topo, dw1, stream);
}

static moe_status dds_launch(const moe_config* cfg, const void* a, int trans_a, const void* s, int trans_s,
                             const moe_topology_t* topo, void* out, void* stream, const void* x_gather) {
  MOE_TRY(moe_check_config(cfg));
  MOE_TRY(check_topo(topo));
  MOE_CHECK_ARG(a && s && out, "moe_dds: NULL operand");
  const int64_t rows = moe_max_padded_rows(cfg), nnz = moe_max_nnz_blocks(cfg);
  const int64_t h = cfg->hidden, N = cfg->num_experts * cfg->ffn_hidden;
  const int64_t drows = cfg->unpadded ? cfg->tokens * cfg->top_k : rows;  // see dsd_launch
  GemmLaunch L{};
  L.p = gemm_params_topo(cfg, topo);
  L.a_mn = trans_a != 0;
  if (!trans_s) {
    // out [h, E*f] = A_eff [h, rows] . S ; walk column pairs via the transpose index
    const bool pair = use_pair(cfg);
    L.name = trans_a ? "moe_dds(T)" : "moe_dds";
    L.mode = DDS_COL;
    L.bn = pick_bn(cfg, true);
    L.b_mn = true;
    L.p.dense_tiles = (int)(h / (pair ? 2 * BM : BM));
    L.max_tiles = L.p.n_block_cols / (L.bn / 128) * L.p.dense_tiles;
    MOE_TRY(make_tmap_bf16_mn(&L.tb, s, 128, nnz * 128, 128, 2, "moe_dds s"));
    if (x_gather) {  // A = X_g^T with the K-rows gathered from x (pair kernel only, see gather_fusable)
      MOE_TRY(make_tmap_bf16(&L.ta, x_gather, h, cfg->tokens, h, 64, 1, "moe_dds_gather x", 128));
      L.p.gather_a = 1;
      L.p.gather_k = (int)cfg->top_k;
      L.p.gather_T = (int)cfg->tokens;
      L.p.row_src = topo->row_src;
      L.p.kskip = 0;  // the gathered token ring walks whole blocks
    } else if (trans_a)
      MOE_TRY(make_tmap_bf16_mn(&L.ta, a, h, drows, h, 2, "moe_dds a^T"));
    else
      MOE_TRY(make_tmap_bf16(&L.ta, a, drows, h, rows, BK, 128, "moe_dds a", KSW));
    MOE_TRY(make_tmap_epi(&L.tc, out, N, h, N, "moe_dds out"));
    set_epi_out(L.p, 0, out, h, N);
    L.td = L.tc;
    return pair ? gemm2_launch(L, as_stream(stream)) : gemm_launch(L, as_stream(stream));
  }
  // out [h, rows] = A_eff [h, E*f] . S^T ; walk rows
  if (cfg->unpadded)
    return set_error(MOE_EUNSUPPORTED, "moe_dds(trans_s=1): the padded layout only (its output columns are dense rows)");
  L.p.dense_tiles = (int)(h / BM);
  L.name = trans_a ? "moe_dds(T,S^T)" : "moe_dds(S^T)";
  L.mode = DDS_ROW;
  L.bn = 128;
  L.b_mn = false;
  L.max_tiles = (int)(rows / BM * L.p.dense_tiles);
  MOE_TRY(make_tmap_bf16(&L.tb, s, 128, nnz * 128, 128, BK, 128, "moe_dds s^T", KSW));
  if (trans_a)
    MOE_TRY(make_tmap_bf16_mn(&L.ta, a, h, N, h, 2, "moe_dds a^T"));
  else
    MOE_TRY(make_tmap_bf16(&L.ta, a, N, h, N, BK, 128, "moe_dds a", KSW));
  MOE_TRY(make_tmap_epi(&L.tc, out, rows, h, rows, "moe_dds out"));
  set_epi_out(L.p, 0, out, h, rows);
  L.td = L.tc;
  return gemm_launch(L, as_stream(stream));
}

}  // extern "C"
