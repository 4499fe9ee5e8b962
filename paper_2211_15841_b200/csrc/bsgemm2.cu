// bsgemm2.cu — the six block-sparse products on CTA pairs (tcgen05.mma
// cta_group::2): one 256 x 256 output tile per 2-SM cluster, each SM holding
// half of A (128 rows) and half of B (128 columns) in shared memory, so per-SM
// operand traffic per MMA flop is two thirds of the 1-SM 128 x 256 tile's
// (bsgemm.cu). Same products, same topology walks (§5.1; P:238,
// P:242):
//
//   SDD     rows (r0, r1) of one expert x block-columns (c, c+1)        K = dense dim
//   DSD_ROW rows (r0, r1) of one expert x 256 dense columns              K walks row r0's blocks
//   DS_COL  block-columns (c, c+1) of one expert x 256 dense columns     K walks column c (transpose index)
//   DDS_COL 256 dense rows x block-columns (c, c+1)                      K walks column c (transpose index)
//
// Rows r0, r1 = r0+1 of the same expert share their block-column set, and
// columns c, c+1 of the same expert share their block-row set, so one walk
// serves both halves. Row pairs come from the topology's pair_bins (an expert
// with an odd number of block-rows leaves one half-empty pair: the second CTA
// computes on padding and stores nothing).
//
// Roles as in bsgemm.cu; the leader CTA (rank 0) issues all MMAs; both CTAs'
// TMA loads signal the leader's full barrier; the MMA commit multicasts to
// both CTAs' empty / tmem-full barriers; both CTAs' epilogues release the
// leader's tmem-empty barrier.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "bsgemm.cuh"
#include "common.cuh"
#include "gemm_util.cuh"
#include "sm100.cuh"
#include "tma.cuh"

#ifndef MOE_MAX_STAGES
#define MOE_MAX_STAGES 16
#endif

namespace moe {

#ifndef MOE_PAIR_NP
#define MOE_PAIR_NP 2
#endif
constexpr int P_NP = MOE_PAIR_NP;              // TMA producer warps per CTA (stage s issued by warp s % P_NP):
                                               // one issuing thread keeps too few boxes in flight
constexpr int P_MMA_WARP = P_NP;
constexpr int P_EPI_WARP0 = P_NP + 1;
constexpr int P_THREADS = 32 * (P_NP + 1 + NUM_EPI_WARPS);
constexpr int P_BN = 256;                      // N of the pair MMA
constexpr int P_BH = 128;                      // B columns held per CTA
constexpr int P_A_BYTES = A_BYTES;             // 128 x 64
constexpr int P_B_BYTES = P_BH * BK * 2;       // 128 x 64
constexpr int P_STAGE = P_A_BYTES + P_B_BYTES;

#ifndef MOE_PAIR_NBUF
#define MOE_PAIR_NBUF 2
#endif
constexpr int P_NBUF = MOE_PAIR_NBUF;                          // staging buffers per epilogue warp
#ifndef MOE_PAIR_WIDE
#define MOE_PAIR_WIDE 1
#endif
// SDD^T: columns per box of the per-warp act'(H) / coded-A ring (64: 4 KB boxes,
// 128B swizzle; 32: 2 KB boxes, 64B swizzle) and its depth. 4 KB boxes three
// deep (the default) leave no room for the coded-activation decode table (R24:
// that SDD^T then runs on the 1-SM kernel); 2 KB boxes five deep fit it beside
// four pipeline stages but measured slower (MoE-XS SDD^T 133 vs 97 us with
// act'(H); 163 us decoding the coded A).
#ifndef MOE_PAIR_HC
#define MOE_PAIR_HC 64
#endif
#ifndef MOE_PAIR_NHW
#define MOE_PAIR_NHW (MOE_PAIR_HC == 64 ? 3 : 5)
#endif

constexpr int P_PB_MAX = 384;  // experts whose pair offsets fit the shared-memory copy (row_pair)

template <bool EPI_H, int MODE = -1>
struct Cfg2 {
  // the forward SDD stores 64-column chunks (4 KB TMA boxes, two staging
  // buffers of 4 KB per warp: one per output); the others 32-column chunks
  // (DS^TD / DD^TS measured no faster with 4 KB boxes: 73.8 / 76.6 us vs
  // 71.4 / 75.5, the larger staging costing two pipeline stages)
  static constexpr bool WIDE = MOE_PAIR_WIDE && MODE == SDD && !EPI_H;
  // SDD^T: a per-warp ring of NHW act'(H) / coded-A boxes (HC x 32), each
  // turned into the dH box in place and stored from the same buffer
  static constexpr bool WIDE_H = MOE_PAIR_WIDE && EPI_H;
  static constexpr int HC = MOE_PAIR_HC;
  static constexpr int HBOX = 32 * HC * 2;
  static constexpr int NHW = MOE_PAIR_NHW;
  static constexpr int NHB = WIDE_H ? NHW : 2;  // act'(H) barriers per epilogue warp
  static constexpr int P_EPI_BYTES = WIDE_H ? 0 : NUM_EPI_WARPS * (WIDE ? 2 * 4096 : P_NBUF * EPI_BUF);
  static constexpr int H_BYTES = EPI_H ? (WIDE_H ? NUM_EPI_WARPS * NHW * HBOX : EPI_BYTES) : 0;
  static constexpr int TOK = MODE == DDS_COL ? 4 * 16 * 16 : 0;  // DDS_COL gather: token ring, 4 K-steps x 16 lanes x int4
  // SDD^T: act'(H) decode table of the coded A (R24), where it fits
  static constexpr bool HAS_TAB = EPI_H && WIDE_H && HC == 32;
  static constexpr int TAB = HAS_TAB ? ACT_CODE_BYTES : 0;
  static constexpr int PB = (MODE == SDD || MODE == DSD_ROW) ? P_PB_MAX * 4 : 0;  // pair offsets (row_pair)
  static constexpr int STAGES_RAW = (SMEM_LIMIT - SMEM_FIXED - P_EPI_BYTES - H_BYTES - TOK - TAB - PB) / P_STAGE;
  static constexpr int STAGES = STAGES_RAW > MOE_MAX_STAGES ? MOE_MAX_STAGES : STAGES_RAW;
  static constexpr int TMEM_COLS = 2 * P_BN;
  static constexpr size_t SMEM = SMEM_FIXED + (size_t)STAGES * P_STAGE + P_EPI_BYTES + H_BYTES + TOK + TAB + PB;
  static_assert(!EPI_H || STAGES >= 4, "SDD^T: four pipeline stages expected");
};

struct Tile2 {
  int kiters;
  int walk_begin;  // row walk: storage index of row r0's first block; column walk: transpose position
  int r0;          // SDD/DSD_ROW: first block-row of the pair
  bool second;     // SDD/DSD_ROW: r0 + 1 belongs to the same expert
  int c0;          // SDD: first block column; DS_COL/DDS_COL: first column of the pair
  int v;           // dense tile (DSD_ROW / DS_COL: 256-wide N tile; DDS_COL: 256-row M tile)
  int q_off;       // DSD_ROW: storage offset of this CTA's row relative to row r0 (= rank * F)
};

__device__ __forceinline__ int num_tiles2(const GemmParams& p, int mode) {
  const int pairs = p.sizes[2];
  switch (mode) {
    case SDD: return pairs * (p.F / 2);
    case DSD_ROW: return pairs * p.dense_tiles;
    default: return (p.n_block_cols / 2) * p.dense_tiles;  // DS_COL, DDS_COL
  }
}

// Row pair p -> (first block-row, whether the second row exists; returns the
// expert), via the per-expert pair offsets `pbins` (binary search over E; a
// shared-memory copy when E is small: the search is on every tile's decode
// path, and six dependent L2 round trips there stalled the TMA producer at
// each tile boundary).
__device__ __forceinline__ int row_pair(const GemmParams& p, const int32_t* pbins, int pr, int& r0, bool& second) {
  int lo = 0, hi = p.E - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (pbins[mid] > pr) hi = mid; else lo = mid + 1;
  }
  const int e = lo;
  const int pb = __ldg(p.padded_bins + e);
  const int pc = pb - (e > 0 ? __ldg(p.padded_bins + e - 1) : 0);
  const int nrows = pc / BM;
  const int i = pr - (pbins[e] - (nrows + 1) / 2);
  r0 = (pb - pc) / BM + 2 * i;
  second = 2 * i + 1 < nrows;
  return e;
}

__device__ __forceinline__ Tile2 decode2(const GemmParams& p, int mode, int tile, int rank, const int32_t* pbins) {
  Tile2 t{};
  if (mode == SDD) {
    const int pr = tile / (p.F / 2), cp = tile % (p.F / 2);
    const int e = row_pair(p, pbins, pr, t.r0, t.second);
    t.c0 = e * p.F + 2 * cp;
    t.kiters = p.k_dense / BK;
  } else if (mode == DSD_ROW) {
    const int pr = tile / p.dense_tiles;
    t.v = tile % p.dense_tiles;
    row_pair(p, pbins, pr, t.r0, t.second);
    const int b = __ldg(p.row_offsets + t.r0), e = __ldg(p.row_offsets + t.r0 + 1);
    t.walk_begin = b;
    t.kiters = KPB * (e - b);
    t.q_off = rank * (e - b);
  } else {  // DS_COL, DDS_COL
    t.c0 = (tile / p.dense_tiles) * 2;
    t.v = tile % p.dense_tiles;
    const int b = __ldg(p.t_col_offsets + t.c0), e = __ldg(p.t_col_offsets + t.c0 + 1);
    t.walk_begin = b;
    t.kiters = KPB * (e - b);
    // the columns' last block-row (the expert's fringe) holds <= 64 assignments:
    // its second K-step multiplies zero rows only (pad rows / zero sparse rows)
    // (the expert's count decides it: (count - 1) % 128 < 64; one load, off the index chain)
    if (KPB == 2 && p.kskip && e > b) {
      const int cnt = __ldg(p.counts + t.c0 / p.F);
      if (cnt > 0 && (cnt - 1) % BM < BM / 2) --t.kiters;
    }
    t.second = true;
  }
  return t;
}

// TMA store coordinates of 32-column chunk c (0..7) for this CTA's rows.
__device__ __forceinline__ void out_coords2(const GemmParams& p, int mode, const Tile2& t, int rank, int c, int row0,
                                            int F, int& x, int& y) {
  const int col = c * EPI_COLS;
  switch (mode) {
    case SDD: {  // blocks (r0+rank, c0), (r0+rank, c0+1) in [nnz*128, 128] storage
      const int r = t.r0 + rank;
      const int blk = r * F + (t.c0 % F) + col / 128;
      x = col % 128;
      y = blk * BM + row0;
      break;
    }
    case DSD_ROW: x = t.v * P_BN + col; y = (t.r0 + rank) * BM + row0; break;
    case DS_COL: x = t.v * P_BN + col; y = (t.c0 + rank) * BM + row0; break;
    default: x = t.c0 * 128 + col; y = (2 * t.v + rank) * BM + row0; break;  // DDS_COL
  }
}

// SDD half pair (p.sdd_half, an expert's lone last block-row r0): one M = 128
// cta_group::2 MMA, each CTA holding 64 of its rows; TMEM lanes 0-63 hold the
// CTA's rows x tile columns 0-127, lanes 64-127 the same rows x columns
// 128-255. TMA store coordinates of 32-column TMEM chunk c (0..3) of lane
// quarter q.
__device__ __forceinline__ void out_coords2_half(const GemmParams& p, const Tile2& t, int rank, int c, int q, int F,
                                                 int& x, int& y) {
  const int blk = t.r0 * F + (t.c0 % F) + (q >> 1);
  x = c * EPI_COLS;
  y = blk * BM + rank * 64 + (q & 1) * 32;
}

template <int MODE, bool A_MN, bool B_MN, bool EPI_H>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(P_THREADS, 1)
    bsgemm2_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                   const __grid_constant__ CUtensorMap tmap_c, const __grid_constant__ CUtensorMap tmap_d,
                   const GemmParams p) {
  using C = Cfg2<EPI_H, MODE>;
  constexpr int STAGES = C::STAGES;
  constexpr int P_EPI_BYTES = C::P_EPI_BYTES;
  constexpr int NCHUNK = P_BN / EPI_COLS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem_a + STAGES * P_A_BYTES;
  uint8_t* smem_epi = smem_b + STAGES * P_B_BYTES;
  uint8_t* smem_h = smem_epi + P_EPI_BYTES;
  int4* tokring = reinterpret_cast<int4*>(smem_h + C::H_BYTES);
  uint8_t* smem_tab = smem_h + C::H_BYTES + C::TOK;
  int32_t* smem_pb = reinterpret_cast<int32_t*>(smem_tab + C::TAB);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_tab + C::TAB + C::PB);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* hbar = tempty + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(hbar + C::NHB * NUM_EPI_WARPS);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int rank = (int)cluster_ctarank();
  const bool leader = rank == 0;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  if (threadIdx.x == 0) trace_ev(p, 0, 13);  // kernel entry (trace slot tile 0, event 13)

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      // epi_alt: each accumulator is drained by one group of NUM_EPI_WARPS / 2 warps per CTA
      mbar_init(&tempty[i], (C::WIDE && p.epi_alt) ? NUM_EPI_WARPS : 2 * NUM_EPI_WARPS);
    }
    for (int i = 0; i < C::NHB * NUM_EPI_WARPS; ++i) mbar_init(&hbar[i], 1);
    fence_barrier_init();
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
  }
  if (warp == P_MMA_WARP) tmem_alloc_pair<C::TMEM_COLS>(tmem_holder);
  if (C::HAS_TAB && p.act_code) act_code_table_to_smem(smem_tab, g_act_code_tab);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  pdl_trigger();
  pdl_wait();
  const int ntiles = num_tiles2(p, MODE);
  // p.reverse: tiles walked last-to-first (the operand rows the previous
  // kernel wrote last are the ones still in L2)
  auto rtile = [&](int tile) { return p.reverse ? ntiles - 1 - tile : tile; };
  // the pair offsets in shared memory for the row-pair decode (E <= P_PB_MAX)
  const int32_t* s_pb = p.pair_bins;
  if (C::PB && p.E <= P_PB_MAX) {
    for (int i = threadIdx.x; i < p.E; i += blockDim.x) smem_pb[i] = __ldg(p.pair_bins + i);
    __syncthreads();
    s_pb = smem_pb;
  }

  if (warp < P_NP) {
    // ===================== TMA producers (both CTAs; warp s % P_NP issues stage s) =====================
    int stage = 0;
    uint32_t phase = 0;
    int tile_i = 0;
    // DDS_COL with gathered A (p.gather_a): the K-rows of a column tile are the
    // contiguous padded rows of its expert; their token ids (row_src / k) are
    // copied by cp.async into a 4-slot ring TD = 3 K-steps ahead of use.
    constexpr int TD = 3;
    const bool gat = MODE == DDS_COL && p.gather_a;
    int la_j = 0, la_kit = 0, la_kiters = 0, la_pstart = 0;  // look-ahead cursor over (tile, K-step)
    long long la_g = 0;                                     // global K-step index of the cursor
    auto la_decode = [&]() {  // settle the cursor on a tile with K-steps (or past the end)
      while (true) {
        const int tl = cid + la_j * ncl;
        if (tl >= ntiles) {
          la_kiters = -1;
          return;
        }
        const int c0 = (tl / p.dense_tiles) * 2;
        const int e = c0 / p.F;
        const int pend = __ldg(p.padded_bins + e);
        la_pstart = e > 0 ? __ldg(p.padded_bins + e - 1) : 0;
        la_kiters = (pend - la_pstart) / (BM / KPB);
        if (la_kiters > 0) return;
        ++la_j;
      }
    };
    auto la_issue = [&]() {  // copy the cursor's 64 row ids (16 lanes x 4), then advance
      if (la_kiters > 0 && lane < 16) {
        const int32_t* src = p.row_src + la_pstart + la_kit * (BM / KPB) + 4 * lane;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(tokring + (la_g & 3) * 16 + lane)),
                     "l"(src)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      if (la_kiters > 0) {
        ++la_g;
        if (++la_kit == la_kiters) {
          la_kit = 0;
          ++la_j;
          la_decode();
        }
      }
    };
    long long g_step = 0;
    // the gathered form keeps its token ring in one warp: warp 0 issues every stage, the others idle
    const bool idle = gat && warp != 0;
    if (gat && !idle) {
      la_decode();
      for (int i = 0; i < TD; ++i) la_issue();
    }
#ifndef MOE_PAIR_SDD_LANE0
#define MOE_PAIR_SDD_LANE0 1
#endif
    // SDD (no index walk): one thread per producer warp runs the whole loop, so the
    // other 31 lanes leave the sub-partition's issue slots to the epilogue warps
    // sharing it
    if (MODE == SDD && MOE_PAIR_SDD_LANE0 && !gat) {
      if (lane == 0) {
        for (int tile = cid; tile < ntiles; tile += ncl, ++tile_i) {
          const Tile2 t = decode2(p, MODE, rtile(tile), rank, s_pb);
          trace_ev(p, tile_i, 0);
          const bool hm = p.sdd_half && !t.second;
          const int sdd_row = hm ? (p.unpadded ? __ldg(p.brow_start + t.r0) : t.r0 * BM) + rank * 64
                                 : (p.unpadded ? __ldg(p.brow_start + t.r0 + ((rank && t.second) ? 1 : 0))
                                               : (t.r0 + rank) * BM);
          for (int kit = 0; kit < t.kiters; ++kit) {
            if (stage % P_NP == warp) {
              mbar_wait_sleep(&empty[stage], phase ^ 1);
              uint8_t* sa = smem_a + stage * P_A_BYTES;
              uint8_t* sb = smem_b + stage * P_B_BYTES;
              uint64_t* fb = &full[stage];
              if (p.dbg & 8) {
                if (leader) mbar_arrive(fb);
              } else {
                if (leader) mbar_arrive_expect_tx(fb, 2 * P_STAGE);
                const int k0 = kit * BK;
                tma_load_2d_pair(sa, &tmap_a, fb, k0, sdd_row);
                if (B_MN)
                  tma_load_3d_pair(sb, &tmap_b, fb, 0, k0, (t.c0 + rank) * 2);
                else
                  tma_load_2d_pair(sb, &tmap_b, fb, k0, (t.c0 + rank) * 128);
              }
            }
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    } else
    for (int tile = cid; tile < ntiles && !idle; tile += ncl, ++tile_i) {
      const Tile2 t = decode2(p, MODE, rtile(tile), rank, s_pb);
      if (lane == 0) trace_ev(p, tile_i, 0);
      int idx_a = 0, idx_b = 0, idx_c = 0;
      // SDD: first dense row of this CTA's block-row (unpadded layout: brow_start; a
      // missing second row of a half-empty pair loads the first row's, stores nothing)
      // half pair (p.sdd_half): both CTAs load the lone block-row, CTA 1 from its 64th row
      const bool hm = MODE == SDD && p.sdd_half && !t.second;
      const int sdd_row = MODE != SDD ? 0
                          : hm        ? (p.unpadded ? __ldg(p.brow_start + t.r0) : t.r0 * BM) + rank * 64
                          : (p.unpadded ? __ldg(p.brow_start + t.r0 + ((rank && t.second) ? 1 : 0)) : (t.r0 + rank) * BM);
      for (int kit = 0; kit < t.kiters; ++kit) {
        const int blk = kit / KPB, kk = kit % KPB;
        if (MODE != SDD && (blk & 31) == 0 && kk == 0) {
          const int qq = t.walk_begin + blk + lane;
          if (qq < t.walk_begin + (t.kiters + KPB - 1) / KPB) {  // (a skipped last half K-step still needs its block)
            if (MODE == DSD_ROW) {
              idx_a = qq + t.q_off;               // this CTA's row: same column, next row
              idx_b = __ldg(p.col_indices + qq);  // block column
            } else {
              idx_a = __ldg(p.t_block_offsets + qq) + rank;  // this CTA's column of the pair
              idx_b = __ldg(p.t_row_indices + qq);
              idx_c = p.unpadded ? __ldg(p.brow_start + idx_b) : idx_b * BM;  // its dense rows
            }
          }
        }
        const int sblk = __shfl_sync(0xffffffffu, idx_a, blk & 31);
        const int oblk = __shfl_sync(0xffffffffu, idx_b, blk & 31);
        const int odrow = __shfl_sync(0xffffffffu, idx_c, blk & 31);
        int4 atok = make_int4(0, 0, 0, 0);
        if (gat) {
          la_issue();  // K-step g_step + TD
          asm volatile("cp.async.wait_group %0;" ::"n"(TD) : "memory");
          __syncwarp();
          const int4 r = tokring[(g_step & 3) * 16 + (lane & 15)];
          const int oob = p.gather_T, kq = p.gather_k;
          atok = make_int4(r.x >= 0 ? r.x / kq : oob, r.y >= 0 ? r.y / kq : oob, r.z >= 0 ? r.z / kq : oob,
                           r.w >= 0 ? r.w / kq : oob);
          ++g_step;
        }
        const bool mine = gat || stage % P_NP == warp;
        if (mine) mbar_wait_sleep(&empty[stage], phase ^ 1);
        if (gat) {
          // A = X_g^T: 64 gathered K-rows x this CTA's 128 h-columns (two 64-wide
          // MN chunks); lane l: chunk l / 16, rows 4 (l % 16) .. +3
          uint8_t* sa = smem_a + stage * P_A_BYTES;
          uint64_t* fb = &full[stage];
          if (leader && lane == 0) mbar_arrive_expect_tx(fb, 2 * P_STAGE);
          __syncwarp();
          const int m0 = (2 * t.v + rank) * BM;
          tma_gather4_pair(sa + (lane >> 4) * (BK * 128) + (lane & 15) * 512, &tmap_a, fb, m0 + (lane >> 4) * 64,
                           atok.x, atok.y, atok.z, atok.w);
          if (lane == 0) tma_load_3d_pair(smem_b + stage * P_B_BYTES, &tmap_b, fb, 0, sblk * BM + kk * BK, 0);
        } else if (mine && lane == 0) {
          uint8_t* sa = smem_a + stage * P_A_BYTES;
          uint8_t* sb = smem_b + stage * P_B_BYTES;
          uint64_t* fb = &full[stage];
          if (p.dbg & 8) {  // experiment: no operand loads (the stage completes at once)
            if (leader) mbar_arrive(fb);
          } else {
          if (leader) mbar_arrive_expect_tx(fb, 2 * P_STAGE);
          if (MODE == SDD) {
            const int k0 = kit * BK;
            tma_load_2d_pair(sa, &tmap_a, fb, k0, sdd_row);
            if (B_MN) {  // W1 [h, E*f]: this CTA's block column c0 + rank (3-D MN box, 2 chunks)
              tma_load_3d_pair(sb, &tmap_b, fb, 0, k0, (t.c0 + rank) * 2);
            } else {     // W2 [E*f, h]
              tma_load_2d_pair(sb, &tmap_b, fb, k0, (t.c0 + rank) * 128);
            }
          } else if (MODE == DSD_ROW) {
            tma_load_2d_pair(sa, &tmap_a, fb, kk * BK, sblk * BM);
            const int n0 = t.v * P_BN + rank * P_BH;
            if (B_MN) {
              tma_load_3d_pair(sb, &tmap_b, fb, 0, oblk * BM + kk * BK, n0 / 64);
            } else {
              tma_load_2d_pair(sb, &tmap_b, fb, oblk * BM + kk * BK, n0);
            }
          } else if (MODE == DS_COL) {
            tma_load_3d_pair(sa, &tmap_a, fb, 0, sblk * BM + kk * BK, 0);
            const int n0 = t.v * P_BN + rank * P_BH;
            if (B_MN) {
              tma_load_3d_pair(sb, &tmap_b, fb, 0, odrow + kk * BK, n0 / 64);
            } else {
              tma_load_2d_pair(sb, &tmap_b, fb, odrow + kk * BK, n0);
            }
          } else {  // DDS_COL: A = dense rows (2v + rank) tile, B = block sblk (this CTA's column)
            const int m0 = (2 * t.v + rank) * BM;
            if (A_MN) {
              tma_load_3d_pair(sa, &tmap_a, fb, 0, odrow + kk * BK, m0 / 64);
            } else {
              tma_load_2d_pair(sa, &tmap_a, fb, odrow + kk * BK, m0);
            }
            tma_load_3d_pair(sb, &tmap_b, fb, 0, sblk * BM + kk * BK, 0);
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
  } else if (warp == P_MMA_WARP) {
    // ===================== MMA issuer (leader CTA, one thread) =====================
    if (leader && lane == 0) {
      constexpr uint32_t idesc_full = make_idesc_bf16(2 * BM, P_BN, A_MN, B_MN);
      constexpr uint32_t idesc_half = make_idesc_bf16(BM, P_BN, A_MN, B_MN);  // SDD half pair: M = 128
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int tile_i = -1;
      for (int tile = cid; tile < ntiles; tile += ncl) {
        const Tile2 t = decode2(p, MODE, rtile(tile), 0, s_pb);
        ++tile_i;
        if (t.kiters == 0) continue;
        const uint32_t idesc = (MODE == SDD && p.sdd_half && !t.second) ? idesc_half : idesc_full;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        trace_ev(p, tile_i, 1);
        const uint32_t d_tmem = tmem_base + acc * P_BN;
        for (int kit = 0; kit < t.kiters; ++kit) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(smem_a + stage * P_A_BYTES);
          const uint32_t b_base = smem_u32(smem_b + stage * P_B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t adesc =
                A_MN ? make_sdesc(a_base + k * 2048, BK * 128, 1024) : make_sdesc(a_base + k * 32, 16, KSW * 8, KSW);
            const uint64_t bdesc =
                B_MN ? make_sdesc(b_base + k * 2048, BK * 128, 1024) : make_sdesc(b_base + k * 32, 16, KSW * 8, KSW);
            if (!(p.dbg & 2)) mma_bf16_pair(d_tmem, adesc, bdesc, idesc, (kit | k) != 0);
          }
          mma_commit_pair(&empty[stage], 0x3);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit_pair(&tfull[acc], 0x3);
        trace_ev(p, tile_i, 2);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // ===================== epilogue (warps 2..9, both CTAs) =====================
    const int q = warp & 3;
    const int wq = warp - P_EPI_WARP0;
    const int half = wq >> 2;                  // this warp's first chunk; it takes every EPG-th
    constexpr int EPG = NUM_EPI_WARPS / 4;     // epilogue warps per TMEM lane quarter
    const int row0 = q * 32;
    uint8_t* stg = smem_epi + wq * (C::WIDE ? 2 * 4096 : P_NBUF * EPI_BUF);
    uint8_t* hst = smem_h + wq * (C::WIDE_H ? C::NHW * C::HBOX : 2 * EPI_BUF);
    uint64_t* hb = hbar + wq * C::NHB;
    uint32_t hphase[2] = {0, 0};
    int hslot = 0;
    int sbuf = 0;
    int acc = 0;
    uint32_t acc_phase = 0;

    auto store_chunk = [&](const CUtensorMap* map, const float* v, int x, int y) {
      if (lane == 0) bulk_wait_read<P_NBUF - 1>();
      __syncwarp();
      stage_row(stg + sbuf * EPI_BUF, lane, v);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(map, stg + sbuf * EPI_BUF, x, y);
        bulk_commit();
      }
      sbuf = sbuf + 1 == P_NBUF ? 0 : sbuf + 1;
    };
    auto load_h = [&](const Tile2& t, int c, int b) {
      if (lane == 0) {
        fence_proxy_async_smem();
        int x, y;
        out_coords2(p, MODE, t, rank, c, row0, p.F, x, y);
        mbar_arrive_expect_tx(&hb[b], EPI_BUF);
        tma_load_2d(hst + b * EPI_BUF, &tmap_d, &hb[b], x, y);
      }
    };

    // SDD^T ring: this warp's HC-column boxes form one sequence j over its
    // tiles (tile cid + (j / SPW) * ncl, box half + (j % SPW) * EPG); the
    // act'(H) / coded-A box of j + NHW - 1 is loaded while j is processed
    constexpr int HSUB = C::HC / 32;  // 32-column TMEM loads per box
    constexpr int SPW = (P_BN / C::HC) / EPG;
    const int hw_end = (ntiles > cid ? (ntiles - 1 - cid) / ncl + 1 : 0) * SPW;
    int hw_seq = 0;
    uint32_t hw_phase = 0;  // bit b: parity of slot b's next completion
    // coordinates of ring item j (false: nothing is stored for it on this CTA)
    auto coords_hw = [&](int j, int& x, int& y) {
      const Tile2 tj = decode2(p, MODE, rtile(cid + (j / SPW) * ncl), rank, s_pb);
      const bool hmj = MODE == SDD && p.sdd_half && !tj.second;
      const int scj = half + (j % SPW) * EPG;
      if (hmj ? HSUB * scj >= 4 : !(rank == 0 || tj.second)) return false;
      if (hmj)
        out_coords2_half(p, tj, rank, HSUB * scj, q, p.F, x, y);
      else
        out_coords2(p, MODE, tj, rank, HSUB * scj, row0, p.F, x, y);
      return true;
    };
#ifndef MOE_PAIR_HPF
#define MOE_PAIR_HPF 0  // ring items ahead that the act'(H) boxes are prefetched into L2 (measured: 4 -> SDD^T 114 vs 94.5 us; 0: none)
#endif
    auto load_hw = [&](int j) {  // lane 0
      if (MOE_PAIR_HPF > 0 && j + MOE_PAIR_HPF < hw_end) {  // the box MOE_PAIR_HPF items on: into L2 now
        int px, py;
        if (coords_hw(j + MOE_PAIR_HPF, px, py)) tma_prefetch_2d(&tmap_d, px, py);
      }
      if (j >= hw_end) return;
      int x, y;
      if (!coords_hw(j, x, y)) return;  // nothing stored here: nothing loaded
      const int b = j % C::NHW;
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&hb[b], C::HBOX);
      tma_load_2d(hst + b * C::HBOX, &tmap_d, &hb[b], x, y);
    };
    // h_direct: each lane reads its row's 64 act'(H) values of ring item j
    // straight from global memory into registers (8 x 16 B, L1-allocating),
    // one item ahead, so the act'(H) stream bypasses the SM's TMA unit (which
    // the operand loads and the dH stores keep busy)
    const bool hdir = C::WIDE_H && C::HC == 64 && p.h_direct;
    uint4 hnx[8];
    auto ldg_hw = [&](int j) {
      int x, y;
      if (j < hw_end && coords_hw(j, x, y)) {
        const uint4* src = reinterpret_cast<const uint4*>(p.h_src + ((long long)(y + lane) * 128 + x));
#pragma unroll
        for (int u = 0; u < 8; ++u) hnx[u] = __ldg(src + u);
      }
    };
    if (hdir) ldg_hw(0);
    if (C::WIDE_H && !hdir && lane == 0) {
      for (int j = 0; j < MOE_PAIR_HPF; ++j) {  // the first items' boxes into L2
        int px, py;
        if (j + C::NHW - 1 < hw_end && coords_hw(j + C::NHW - 1, px, py)) tma_prefetch_2d(&tmap_d, px, py);
      }
      for (int j = 0; j < C::NHW - 1; ++j) load_hw(j);
    }

    int tile_i = -1;
    // epi_alt (forward SDD, 4 KB boxes): warp group `half` drains accumulator
    // `half`, i.e. every other tile, all of its columns; the two groups work on
    // consecutive tiles at different phases instead of splitting each tile
    const bool ealt = C::WIDE && p.epi_alt && p.wide;
    uint32_t aphase = 0;
    for (int tile = cid; tile < ntiles; tile += ncl) {
      const Tile2 t = decode2(p, MODE, rtile(tile), rank, s_pb);
      ++tile_i;
      if (ealt && (tile_i & 1) != half) continue;  // the other group's tile
      const int acc_t = ealt ? half : acc;
      const uint32_t ph_t = ealt ? aphase : acc_phase;
      const bool has_acc = t.kiters > 0;
      // SDD half pair (an expert's lone last block-row, p.sdd_half): both CTAs own 64 of its rows
      const bool hm = MODE == SDD && p.sdd_half && !t.second;
      const bool mine = rank == 0 || t.second || hm;  // does this CTA own real output rows?
      // unpadded layout: this lane's row of the CTA's SDD block-row is the fringe: zeros
      const bool fringe =
          MODE == SDD && p.unpadded && mine &&
          (hm ? rank * 64 + (q & 1) * 32 + lane >= __ldg(p.brow_rows + t.r0)
              : row0 + lane >= __ldg(p.brow_rows + t.r0 + rank));
      if (EPI_H && !C::WIDE_H && p.epi == EPI_ACT_BWD && mine) load_h(t, half, hslot);
      if (has_acc) {
        mbar_wait_sleep(&tfull[acc_t], ph_t);
        tc_fence_after();
      }
      if (wq == 0 && lane == 0) trace_ev(p, tile_i, 3);
      const uint32_t taddr = tmem_base + ((uint32_t)row0 << 16) + acc_t * P_BN;
      if (p.dbg & 1) {
        if (has_acc) {
          uint32_t r[32];
          tmem_ld32(taddr, r);
          tmem_ld_wait();
          if (r[0] == 0x7fffffffu && r[1] == 0x12345u) p.gates[0] = 1.f;
        }
      } else if (C::WIDE_H && hdir) {
        // dH = dA (x) act'(H) per 64-column box, act'(H) from registers (h_direct);
        // the dH box is staged in the item's slot of the (now store-only) ring
#pragma unroll 1
        for (int s = 0; s < SPW; ++s, ++hw_seq) {
          const int sc = half + s * EPG;
          uint4 hcur[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) hcur[u] = hnx[u];
          ldg_hw(hw_seq + 1);  // the next item's rows, in flight while this one is processed
          if (mine && !(hm && 2 * sc >= 4)) {
            uint8_t* slot = hst + (hw_seq % C::NHW) * C::HBOX;
            if (lane == 0) bulk_wait_read<C::NHW - 1>();  // the store NHW items ago has read this slot
            __syncwarp();
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              float v[32];
              if (has_acc) {
                uint32_t r[32];
                tmem_ld32(taddr + (2 * sc + hh) * EPI_COLS, r);
                tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = fringe ? 0.f : __uint_as_float(r[i]);
              } else {
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = 0.f;
              }
              float hf[32];
#pragma unroll
              for (int u = 0; u < 4; ++u) unpack8(hcur[4 * hh + u], hf + 8 * u);
              if (p.aux_deriv) {
                mul32(v, hf);
              } else {
                act_grad_mul32(p.act, v, hf);
              }
              stage_row_half128(slot, lane, v, hh);
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              int x, y;
              if (hm)
                out_coords2_half(p, t, rank, 2 * sc, q, p.F, x, y);
              else
                out_coords2(p, MODE, t, rank, 2 * sc, row0, p.F, x, y);
              if (!(p.dbg & 16)) tma_store_2d(&tmap_c, slot, x, y);
              bulk_commit();
            }
          }
        }
      } else if (C::WIDE_H) {
        // dH = dA (x) act'(H) per HC-column box: HSUB 32-column TMEM loads,
        // the act'(H) / coded-A box read and overwritten in place, one store
#pragma unroll 1
        for (int s = 0; s < SPW; ++s, ++hw_seq) {
          const int b = hw_seq % C::NHW;
          const int sc = half + s * EPG;
          if (mine && !(hm && HSUB * sc >= 4)) {  // a half pair holds TMEM columns 0-127 only
            mbar_wait(&hb[b], (hw_phase >> b) & 1u);
            hw_phase ^= 1u << b;
            uint8_t* slot = hst + b * C::HBOX;
#pragma unroll
            for (int hh = 0; hh < HSUB; ++hh) {
              float v[32];
              if (has_acc) {
                uint32_t r[32];
                tmem_ld32(taddr + (HSUB * sc + hh) * EPI_COLS, r);
                tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = fringe ? 0.f : __uint_as_float(r[i]);
              } else {
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = 0.f;
              }
              if (C::HAS_TAB && p.act_code) {  // the slot holds the coded A (R24): act'(H) by table lookup
                uint32_t wa[16];
                if (HSUB == 2) load_row_half128_raw(slot, lane, wa, hh); else load_row_raw(slot, lane, wa);
                if (!(p.dbg & 4)) act_code_mul32(p.act, v, wa, smem_u32(smem_tab));
              } else {
                float hf[32];
                if (HSUB == 2) load_row_half128(slot, lane, hf, hh); else load_row(slot, lane, hf);
                if (p.aux_deriv) {
                  mul32(v, hf);
                } else {
                  act_grad_mul32(p.act, v, hf);
                }
              }
              // this lane's row only: in place is safe
              if (HSUB == 2) stage_row_half128(slot, lane, v, hh); else stage_row(slot, lane, v);
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              int x, y;
              if (hm)
                out_coords2_half(p, t, rank, HSUB * sc, q, p.F, x, y);
              else
                out_coords2(p, MODE, t, rank, HSUB * sc, row0, p.F, x, y);
              if (!(p.dbg & 16)) tma_store_2d(&tmap_c, slot, x, y);
              bulk_commit();
            }
          }
          if (lane == 0) {
            bulk_wait_read<1>();  // the store of step hw_seq - 1 has read its slot: refill it
            load_hw(hw_seq + C::NHW - 1);
          }
          __syncwarp();
        }
      } else if (C::WIDE && p.wide && mine) {
        // 64-column super-chunks C = half, half + EPG (2 per warp per tile),
        // each two 32-column TMEM loads staged into 128B-swizzled rows, then
        // one 4 KB TMA store per output (act(H) to tmap_c; the forward SDD's
        // H or act'(H) to tmap_d)
        uint8_t* bufc = stg;
        uint8_t* bufd = stg + 4096;
        // p.tall: the warps of lane quarters 2j and 2j+1 (same column group)
        // stage one 64 x 64 (8 KB) box per output together — the even
        // quarter's staging holds act(H), the odd one's act'(H), each warp's 32
        // rows at (q & 1) * 4 KB — and the even-quarter warp issues the stores
        const bool tall = p.tall != 0;
        const bool issuer = !tall || !(q & 1);
        const int pbar = 7 + half * 2 + (q >> 1);
        if (tall) {
          const int pair_wq = 4 * half + (((q ^ 1) + 1) & 3);  // warp wq + 3 holds lane quarter (wq + 3) & 3
          bufc = smem_epi + ((q & 1) ? pair_wq : wq) * (2 * 4096) + (q & 1) * 4096;
          bufd = smem_epi + ((q & 1) ? wq : pair_wq) * (2 * 4096) + (q & 1) * 4096;
        }
        const bool two = p.epi == EPI_ACT_FWD && p.has_pre;
        // one output (the coded A, R24): the two buffers alternate, so a
        // super-chunk waits only for the store issued two super-chunks ago
        const bool alt = p.epi == EPI_ACT_FWD && p.act_code;
#pragma unroll 1
        for (int sc = ealt ? 0 : half; sc < (hm ? 2 : P_BN / 64); sc += ealt ? 1 : EPG) {  // a half pair: TMEM columns 0-127
          // both 32-column TMEM loads of the super-chunk in flight while this
          // warp waits for its staging buffers
          uint32_t r[2][32];
          if (has_acc) {
            tmem_ld32(taddr + (2 * sc) * EPI_COLS, r[0]);
            tmem_ld32(taddr + (2 * sc + 1) * EPI_COLS, r[1]);
          }
          uint8_t* bc = bufc;
          if (alt) {
            if (lane == 0) bulk_wait_read<1>();
            bc = stg + sbuf * 4096;
            sbuf ^= 1;
          } else if (lane == 0 && issuer) {
            bulk_wait_read<0>();  // the previous super-chunk's stores have read both buffers
          }
          if (tall)
            named_bar_sync(pbar, 64);
          else
            __syncwarp();
          if (has_acc) tmem_ld_wait();
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            float* v = reinterpret_cast<float*>(r[hh]);
            if (!has_acc || (p.unpadded && fringe)) {  // no accumulator / the fringe rows: zeros
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = 0.f;
            }
            if (p.epi == EPI_ACT_FWD && p.act_code) {  // coded A only (R24)
              uint32_t wcode[16];
              act_fwd_code32((p.dbg & 4) ? MOE_ACT_IDENTITY : p.act, v, wcode);
              stage_row_half128_raw(bc, lane, wcode, hh);
              continue;
            }
            if (p.epi == EPI_ACT_FWD) {
              if (p.has_pre && p.aux_deriv) {
                float g[32];
                act_fwd_deriv32((p.dbg & 4) ? MOE_ACT_IDENTITY : p.act, v, g);
                if (p.unpadded && fringe) {
#pragma unroll
                  for (int i = 0; i < 32; ++i) g[i] = 0.f;
                }
                stage_row_half128(bufd, lane, g, hh);
              } else {
                if (p.has_pre) stage_row_half128(bufd, lane, v, hh);
                act_fwd32(p.act, v);
              }
            }
            stage_row_half128(bc, lane, v, hh);
          }
          fence_proxy_async_smem();
          if (tall)
            named_bar_sync(pbar, 64);
          else
            __syncwarp();
          if (lane == 0 && issuer) {
            int x, y;
            if (hm)
              out_coords2_half(p, t, rank, 2 * sc, q, p.F, x, y);
            else
              out_coords2(p, MODE, t, rank, 2 * sc, row0, p.F, x, y);
            if (!(p.dbg & 16)) tma_store_2d(&tmap_c, bc, x, y);
            if (two && !(p.dbg & 16)) tma_store_2d(&tmap_d, bufd, x, y);
            bulk_commit();
          }
        }
      } else if (mine) {
        // chunks c = half, half + EPG, ...; MOE_PAIR_PINGPONG=1 at build time:
        // fully unrolled with ping-pong TMEM registers (the next chunk's
        // tcgen05.ld in flight while this one is stored) — measured slower for
        // the forward SDD (114 vs 107 us, 168 vs 138 registers)
#ifndef MOE_PAIR_PINGPONG
#define MOE_PAIR_PINGPONG 0
#endif
        constexpr bool PP = MOE_PAIR_PINGPONG != 0;
        uint32_t rr[2][32];
        if (PP && has_acc) {
          tmem_ld32(taddr + half * EPI_COLS, rr[0]);
          tmem_ld_wait();
        }
#pragma unroll
        for (int ci = 0; ci < NCHUNK / EPG; ++ci) {
          const int c = half + ci * EPG;
          float v[32];
          if (has_acc && PP) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(rr[ci & 1][i]);
            if (ci + 1 < NCHUNK / EPG) tmem_ld32(taddr + (c + EPG) * EPI_COLS, rr[(ci + 1) & 1]);  // in flight
          } else if (has_acc) {
            tmem_ld32(taddr + c * EPI_COLS, rr[0]);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(rr[0][i]);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.f;
          }
          if (fringe) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.f;
          }
          int x, y;
          out_coords2(p, MODE, t, rank, c, row0, p.F, x, y);
          if (p.epi == EPI_ACT_FWD) {
            if (p.has_pre && p.aux_deriv) {
              float g[32];
              act_fwd_deriv32(p.act, v, g);
              if (fringe) {
#pragma unroll
                for (int i = 0; i < 32; ++i) g[i] = 0.f;
              }
              store_chunk(&tmap_d, g, x, y);
            } else {
              if (p.has_pre) store_chunk(&tmap_d, v, x, y);
              act_fwd32(p.act, v);
            }
          } else if (EPI_H && p.epi == EPI_ACT_BWD) {
            mbar_wait(&hb[hslot], hphase[hslot]);
            hphase[hslot] ^= 1;
            float hf[32];
            load_row(hst + hslot * EPI_BUF, lane, hf);
            if (p.aux_deriv) {
              mul32(v, hf);
            } else {
              act_grad_mul32(p.act, v, hf);
            }
            __syncwarp();
            hslot ^= 1;
            if (c + EPG < NCHUNK) load_h(t, c + EPG, hslot);
          }
          store_chunk(&tmap_c, v, x, y);
          if (PP && has_acc && ci + 1 < NCHUNK / EPG) tmem_ld_wait();
        }
      }
      if (has_acc) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(&tempty[acc_t]);
        if (ealt) {
          aphase ^= 1;
        } else {
          acc ^= 1;
          if (acc == 0) acc_phase ^= 1;
        }
      }
      if (wq == 0 && lane == 0) trace_ev(p, tile_i, 4);
      if (lane == 0 && wq < 8) trace_ev(p, tile_i, 5 + wq);  // each epilogue warp's finish
    }
    if (lane == 0) bulk_wait<0>();
  }

  tc_fence_before();
  cluster_sync();
  if (warp == P_MMA_WARP) {
    tc_fence_after();
    tmem_dealloc_pair<C::TMEM_COLS>(tmem_base);
  }
  if (threadIdx.x == 0) trace_ev(p, 1, 13);  // kernel exit (trace slot tile 1, event 13)
}

template <int MODE, bool A_MN, bool B_MN, bool EPI_H>
static moe_status launch2_t(const GemmLaunch& L, cudaStream_t stream) {
  using C = Cfg2<EPI_H, MODE>;
  if (C::WIDE_H && (C::HC == 64) != (L.p.wide != 0))
    return set_error(MOE_EUNSUPPORTED, "%s: the CTA-pair SDD^T ring needs %d-column act'(H) / dH maps", L.name, C::HC);
  if (EPI_H && L.p.act_code && !C::HAS_TAB)
    return set_error(MOE_EUNSUPPORTED, "%s: no room for the coded-activation table in this CTA-pair build", L.name);
  auto kern = bsgemm2_kernel<MODE, A_MN, B_MN, EPI_H>;
  {
    static unsigned long long smem_mask = 0;  // per device (the attribute is per device)
    static int smem_set = 0;
    cudaError_t e = set_smem_attr_once(kern, (int)C::SMEM, smem_mask, smem_set);
    if (e != cudaSuccess) return set_error(MOE_ECUDA, "%s: smem attribute: %s", L.name, cudaGetErrorString(e));
  }
  int grid = gemm_sm_budget() & ~1;
  if (2 * L.max_tiles < grid) grid = 2 * L.max_tiles;
  if (grid < 2) grid = 2;
  GemmParams p = L.p;
  p.dbg = gemm_dbg();
  {
    static int rev = -1;  // MOE_GEMM_REVERSE bit m: walk mode m's tiles last-to-first (default as bsgemm.cu)
    if (rev < 0) {
      const char* e = getenv("MOE_GEMM_REVERSE");
      rev = e ? atoi(e) : (1 << DSD_ROW) | (1 << DS_COL) | (1 << DDS_COL);
    }
    // (the gathered DD^TS token ring is prefetched in forward tile order: no reversal there)
    p.reverse = ((rev >> MODE) & 1) && !(MODE != SDD && p.gather_a) ? 1 : 0;
  }
  p.trace = gemm_trace_slot();
  cudaError_t le = launch_k(kern, dim3(grid), dim3(P_THREADS), C::SMEM, stream, L.ta, L.tb, L.tc, L.td, p);
  if (le != cudaSuccess) return set_error(MOE_ECUDA, "%s: %s", L.name, cudaGetErrorString(le));
  MOE_CHECK_LAUNCH(L.name);
  return MOE_OK;
}

#define MOE_GEMM2_CASE(MODE, AMN, BMN, H) \
  if (L.mode == MODE && L.a_mn == AMN && L.b_mn == BMN && L.epi_h == H) return launch2_t<MODE, AMN, BMN, H>(L, stream);

bool gemm2_wide_h() { return Cfg2<true, SDD>::WIDE_H && Cfg2<true, SDD>::HC == 64; }
bool gemm2_h_coded() { return Cfg2<true, SDD>::HAS_TAB; }
bool gemm2_h_ring() { return Cfg2<true, SDD>::WIDE_H; }

moe_status gemm2_launch(const GemmLaunch& L, cudaStream_t stream) {
  MOE_GEMM2_CASE(SDD, false, true, false)      // SDD      X_g . W1 (+act, +pre)
  MOE_GEMM2_CASE(SDD, false, false, true)      // SDD^T    dY_g . W2^T (+act')
  MOE_GEMM2_CASE(SDD, false, false, false)
  MOE_GEMM2_CASE(DSD_ROW, false, true, false)  // DSD      A . W2
  MOE_GEMM2_CASE(DSD_ROW, false, false, false) // DSD^T    dH . W1^T
  MOE_GEMM2_CASE(DS_COL, true, true, false)    // DS^TD    A^T . dY_g
  MOE_GEMM2_CASE(DS_COL, true, false, false)
  MOE_GEMM2_CASE(DDS_COL, true, true, false)   // DD^TS    X_g^T . dH
  MOE_GEMM2_CASE(DDS_COL, false, true, false)
  return set_error(MOE_EUNSUPPORTED, "%s: no CTA-pair kernel for mode=%d a_mn=%d b_mn=%d", L.name, L.mode,
                   (int)L.a_mn, (int)L.b_mn);
}

}  // namespace moe
