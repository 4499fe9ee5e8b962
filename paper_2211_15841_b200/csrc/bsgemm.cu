// bsgemm.cu — block-sparse SDD / DSD / DDS on sm_100a tensor cores.
//
// The paper's products (§5.1; Triton notation P:177) over the
// hybrid blocked-CSR-COO topology with transpose indices
// (P:287-292). One persistent, warp-specialised kernel template serves all of
// them; the modes differ only in how a 128 x BN output tile enumerates its
// K-steps and where TMA fetches the two operand tiles from:
//
//   SDD     out block s=(r,c)          K = dense dim, COO (row_indices, col_indices) lookup
//   DSD_ROW out [r-block, n-tile]      K walks the BCSR row r (row_offsets, col_indices)
//   DS_COL  out [c-block, n-tile]      K walks column c through the transpose index
//   DDS_COL out [m-tile, c-block]      K walks column c through the transpose index
//   DDS_ROW out [m-tile, r-block]      K walks the BCSR row r
//
// Transposition never moves values: a transposed sparse or dense operand is
// fed to tcgen05.mma as an MN-major instead of K-major shared-memory tile
// (descriptor bit), loaded by TMA from the same row-major storage.
//
// Warp roles (192 threads, 1 CTA/SM): warp 0 = TMA producer, warp 1 = TMEM
// allocator + single-thread MMA issuer, warps 2-5 = epilogue (TMEM -> regs ->
// global). Pipelines: STAGES-deep smem ring (full/empty mbarriers) and a
// double-buffered TMEM accumulator (tfull/tempty) so the epilogue of tile i
// overlaps the main loop of tile i+1.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "sm100.cuh"
#include "tma.cuh"

namespace moe {

using namespace sm100;

enum GemmMode { SDD = 0, DSD_ROW = 1, DS_COL = 2, DDS_COL = 3, DDS_ROW = 4 };
enum EpiKind { EPI_STORE = 0, EPI_ACT_FWD = 1, EPI_ACT_BWD = 2 };

struct GemmParams {
  const int32_t* sizes;  // {Tp, nnz}
  const int32_t* row_offsets;
  const int32_t* col_indices;
  const int32_t* row_indices;
  const int32_t* t_col_offsets;
  const int32_t* t_block_offsets;
  const int32_t* t_row_indices;
  int n_block_cols;  // E*F
  int dense_tiles;   // 128-wide tiles along the dense output dimension
  int k_dense;       // SDD: contraction length (multiple of 64)
  __nv_bfloat16* out;
  __nv_bfloat16* out_pre;
  const __nv_bfloat16* act_src;
  long long ld_out;
  int epi;
  int act;
};

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int BK = 64;
constexpr int STAGES = 6;
constexpr int A_BYTES = BM * BK * 2;
constexpr int B_BYTES = BN * BK * 2;
constexpr int STAGE_TX = A_BYTES + B_BYTES;
constexpr int TMEM_COLS = 2 * BN;
constexpr int NUM_THREADS = 192;
constexpr size_t SMEM_BYTES = 1024 + (size_t)STAGES * (A_BYTES + B_BYTES) + 256;

__device__ __forceinline__ int num_tiles(const GemmParams& p, int mode) {
  const int Tp = p.sizes[0], nnz = p.sizes[1];
  switch (mode) {
    case SDD: return nnz;
    case DSD_ROW: return (Tp / BM) * p.dense_tiles;
    case DS_COL: return p.n_block_cols * p.dense_tiles;
    case DDS_COL: return p.n_block_cols * p.dense_tiles;
    default: return (Tp / BM) * p.dense_tiles;  // DDS_ROW
  }
}

// Per-tile decode: number of 64-wide K steps, the sparse walk start, and the
// output-tile coordinates (major index `u` = block row/col, minor `v` = dense tile).
struct TileInfo {
  int kiters;
  int walk_begin;  // first storage index (row walk) or transpose position (col walk)
  int u, v;        // SDD: (r, c); DSD_ROW/DDS_ROW: (r, dense tile); DS_COL/DDS_COL: (c, dense tile)
  int s;           // SDD: block storage index
};

__device__ __forceinline__ TileInfo decode(const GemmParams& p, int mode, int tile) {
  TileInfo t;
  t.s = tile;
  if (mode == SDD) {
    t.u = __ldg(p.row_indices + tile);
    t.v = __ldg(p.col_indices + tile);
    t.kiters = p.k_dense / BK;
    t.walk_begin = 0;
  } else if (mode == DSD_ROW || mode == DDS_ROW) {
    t.u = tile / p.dense_tiles;
    t.v = tile % p.dense_tiles;
    const int b = __ldg(p.row_offsets + t.u), e = __ldg(p.row_offsets + t.u + 1);
    t.walk_begin = b;
    t.kiters = 2 * (e - b);
  } else {
    t.u = tile / p.dense_tiles;
    t.v = tile % p.dense_tiles;
    const int b = __ldg(p.t_col_offsets + t.u), e = __ldg(p.t_col_offsets + t.u + 1);
    t.walk_begin = b;
    t.kiters = 2 * (e - b);
  }
  return t;
}

__device__ __forceinline__ float act_fwd(int kind, float x) {
  if (kind == MOE_ACT_GELU_TANH) {
    const float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
    return 0.5f * x * (1.0f + tanhf(u));
  }
  if (kind == MOE_ACT_RELU) return x > 0.f ? x : 0.f;
  return x;
}
__device__ __forceinline__ float act_grad(int kind, float x) {
  if (kind == MOE_ACT_GELU_TANH) {
    const float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
    const float t = tanhf(u);
    const float du = 0.7978845608028654f * (1.0f + 3.0f * 0.044715f * x * x);
    return 0.5f * (1.0f + t) + 0.5f * x * (1.0f - t * t) * du;
  }
  if (kind == MOE_ACT_RELU) return x > 0.f ? 1.f : 0.f;
  return 1.f;
}

// Output tile origin (element offset) and leading dimension.
__device__ __forceinline__ long long out_origin(const GemmParams& p, int mode, const TileInfo& t) {
  switch (mode) {
    case SDD: return (long long)t.s * (BM * BN);
    case DSD_ROW: return (long long)t.u * BM * p.ld_out + (long long)t.v * BN;
    case DS_COL: return (long long)t.u * BM * p.ld_out + (long long)t.v * BN;
    case DDS_COL: return (long long)t.v * BM * p.ld_out + (long long)t.u * BN;
    default: return (long long)t.v * BM * p.ld_out + (long long)t.u * BN;  // DDS_ROW
  }
}

template <int MODE, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    bsgemm_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                  const GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_b + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
  }
  if (warp == 1) tmem_alloc<TMEM_COLS>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const int ntiles = num_tiles(p, MODE);

  if (warp == 0) {
    // ===================== TMA producer (whole warp walks, lane 0 issues) =====================
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const TileInfo t = decode(p, MODE, tile);
      int idx_a = 0, idx_b = 0;  // per-lane cached walk entries (32 sparse blocks at a time)
      for (int kit = 0; kit < t.kiters; ++kit) {
        const int blk = kit >> 1, kk = kit & 1;
        if (MODE != SDD && (blk & 31) == 0 && kk == 0) {
          const int q = t.walk_begin + blk + lane;
          const int lim = t.walk_begin + (t.kiters >> 1);
          if (q < lim) {
            if (MODE == DSD_ROW || MODE == DDS_ROW) {
              idx_a = q;                            // storage index
              idx_b = __ldg(p.col_indices + q);     // block column
            } else {
              idx_a = __ldg(p.t_block_offsets + q); // storage index
              idx_b = __ldg(p.t_row_indices + q);   // block row
            }
          }
        }
        const int sblk = __shfl_sync(0xffffffffu, idx_a, blk & 31);
        const int oblk = __shfl_sync(0xffffffffu, idx_b, blk & 31);
        mbar_wait(&empty[stage], phase ^ 1);
        if (lane == 0) {
          uint8_t* sa = smem_a + stage * A_BYTES;
          uint8_t* sb = smem_b + stage * B_BYTES;
          mbar_arrive_expect_tx(&full[stage], STAGE_TX);
          if (MODE == SDD) {
            const int k0 = kit * BK;
            // A: dense [rows, K] K-major tile at (k0, r*128)
            tma_load_2d(sa, &tmap_a, &full[stage], k0, t.u * BM);
            if (B_MN) {  // b [K, N] row-major: two 64-wide N chunks
              tma_load_2d(sb, &tmap_b, &full[stage], t.v * BN, k0);
              tma_load_2d(sb + 8192, &tmap_b, &full[stage], t.v * BN + 64, k0);
            } else {     // b [N, K] row-major
              tma_load_2d(sb, &tmap_b, &full[stage], k0, t.v * BN);
            }
          } else if (MODE == DSD_ROW) {
            // A = S_s (K-major); B rows of block column c
            tma_load_2d(sa, &tmap_a, &full[stage], kk * BK, sblk * BM);
            if (B_MN) {
              tma_load_2d(sb, &tmap_b, &full[stage], t.v * BN, oblk * BM + kk * BK);
              tma_load_2d(sb + 8192, &tmap_b, &full[stage], t.v * BN + 64, oblk * BM + kk * BK);
            } else {
              tma_load_2d(sb, &tmap_b, &full[stage], oblk * BM + kk * BK, t.v * BN);
            }
          } else if (MODE == DS_COL) {
            // A = S_blk^T (MN-major view of the row-major block); B = dense rows of block row r
            tma_load_2d(sa, &tmap_a, &full[stage], 0, sblk * BM + kk * BK);
            tma_load_2d(sa + 8192, &tmap_a, &full[stage], 64, sblk * BM + kk * BK);
            if (B_MN) {
              tma_load_2d(sb, &tmap_b, &full[stage], t.v * BN, oblk * BM + kk * BK);
              tma_load_2d(sb + 8192, &tmap_b, &full[stage], t.v * BN + 64, oblk * BM + kk * BK);
            } else {
              tma_load_2d(sb, &tmap_b, &full[stage], oblk * BM + kk * BK, t.v * BN);
            }
          } else if (MODE == DDS_COL) {
            // A = dense [m-tile, r-block]; B = S_blk (MN-major: N = block column contiguous)
            if (A_MN) {
              tma_load_2d(sa, &tmap_a, &full[stage], t.v * BM, oblk * BM + kk * BK);
              tma_load_2d(sa + 8192, &tmap_a, &full[stage], t.v * BM + 64, oblk * BM + kk * BK);
            } else {
              tma_load_2d(sa, &tmap_a, &full[stage], oblk * BM + kk * BK, t.v * BM);
            }
            tma_load_2d(sb, &tmap_b, &full[stage], 0, sblk * BM + kk * BK);
            tma_load_2d(sb + 8192, &tmap_b, &full[stage], 64, sblk * BM + kk * BK);
          } else {  // DDS_ROW: A = dense [m-tile, c-block]; B = S_s^T (K-major view)
            if (A_MN) {
              tma_load_2d(sa, &tmap_a, &full[stage], t.v * BM, oblk * BM + kk * BK);
              tma_load_2d(sa + 8192, &tmap_a, &full[stage], t.v * BM + 64, oblk * BM + kk * BK);
            } else {
              tma_load_2d(sa, &tmap_a, &full[stage], oblk * BM + kk * BK, t.v * BM);
            }
            tma_load_2d(sb, &tmap_b, &full[stage], kk * BK, sblk * BM);
          }
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (one thread) =====================
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(BM, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const TileInfo t = decode(p, MODE, tile);
        if (t.kiters == 0) continue;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kit = 0; kit < t.kiters; ++kit) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(smem_a + stage * A_BYTES);
          const uint32_t b_base = smem_u32(smem_b + stage * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t adesc =
                A_MN ? make_sdesc(a_base + k * 2048, 8192, 1024) : make_sdesc(a_base + k * 32, 16, 1024);
            const uint64_t bdesc =
                B_MN ? make_sdesc(b_base + k * 2048, 8192, 1024) : make_sdesc(b_base + k * 32, 16, 1024);
            mma_bf16(d_tmem, adesc, bdesc, idesc, (kit | k) != 0);
          }
          mma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // ===================== epilogue (warps 2..5) =====================
    const int q = warp & 3;          // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;   // output row within the tile
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const TileInfo t = decode(p, MODE, tile);
      __nv_bfloat16* out_row = p.out + out_origin(p, MODE, t) + (long long)row * (MODE == SDD ? BN : p.ld_out);
      if (t.kiters == 0) {  // empty block column (expert without tokens): zero output
        uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int c = 0; c < BN; c += 8) *reinterpret_cast<uint4*>(out_row + c) = z;
        continue;
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int chunk = 0; chunk < BN / 32; ++chunk) {
        uint32_t r[32];
        tmem_ld32(taddr + chunk * 32, r);
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
        const int col = chunk * 32;
        if (p.epi == EPI_ACT_FWD) {
          if (p.out_pre) {
            __nv_bfloat16* pre_row = p.out_pre + (long long)t.s * (BM * BN) + (long long)row * BN + col;
#pragma unroll
            for (int i = 0; i < 32; i += 8) {
              uint4 w = make_uint4(pack_bf16x2(v[i], v[i + 1]), pack_bf16x2(v[i + 2], v[i + 3]),
                                   pack_bf16x2(v[i + 4], v[i + 5]), pack_bf16x2(v[i + 6], v[i + 7]));
              *reinterpret_cast<uint4*>(pre_row + i) = w;
            }
          }
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = act_fwd(p.act, v[i]);
        } else if (p.epi == EPI_ACT_BWD) {
          const __nv_bfloat16* src = p.act_src + (long long)t.s * (BM * BN) + (long long)row * BN + col;
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            uint4 w = *reinterpret_cast<const uint4*>(src + i);
            const __nv_bfloat16* hv = reinterpret_cast<const __nv_bfloat16*>(&w);
#pragma unroll
            for (int j = 0; j < 8; ++j) v[i + j] *= act_grad(p.act, __bfloat162float(hv[j]));
          }
        }
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 w = make_uint4(pack_bf16x2(v[i], v[i + 1]), pack_bf16x2(v[i + 2], v[i + 3]),
                               pack_bf16x2(v[i + 4], v[i + 5]), pack_bf16x2(v[i + 6], v[i + 7]));
          *reinterpret_cast<uint4*>(out_row + col + i) = w;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<TMEM_COLS>(tmem_base);
  }
}

// ------------------------------------------------------------------ host side

template <int MODE, bool A_MN, bool B_MN>
static moe_status launch(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p, int max_tiles,
                         cudaStream_t stream, const char* name) {
  auto kern = bsgemm_kernel<MODE, A_MN, B_MN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES);
    if (e != cudaSuccess) return set_error(MOE_ECUDA, "%s: smem attribute: %s", name, cudaGetErrorString(e));
    attr_set = true;
  }
  int grid = moe_device_sm_count();
  if (max_tiles < grid) grid = max_tiles;
  if (grid < 1) grid = 1;
  kern<<<grid, NUM_THREADS, SMEM_BYTES, stream>>>(ta, tb, p);
  MOE_CHECK_LAUNCH(name);
  return MOE_OK;
}

static GemmParams base_params(const moe_config* cfg, const moe_topology_t* topo) {
  GemmParams p{};
  p.sizes = topo->sizes;
  p.row_offsets = topo->row_offsets;
  p.col_indices = topo->col_indices;
  p.row_indices = topo->row_indices;
  p.t_col_offsets = topo->t_col_offsets;
  p.t_block_offsets = topo->t_block_offsets;
  p.t_row_indices = topo->t_row_indices;
  p.n_block_cols = (int)(cfg->num_experts * cfg->ffn_hidden / cfg->block_size);
  p.dense_tiles = (int)(cfg->hidden / BN);
  p.k_dense = (int)cfg->hidden;
  p.epi = EPI_STORE;
  p.act = MOE_ACT_IDENTITY;
  return p;
}

}  // namespace moe

using namespace moe;

extern "C" {

moe_status moe_sdd(const moe_config* cfg, const void* a, const void* b, int trans_b, const moe_topology_t* topo,
                   int32_t act, const void* act_grad_src, void* out_s, void* out_pre, void* stream) {
  MOE_TRY(moe_check_config(cfg));
  MOE_TRY(check_topo(topo));
  MOE_CHECK_ARG(a && b && out_s, "moe_sdd: NULL operand");
  MOE_CHECK_ARG(act >= 0 && act <= 2, "moe_sdd: bad act %d", act);
  const int64_t rows = moe_max_padded_rows(cfg), nnz = moe_max_nnz_blocks(cfg);
  const int64_t h = cfg->hidden, N = cfg->num_experts * cfg->ffn_hidden;
  CUtensorMap ta, tb;
  MOE_TRY(make_tmap_bf16(&ta, a, h, rows, h, 64, 128, "moe_sdd a"));
  GemmParams p = base_params(cfg, topo);
  p.out = reinterpret_cast<__nv_bfloat16*>(out_s);
  p.out_pre = reinterpret_cast<__nv_bfloat16*>(out_pre);
  p.act_src = reinterpret_cast<const __nv_bfloat16*>(act_grad_src);
  p.ld_out = BN;
  p.act = act;
  p.epi = act_grad_src ? EPI_ACT_BWD : ((act != MOE_ACT_IDENTITY || out_pre) ? EPI_ACT_FWD : EPI_STORE);
  if (!trans_b) {  // b [h, E*f]
    MOE_TRY(make_tmap_bf16(&tb, b, N, h, N, 64, 64, "moe_sdd b"));
    return launch<SDD, false, true>(ta, tb, p, (int)nnz, as_stream(stream), "moe_sdd");
  } else {  // b [E*f, h]
    MOE_TRY(make_tmap_bf16(&tb, b, h, N, h, 64, 128, "moe_sdd b^T"));
    return launch<SDD, false, false>(ta, tb, p, (int)nnz, as_stream(stream), "moe_sdd(T)");
  }
}

moe_status moe_dsd(const moe_config* cfg, const void* s, int trans_s, const void* b, int trans_b,
                   const moe_topology_t* topo, void* out, void* stream) {
  MOE_TRY(moe_check_config(cfg));
  MOE_TRY(check_topo(topo));
  MOE_CHECK_ARG(s && b && out, "moe_dsd: NULL operand");
  const int64_t rows = moe_max_padded_rows(cfg), nnz = moe_max_nnz_blocks(cfg);
  const int64_t h = cfg->hidden, N = cfg->num_experts * cfg->ffn_hidden;
  GemmParams p = base_params(cfg, topo);
  p.out = reinterpret_cast<__nv_bfloat16*>(out);
  p.ld_out = h;
  CUtensorMap ta, tb;
  if (!trans_s) {
    // S [rows, E*f] values as [nnz*128, 128] row-major, K-major A
    MOE_TRY(make_tmap_bf16(&ta, s, 128, nnz * 128, 128, 64, 128, "moe_dsd s"));
    const int max_tiles = (int)(rows / BM * p.dense_tiles);
    if (!trans_b) {  // b [E*f, h]: MN-major B
      MOE_TRY(make_tmap_bf16(&tb, b, h, N, h, 64, 64, "moe_dsd b"));
      return launch<DSD_ROW, false, true>(ta, tb, p, max_tiles, as_stream(stream), "moe_dsd");
    } else {  // b [h, E*f]: K-major B
      MOE_TRY(make_tmap_bf16(&tb, b, N, h, N, 64, 128, "moe_dsd b^T"));
      return launch<DSD_ROW, false, false>(ta, tb, p, max_tiles, as_stream(stream), "moe_dsd(T)");
    }
  } else {
    MOE_TRY(make_tmap_bf16(&ta, s, 128, nnz * 128, 128, 64, 64, "moe_dsd s^T"));
    const int max_tiles = p.n_block_cols * p.dense_tiles;
    if (!trans_b) {  // b [rows, h]
      MOE_TRY(make_tmap_bf16(&tb, b, h, rows, h, 64, 64, "moe_dsd b"));
      return launch<DS_COL, true, true>(ta, tb, p, max_tiles, as_stream(stream), "moe_dsd(S^T)");
    } else {  // b [h, rows]
      MOE_TRY(make_tmap_bf16(&tb, b, rows, h, rows, 64, 128, "moe_dsd b^T"));
      return launch<DS_COL, true, false>(ta, tb, p, max_tiles, as_stream(stream), "moe_dsd(S^T,T)");
    }
  }
}

moe_status moe_dds(const moe_config* cfg, const void* a, int trans_a, const void* s, int trans_s,
                   const moe_topology_t* topo, void* out, void* stream) {
  MOE_TRY(moe_check_config(cfg));
  MOE_TRY(check_topo(topo));
  MOE_CHECK_ARG(a && s && out, "moe_dds: NULL operand");
  const int64_t rows = moe_max_padded_rows(cfg), nnz = moe_max_nnz_blocks(cfg);
  const int64_t h = cfg->hidden, N = cfg->num_experts * cfg->ffn_hidden;
  GemmParams p = base_params(cfg, topo);
  p.out = reinterpret_cast<__nv_bfloat16*>(out);
  CUtensorMap ta, tb;
  if (!trans_s) {
    // out [h, E*f] = A_eff [h, rows] . S ; walk columns via the transpose index
    p.ld_out = N;
    MOE_TRY(make_tmap_bf16(&tb, s, 128, nnz * 128, 128, 64, 64, "moe_dds s"));
    const int max_tiles = p.n_block_cols * p.dense_tiles;
    if (trans_a) {  // a = [rows, h]: A_eff = a^T, MN-major
      MOE_TRY(make_tmap_bf16(&ta, a, h, rows, h, 64, 64, "moe_dds a^T"));
      return launch<DDS_COL, true, true>(ta, tb, p, max_tiles, as_stream(stream), "moe_dds(T)");
    } else {  // a = [h, rows]: K-major
      MOE_TRY(make_tmap_bf16(&ta, a, rows, h, rows, 64, 128, "moe_dds a"));
      return launch<DDS_COL, false, true>(ta, tb, p, max_tiles, as_stream(stream), "moe_dds");
    }
  } else {
    // out [h, rows] = A_eff [h, E*f] . S^T ; walk rows
    p.ld_out = rows;
    MOE_TRY(make_tmap_bf16(&tb, s, 128, nnz * 128, 128, 64, 128, "moe_dds s^T"));
    const int max_tiles = (int)(rows / BM * p.dense_tiles);
    if (trans_a) {  // a = [E*f, h]
      MOE_TRY(make_tmap_bf16(&ta, a, h, N, h, 64, 64, "moe_dds a^T"));
      return launch<DDS_ROW, true, false>(ta, tb, p, max_tiles, as_stream(stream), "moe_dds(T,S^T)");
    } else {  // a = [h, E*f]
      MOE_TRY(make_tmap_bf16(&ta, a, N, h, N, 64, 128, "moe_dds a"));
      return launch<DDS_ROW, false, false>(ta, tb, p, max_tiles, as_stream(stream), "moe_dds(S^T)");
    }
  }
}

}  // extern "C"
