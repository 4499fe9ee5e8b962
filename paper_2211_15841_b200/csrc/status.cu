// status.cu — error reporting, config validation and size queries of the C ABI
// (include/moe.h). Host only; no CUDA calls except the SM-count query.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>

#include "common.cuh"

namespace moe {

bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    // measured no gain inside a CUDA graph at MoE-XS (the kernel tails are
    // short and the persistent GEMMs leave no room to co-schedule): opt-in
    const char* e = getenv("MOE_PDL");
    on = (e && e[0] == '1') ? 1 : 0;
  }
  return on == 1;
}


void prefer_max_smem(const void* kern) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("MOE_CARVEOUT");
    on = (e && e[0] == '1') ? 1 : 0;
  }
  if (!on) return;
  // per thread: (kernel, device) pairs already set (a few dozen kernels)
  thread_local const void* done_k[256];
  thread_local int done_d[256];
  thread_local int n_done = 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  for (int i = 0; i < n_done; ++i)
    if (done_k[i] == kern && done_d[i] == dev) return;
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
  cudaGetLastError();
  if (n_done < 256) {
    done_k[n_done] = kern;
    done_d[n_done] = dev;
    ++n_done;
  }
}

static thread_local char g_err[512] = "";
static thread_local int g_launches = 0;
static std::atomic<long long> g_total_launches{0};

moe_status set_error(moe_status st, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return st;
}
void clear_error() { g_err[0] = 0; }
void count_launch(int n) {
  g_launches += n;
  g_total_launches += n;
}
void reset_launch_count() { g_launches = 0; }

moe_status check_config_gpu(const moe_config* cfg) {
  moe_status st = moe_check_config(cfg);
  return st;
}

moe_status check_topo(const moe_topology_t* t) {
  if (!t) return set_error(MOE_EINVAL, "topology pointer is NULL");
  if (!t->counts || !t->bins || !t->padded_bins || !t->sorted_idx || !t->pos || !t->sorted_pos ||
      !t->row_offsets || !t->col_indices || !t->row_indices || !t->t_col_offsets || !t->t_block_offsets ||
      !t->t_row_indices || !t->pair_bins || !t->row_src || !t->sizes || !t->brow_start || !t->brow_rows)
    return set_error(MOE_EINVAL, "topology has a NULL array");
  return MOE_OK;
}

bool router_on_tensor_cores(const moe_config* cfg) {
  return cfg->num_experts % 64 == 0 && cfg->num_experts <= 256 && cfg->top_k <= 8;
}

int router_bwd_parts(const moe_config* cfg) {
  // split of the token (K) dimension of dWr = x^T dlogits; fixed per config
  // (independent of the device) so the reduction order is deterministic
  int64_t parts;
  if (router_on_tensor_cores(cfg)) {
    const int64_t m_tiles = ceil_div(cfg->hidden, 128), k_iters = ceil_div(cfg->tokens, 64);
    parts = ceil_div(148, m_tiles);
    if (parts > k_iters) parts = k_iters;
  } else {
    parts = ceil_div(cfg->tokens, 256);
    if (parts > 256) parts = 256;
  }
  if (parts < 1) parts = 1;
  return (int)parts;
}

static size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

WsLayout ws_layout(const moe_config* cfg) {
  WsLayout L{};
  const int64_t R = cfg->tokens * cfg->top_k;
  const int64_t n_chunks = ceil_div(R > 0 ? R : 1, kTopoChunk);
  const int64_t rows = moe_max_padded_rows(cfg);
  const int64_t nnz = moe_max_nnz_blocks(cfg);
  const int64_t bs = cfg->block_size, h = cfg->hidden, E = cfg->num_experts;
  size_t off = 0;
  L.topo_chunk_counts = off;
  off = align256(off + sizeof(int32_t) * n_chunks * E);
  L.router_hist = off;
  off = align256(off + sizeof(int32_t) * ceil_div(cfg->tokens > 0 ? cfg->tokens : 1, 128) * E);
  L.topo_end = off;
  L.dy_g = off;
  off = align256(off + 2 * rows * h);
  L.dh = off;
  off = align256(off + 2 * nnz * bs * bs);
  L.dx_g = off;
  off = align256(off + 2 * rows * h);
  L.dgates = off;
  off = align256(off + 4 * R);
  L.dlogits = off;
  off = align256(off + 4 * cfg->tokens * E);
  L.dwr_part = off;
  off = align256(off + 4 * (size_t)router_bwd_parts(cfg) * h * E);
  L.aux = off;  // {loss, c[E]}, then per-part column sums and top-1 counts
  off = align256(off + 4 * (size_t)(1 + E) + 8 * (size_t)kAuxParts * E);
  L.total = off;
  return L;
}

}  // namespace moe

using namespace moe;

extern "C" {

const char* moe_last_error(void) { return g_err; }

int moe_last_launch_count(void) { return g_launches; }

int64_t moe_total_launch_count(void) { return g_total_launches.load(); }

moe_status moe_check_config(const moe_config* cfg) {
  if (!cfg) return set_error(MOE_EINVAL, "config pointer is NULL");
  if (cfg->tokens < 1) return set_error(MOE_EINVAL, "tokens=%lld must be >= 1", (long long)cfg->tokens);
  if (cfg->hidden < 1) return set_error(MOE_EINVAL, "hidden=%lld must be >= 1", (long long)cfg->hidden);
  if (cfg->num_experts < 1)
    return set_error(MOE_EINVAL, "num_experts=%lld must be >= 1", (long long)cfg->num_experts);
  if (cfg->top_k < 1 || cfg->top_k > cfg->num_experts)
    return set_error(MOE_EINVAL, "top_k=%lld must be in [1, num_experts=%lld]", (long long)cfg->top_k,
                     (long long)cfg->num_experts);
  if (cfg->block_size < 1) return set_error(MOE_EINVAL, "block_size must be >= 1");
  if (cfg->ffn_hidden < 1 || cfg->ffn_hidden % cfg->block_size)
    return set_error(MOE_ESHAPE, "ffn_hidden=%lld must be a positive multiple of block_size=%lld",
                     (long long)cfg->ffn_hidden, (long long)cfg->block_size);
  if (cfg->act < MOE_ACT_IDENTITY || cfg->act > MOE_ACT_RELU)
    return set_error(MOE_EINVAL, "act=%d is not a moe_act", cfg->act);
  if (cfg->capacity < 0) return set_error(MOE_EINVAL, "capacity=%d must be >= 0 (0 = dropless)", cfg->capacity);
  if (cfg->renormalize != 0 && cfg->renormalize != 1)
    return set_error(MOE_EINVAL, "renormalize=%d must be 0 or 1", cfg->renormalize);
  if (!(cfg->aux_loss_coeff >= 0.f) || isinf(cfg->aux_loss_coeff))
    return set_error(MOE_EINVAL, "aux_loss_coeff=%g must be finite and >= 0", (double)cfg->aux_loss_coeff);
  if (cfg->unpadded != 0 && cfg->unpadded != 1)
    return set_error(MOE_EINVAL, "unpadded=%d must be 0 or 1", cfg->unpadded);
  if (cfg->unpadded && cfg->capacity > 0)
    return set_error(MOE_EUNSUPPORTED, "unpadded=1 is dropless only (capacity=%d)", cfg->capacity);
  if (cfg->block_size != 128)
    return set_error(MOE_EUNSUPPORTED, "block_size=%lld: the sm_100a path implements 128x128 blocks (P:222)",
                     (long long)cfg->block_size);
  if (cfg->hidden % 256 || cfg->hidden > 2048)
    return set_error(MOE_EUNSUPPORTED, "hidden=%lld must be a multiple of 256 and <= 2048 on the GPU path",
                     (long long)cfg->hidden);
  if (cfg->num_experts > 1024)
    return set_error(MOE_EUNSUPPORTED, "num_experts=%lld > 1024", (long long)cfg->num_experts);
  if (cfg->tokens * cfg->top_k > (int64_t)1 << 30)
    return set_error(MOE_EUNSUPPORTED, "tokens*top_k too large for int32 indices");
  return MOE_OK;
}

int64_t moe_expert_capacity(int64_t tokens, int64_t num_experts, double capacity_factor) {
  if (tokens < 1 || num_experts < 1 || !(capacity_factor > 0)) return 0;
  return (int64_t)ceil((double)tokens * capacity_factor / (double)num_experts - 1e-12);
}

int64_t moe_max_padded_rows(const moe_config* cfg) {
  if (!cfg || cfg->block_size < 1) return 0;
  const int64_t R = cfg->tokens * cfg->top_k, bs = cfg->block_size;
  const int64_t nonempty = R < cfg->num_experts ? R : cfg->num_experts;
  return bs * ((R + nonempty * (bs - 1)) / bs);
}

int64_t moe_max_nnz_blocks(const moe_config* cfg) {
  if (!cfg || cfg->block_size < 1) return 0;
  return moe_max_padded_rows(cfg) / cfg->block_size * (cfg->ffn_hidden / cfg->block_size);
}

size_t moe_workspace_bytes(const moe_config* cfg) {
  if (!cfg) return 0;
  return ws_layout(cfg).total;
}

size_t moe_workspace_offset(const moe_config* cfg, int which) {
  if (!cfg) return (size_t)-1;
  const WsLayout L = ws_layout(cfg);
  switch (which) {
    case 0: return L.dy_g;
    case 1: return L.dh;
    case 2: return L.dx_g;
    case 3: return L.dgates;
    case 4: return L.dlogits;
    case 5: return L.aux;
    default: return (size_t)-1;
  }
}

int moe_device_sm_count(void) {
  static int cached = 0;
  if (!cached) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) ==
                                                   cudaSuccess)
      cached = n;
    else
      return 148;
  }
  return cached;
}

}  // extern "C"

// Host decode of the branch-coded activation (reading R24): the same table and
// index arithmetic as act_code_mul32 in gemm_util.cuh, for CPU tests.
#include "act_code_table.h"
namespace {
const uint16_t kActCodeTableHost[moe::kActCodeN] = MOE_ACT_CODE_TABLE_INIT;
float half_bits_to_float(uint16_t h) {
  const uint32_t s = (uint32_t)(h >> 15) << 31, e = (h >> 10) & 0x1f, m = h & 0x3ff;
  float f;
  if (e == 0) {
    f = ldexpf((float)m, -24);  // zero / subnormal
    return s ? -f : f;
  }
  uint32_t bits = s | ((e == 31 ? 255u : e - 15 + 127) << 23) | (m << 13);
  memcpy(&f, &bits, 4);
  return f;
}
}  // namespace

extern "C" moe_status moe_act_code_decode_host(int32_t act, const uint16_t* a_bits, float* out, int64_t n) {
  if (!a_bits || !out || n < 0) return moe::set_error(MOE_EINVAL, "moe_act_code_decode_host: bad arguments");
  if (act < 0 || act > 2) return moe::set_error(MOE_EINVAL, "moe_act_code_decode_host: bad act %d", act);
  for (int64_t i = 0; i < n; ++i) {
    const uint32_t u = a_bits[i];
    if (act == MOE_ACT_IDENTITY) {
      out[i] = 1.f;
    } else if (act == MOE_ACT_RELU) {
      out[i] = (u != 0u && u < 0x8000u) ? 1.f : 0.f;
    } else {
      // the key clamped to its sign's range (a negative key keeps its branch LSB), then rebased
      const uint32_t p_lo = (uint32_t)moe::kActCodeELo << 7, p_hi = ((uint32_t)moe::kActCodeEHiPos << 7) | 0x7fu;
      const uint32_t n_lo = 0x8000u | p_lo | (u & 1u), n_hi = 0x8000u | ((uint32_t)moe::kActCodeEHiNeg << 7) | 0x7fu;
      const bool neg = u >> 15;
      uint32_t c = u < (neg ? n_lo : p_lo) ? (neg ? n_lo : p_lo) : u;
      if (c > (neg ? n_hi : p_hi)) c = neg ? n_hi : p_hi;
      const uint32_t idx = neg ? c - (0x8000u | p_lo) + (uint32_t)moe::kActCodeNPos : c - p_lo;
      out[i] = half_bits_to_float(kActCodeTableHost[idx]);
    }
  }
  return MOE_OK;
}
