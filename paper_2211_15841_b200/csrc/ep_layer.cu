// ep_layer.cu — the expert-parallel dMoE layer as one C-ABI object (SURVEY
// §8(b) moe_ep_init / moe_ep_forward / moe_ep_backward / moe_ep_destroy).
//
// Expert parallelism ("data and expert model parallelism"; P:355
// "8-way expert model parallelism for MoE layers and data parallelism for all
// other layers"): rank r of P owns experts [r E/P, (r+1) E/P) and their W1 /
// W2 slices; the router Wr is replicated. The token exchange is the
// device-initiated peer-memory transport of ep_p2p.cu (stores into every
// owner's IPC window over NVLink, on-device count exchange), so
// a whole forward + backward is stream-ordered with no host synchronisation
// and can be captured in a CUDA graph.
//
// Forward (Fig. 5, split at the exchange):
//   token owner:  router + top-k -> topology over the global experts
//                  -> count exchange -> dispatch of x rows straight
//                 into the owners' padded expert-grouped layout
//   expert side:  topology from the per-source counts -> zero pad rows ->
//                 SDD (+act, act' saved) -> DSD -> combine back
//   token owner:  gate-weighted un-permutation
// Backward (§5.1), mirrored: scatter-backward + softmax backward
// on the owner (b1, b7), dy dispatch, SDD^T (b2), DS^TD (b3), DD^TS (b5),
// DSD^T (b4) on the expert side, dX combine, gather-backward + router dx
// (b6, b7) on the owner; dWr = x^T dlogits on a side stream. dWr is this
// rank's partial: the data-parallel sum over ranks is the caller's collective
// (moe.h: MOE_ENCCL is reserved; the library issues no collective).
//
// The object owns every buffer (allocated once at init) and the state of ONE
// forward in flight: moe_ep_backward must follow the forward it differentiates
// (a step counter enforces it).
#include <cuda_runtime.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "bsgemm.cuh"
#include "common.cuh"
#include "permute.cuh"

using namespace moe;

struct moe_ep {
  moe_ep_desc d;
  int device = -1;
  moe_config cfg_l{};  // token owner: tokens = max_tokens, E global experts, top_k
  moe_config cfg_e{};  // expert side at capacity: tokens = recv rows cap, E/P experts, top_k 1
  moe_ep_t ex{};       // exchange descriptor (ep_p2p.cu)
  void* window = nullptr;
  std::vector<void*> mapped;  // peers' windows opened here
  bool connected = false;
  std::vector<void*> allocs;
  // token-owner state
  moe_topology_t topo_l{};
  void* ws_l = nullptr;
  float* logits = nullptr;
  int32_t* idx = nullptr;
  float* gates = nullptr;
  float* dgates = nullptr;
  void* dlogits = nullptr;    // bf16 [T, E]
  void* dy_sorted = nullptr;  // bf16 [T*k, h]
  // expert-side state
  moe_topology_t topo_e{};
  void* ws_e = nullptr;
  void* a = nullptr;          // bf16 [max_nnz_e, bs, bs]
  void* act_deriv = nullptr;  // bf16 [max_nnz_e, bs, bs] (NULL for identity)
  void* dh = nullptr;         // bf16 [max_nnz_e, bs, bs]
  void* y_g = nullptr;        // bf16 [max_rows_e, h]
  void* dx_g = nullptr;       // bf16 [max_rows_e, h]
  // the combine fused into the DSD / DSD^T (NEXT-1): each padded row's address
  // in its source's return region (moe_ep_combine_dest), the rows stored there
  // by moe_dsd_rows; y_g / dx_g then stay unused
  uint64_t* dest_y = nullptr;   // [max_rows_e]
  uint64_t* dest_dx = nullptr;  // [max_rows_e]
  int64_t rows_e = 0;
  bool fused_combine = true;
  // side stream for dWr
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  long long fwd_step = 0, bwd_of = -1;
  int64_t tokens = 0;  // of the forward in flight
};

namespace {

moe_status ep_alloc(moe_ep* ep, void** p, size_t bytes) {
  bytes = bytes ? (bytes + 255) & ~size_t(255) : 256;
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess) return set_error(MOE_ECUDA, "moe_ep_init: cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
  ep->allocs.push_back(*p);
  return MOE_OK;
}

// Device arrays of a topology sized to the worst case of cfg (moe.h moe_topology_t).
moe_status ep_topology(moe_ep* ep, const moe_config* cfg, moe_topology_t* t) {
  const int64_t E = cfg->num_experts, bs = cfg->block_size, R = cfg->tokens * cfg->top_k;
  const int64_t rows = moe_max_padded_rows(cfg), nnz = moe_max_nnz_blocks(cfg), F = cfg->ffn_hidden / bs;
  const int64_t n[] = {E, E, E, R, R, R, rows / bs + 1, nnz, nnz, E * F + 1, nnz, nnz, E, rows, 3, rows / bs, rows / bs};
  int64_t total = 0;
  for (int64_t v : n) total += (v + 3) / 4 * 4;  // 16-byte aligned fields (int4 loads of row_src)
  void* buf;
  MOE_TRY(ep_alloc(ep, &buf, sizeof(int32_t) * total));
  int32_t* p = reinterpret_cast<int32_t*>(buf);
  int32_t** f[] = {&t->counts, &t->bins, &t->padded_bins, &t->sorted_idx, &t->pos, &t->sorted_pos,
                   &t->row_offsets, &t->col_indices, &t->row_indices, &t->t_col_offsets, &t->t_block_offsets,
                   &t->t_row_indices, &t->pair_bins, &t->row_src, &t->sizes, &t->brow_start, &t->brow_rows};
  static_assert(sizeof(f) / sizeof(f[0]) == 17, "moe_topology_t has 17 arrays");
  for (int i = 0; i < 17; ++i) {
    *f[i] = p;
    p += (n[i] + 3) / 4 * 4;
  }
  return MOE_OK;
}

void ep_free_all(moe_ep* ep) {
  for (void* m : ep->mapped)
    if (m) cudaIpcCloseMemHandle(m);
  ep->mapped.clear();
  for (void* p : ep->allocs) cudaFree(p);
  ep->allocs.clear();
  if (ep->window) cudaFree(ep->window);
  ep->window = nullptr;
  if (ep->side) cudaStreamDestroy(ep->side);
  if (ep->fork) cudaEventDestroy(ep->fork);
  if (ep->join) cudaEventDestroy(ep->join);
  ep->side = nullptr;
  ep->fork = ep->join = nullptr;
}

char* win_region(const moe_ep* ep, int which) {
  return reinterpret_cast<char*>(ep->window) +
         moe_ep_window_offset(ep->d.nranks, (int)ep->d.num_experts, ep->d.hidden, ep->ex.cap_rows,
                              ep->ex.owner_rows, which);
}

moe_status ep_ready(const moe_ep* ep, const char* fn) {
  MOE_CHECK_ARG(ep, "%s: NULL layer", fn);
  MOE_CHECK_ARG(ep->connected, "%s: moe_ep_connect has not been called", fn);
  int dev = -1;
  cudaGetDevice(&dev);
  MOE_CHECK_ARG(dev == ep->device, "%s: current device %d, the layer lives on device %d", fn, dev, ep->device);
  return MOE_OK;
}

}  // namespace

extern "C" {

moe_status moe_ep_init(moe_ep** out, const moe_ep_desc* d, int device) {
  MOE_CHECK_ARG(out && d, "moe_ep_init: NULL pointer");
  *out = nullptr;
  MOE_CHECK_ARG(d->nranks >= 1 && d->rank >= 0 && d->rank < d->nranks, "moe_ep_init: rank %d of %d", d->rank,
                d->nranks);
  MOE_CHECK_ARG(d->num_experts % d->nranks == 0, "moe_ep_init: num_experts=%lld not divisible by nranks=%d",
                (long long)d->num_experts, d->nranks);
  MOE_CHECK_ARG(d->max_tokens >= 1, "moe_ep_init: max_tokens must be >= 1");
  moe_config cl{};
  cl.tokens = d->max_tokens;
  cl.hidden = d->hidden;
  cl.num_experts = d->num_experts;
  cl.top_k = d->top_k;
  cl.ffn_hidden = d->ffn_hidden;
  cl.block_size = d->block_size;
  cl.act = d->act;
  cl.renormalize = d->renormalize;
  cl.aux_loss_coeff = d->aux_loss_coeff;
  MOE_TRY(moe_check_config(&cl));
  MOE_CHECK_ARG(d->hidden % 256 == 0 && d->hidden <= 2048,
                "moe_ep_init: hidden=%lld: the exchange kernels move rows in 512-byte vectors (hidden %% 256 == 0, "
                "<= 2048)", (long long)d->hidden);
  const int64_t full = (int64_t)d->nranks * d->max_tokens * d->top_k;
  const int64_t cap = d->recv_rows_cap > 0 ? d->recv_rows_cap : full;
  MOE_CHECK_ARG(cap <= full, "moe_ep_init: recv_rows_cap=%lld above nranks*max_tokens*top_k=%lld",
                (long long)cap, (long long)full);
  int prev_device = 0;
  cudaGetDevice(&prev_device);
  cudaError_t ce = cudaSetDevice(device);
  if (ce != cudaSuccess) return set_error(MOE_ECUDA, "moe_ep_init: cudaSetDevice(%d): %s", device, cudaGetErrorString(ce));
  struct RestoreDevice {  // the caller's current device is left as it was
    int d;
    ~RestoreDevice() { cudaSetDevice(d); }
  } restore{prev_device};

  moe_ep* ep = new moe_ep();
  ep->d = *d;
  ep->device = device;
  ep->cfg_l = cl;
  ep->cfg_e = cl;
  ep->cfg_e.tokens = cap;
  ep->cfg_e.num_experts = d->num_experts / d->nranks;
  ep->cfg_e.top_k = 1;
  ep->cfg_e.renormalize = 0;
  ep->cfg_e.aux_loss_coeff = 0.f;
  ep->cfg_e.capacity = 0;
  auto fail = [&](moe_status st) {
    ep_free_all(ep);
    delete ep;
    return st;
  };
  moe_status st;
  // this rank's window (receive and return regions, counters, histograms)
  const int P = d->nranks, E = (int)d->num_experts;
  const size_t wb = moe_ep_window_bytes(P, E, d->hidden, cap, d->max_tokens * d->top_k);
  if ((st = moe_ep_window_alloc(wb, &ep->window)) != MOE_OK) return fail(st);
  ep->mapped.assign(P, nullptr);
  void *peers, *plan;
  if ((st = ep_alloc(ep, &peers, sizeof(uint64_t) * P)) != MOE_OK) return fail(st);
  if ((st = ep_alloc(ep, &plan, sizeof(int32_t) * moe_ep_plan_ints(P, E))) != MOE_OK) return fail(st);
  cudaMemset(plan, 0, sizeof(int32_t) * moe_ep_plan_ints(P, E));
  ep->ex.nranks = P;
  ep->ex.rank = d->rank;
  ep->ex.num_experts = E;
  ep->ex.hidden = (int32_t)d->hidden;
  ep->ex.cap_rows = cap;
  ep->ex.owner_rows = d->max_tokens * d->top_k;
  ep->ex.peers = peers;
  ep->ex.plan = reinterpret_cast<int32_t*>(plan);
  // token-owner buffers
  const int64_t T = d->max_tokens, k = d->top_k, h = d->hidden;
  if ((st = ep_topology(ep, &ep->cfg_l, &ep->topo_l)) != MOE_OK) return fail(st);
  if ((st = ep_alloc(ep, &ep->ws_l, moe_workspace_bytes(&ep->cfg_l))) != MOE_OK) return fail(st);
  if ((st = ep_alloc(ep, (void**)&ep->logits, sizeof(float) * T * E)) != MOE_OK) return fail(st);
  if ((st = ep_alloc(ep, (void**)&ep->idx, sizeof(int32_t) * T * k)) != MOE_OK) return fail(st);
  if ((st = ep_alloc(ep, (void**)&ep->gates, sizeof(float) * T * k)) != MOE_OK) return fail(st);
  if ((st = ep_alloc(ep, (void**)&ep->dgates, sizeof(float) * T * k)) != MOE_OK) return fail(st);
  if ((st = ep_alloc(ep, &ep->dlogits, 2 * T * E)) != MOE_OK) return fail(st);
  if ((st = ep_alloc(ep, &ep->dy_sorted, 2 * T * k * h)) != MOE_OK) return fail(st);
  // expert-side buffers at capacity
  const int64_t nnz_e = moe_max_nnz_blocks(&ep->cfg_e), rows_e = moe_max_padded_rows(&ep->cfg_e);
  const int64_t blk = d->block_size * d->block_size;
  if ((st = ep_topology(ep, &ep->cfg_e, &ep->topo_e)) != MOE_OK) return fail(st);
  if ((st = ep_alloc(ep, &ep->ws_e, moe_workspace_bytes(&ep->cfg_e))) != MOE_OK) return fail(st);
  if ((st = ep_alloc(ep, &ep->a, 2 * nnz_e * blk)) != MOE_OK) return fail(st);
  if (d->act != MOE_ACT_IDENTITY && (st = ep_alloc(ep, &ep->act_deriv, 2 * nnz_e * blk)) != MOE_OK) return fail(st);
  if ((st = ep_alloc(ep, &ep->dh, 2 * nnz_e * blk)) != MOE_OK) return fail(st);
  if ((st = ep_alloc(ep, &ep->y_g, 2 * rows_e * h)) != MOE_OK) return fail(st);
  if ((st = ep_alloc(ep, &ep->dx_g, 2 * rows_e * h)) != MOE_OK) return fail(st);
  if ((st = ep_alloc(ep, (void**)&ep->dest_y, sizeof(uint64_t) * rows_e)) != MOE_OK) return fail(st);
  if ((st = ep_alloc(ep, (void**)&ep->dest_dx, sizeof(uint64_t) * rows_e)) != MOE_OK) return fail(st);
  ep->rows_e = rows_e;
  {
    const char* fc = getenv("MOE_EP_FUSED_COMBINE");  // 0: the separate combine copy (A/B)
    ep->fused_combine = !(fc && fc[0] == '0');
  }
  if (cudaStreamCreateWithFlags(&ep->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ep->fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ep->join, cudaEventDisableTiming) != cudaSuccess)
    return fail(set_error(MOE_ECUDA, "moe_ep_init: stream / event creation failed"));
  if ((ce = cudaDeviceSynchronize()) != cudaSuccess)
    return fail(set_error(MOE_ECUDA, "moe_ep_init: %s", cudaGetErrorString(ce)));
  *out = ep;
  return MOE_OK;
}

moe_status moe_ep_get_handle(const moe_ep* ep, void* handle) {
  MOE_CHECK_ARG(ep && handle, "moe_ep_get_handle: NULL pointer");
  return moe_ipc_get_handle(ep->window, handle);
}

moe_status moe_ep_connect(moe_ep* ep, const void* handles) {
  MOE_CHECK_ARG(ep && handles, "moe_ep_connect: NULL pointer");
  MOE_CHECK_ARG(!ep->connected, "moe_ep_connect: already connected");
  const int P = ep->d.nranks;
  std::vector<uint64_t> ptrs(P);
  for (int q = 0; q < P; ++q) {
    if (q == ep->d.rank) {
      ptrs[q] = reinterpret_cast<uint64_t>(ep->window);
      continue;
    }
    void* w = nullptr;
    const moe_status st = moe_ipc_open_handle(reinterpret_cast<const char*>(handles) + 64 * q, &w);
    if (st != MOE_OK) return set_error(st, "moe_ep_connect: rank %d's window: %s", q, moe_last_error());
    ep->mapped[q] = w;
    ptrs[q] = reinterpret_cast<uint64_t>(w);
  }
  cudaError_t e = cudaMemcpy(const_cast<void*>(ep->ex.peers), ptrs.data(), sizeof(uint64_t) * P,
                             cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return set_error(MOE_ECUDA, "moe_ep_connect: %s", cudaGetErrorString(e));
  ep->connected = true;
  return MOE_OK;
}

moe_status moe_ep_forward(moe_ep* ep, int64_t tokens, const moe_weights* w, const void* x, void* y, void* stream) {
  MOE_TRY(ep_ready(ep, "moe_ep_forward"));
  MOE_CHECK_ARG(w && w->wr && w->w1 && w->w2 && x && y, "moe_ep_forward: NULL pointer");
  MOE_CHECK_ARG(tokens >= 1 && tokens <= ep->d.max_tokens, "moe_ep_forward: tokens=%lld outside [1, max_tokens=%lld]",
                (long long)tokens, (long long)ep->d.max_tokens);
  reset_launch_count();
  moe_config cl = ep->cfg_l;
  cl.tokens = tokens;
  const moe_config* ce = &ep->cfg_e;
  const bool id = ep->d.act == MOE_ACT_IDENTITY;
  // token owner: (1) router + top-k [+ aux loss], (2) topology over the global experts
  MOE_TRY(moe_router_topology(&cl, x, w->wr, ep->logits, ep->idx, ep->gates, &ep->topo_l, ep->ws_l, stream));
  if (cl.aux_loss_coeff > 0.f) MOE_TRY(moe_load_balance_loss(&cl, ep->logits, ep->idx, ep->ws_l, stream));
  // count exchange + dispatch into the owners' padded expert-grouped layouts
  MOE_TRY(moe_ep_exchange_counts(&ep->ex, ep->topo_l.counts, stream));
  MOE_TRY(moe_ep_dispatch_padded(&ep->ex, MOE_EP_RECV_X, x, ep->topo_l.sorted_pos, (int)cl.top_k, stream));
  MOE_TRY(moe_ep_wait(&ep->ex, MOE_EP_RECV_X, stream));
  void* x_g = win_region(ep, MOE_EP_RECV_X);
  // expert side: topology from the per-source counts, SDD (+act, act' saved), DSD
  const int32_t* ccomp = ep->ex.plan + moe_ep_plan_offset(ep->d.nranks, (int)ep->d.num_experts, 0);
  MOE_TRY(moe_topology_counts(ce, ccomp, ep->d.nranks, &ep->topo_e, stream));
  MOE_TRY(moe_zero_pad_rows(ce, &ep->topo_e, x_g, stream));
  MOE_TRY(moe_sdd_deriv(ce, x_g, w->w1, 0, &ep->topo_e, ep->d.act, nullptr, ep->a, id ? nullptr : ep->act_deriv,
                        stream));
  // combine back to the token owners, then the gate-weighted un-permutation;
  // fused (NEXT-1): the DSD stores every row straight into its source's return region
  if (ep->fused_combine) {
    MOE_TRY(moe_ep_combine_dest(&ep->ex, MOE_EP_RET_Y, ep->dest_y, ep->rows_e, stream));
    MOE_TRY(moe_dsd_rows(ce, ep->a, w->w2, 0, &ep->topo_e, ep->dest_y, stream));
    MOE_TRY(moe_ep_signal(&ep->ex, MOE_EP_RET_Y, stream));
  } else {
    MOE_TRY(moe_dsd(ce, ep->a, 0, w->w2, 0, &ep->topo_e, ep->y_g, stream));
    MOE_TRY(moe_ep_combine_padded(&ep->ex, MOE_EP_RET_Y, ep->y_g, stream));
  }
  MOE_TRY(moe_ep_wait(&ep->ex, MOE_EP_RET_Y, stream));
  MOE_TRY(moe_unsort_rows(&cl, win_region(ep, MOE_EP_RET_Y), &ep->topo_l, ep->gates, y, stream));
  ep->tokens = tokens;
  ep->bwd_of = -1;
  ++ep->fwd_step;
  return MOE_OK;
}

moe_status moe_ep_backward(moe_ep* ep, const moe_weights* w, const void* x, const void* dy, void* dx, moe_grads* g,
                           void* stream) {
  MOE_TRY(ep_ready(ep, "moe_ep_backward"));
  MOE_CHECK_ARG(w && w->wr && w->w1 && w->w2 && x && dy && dx && g && g->dwr && g->dw1 && g->dw2,
                "moe_ep_backward: NULL pointer");
  MOE_CHECK_ARG(ep->fwd_step > 0 && ep->bwd_of != ep->fwd_step,
                "moe_ep_backward: no forward in flight (one backward per forward: the layer keeps the state of "
                "the last forward only)");
  reset_launch_count();
  moe_config cl = ep->cfg_l;
  cl.tokens = ep->tokens;
  const moe_config* ce = &ep->cfg_e;
  const bool id = ep->d.act == MOE_ACT_IDENTITY;
  const bool fused = router_on_tensor_cores(&cl);
  cudaStream_t s = as_stream(stream);
  const void* y_sorted = win_region(ep, MOE_EP_RET_Y);
  bool forked = false;
  // b1 (+ b7's softmax backward) on the token owner
  if (fused) {
    MOE_TRY(moe_unsort_rows_bwd_router(&cl, dy, y_sorted, &ep->topo_l, ep->gates, ep->logits, ep->idx,
                                       ep->dy_sorted, ep->dgates, ep->dlogits, stream));
    MOE_TRY(moe_add_aux_dlogits(&cl, ep->logits, ep->dlogits, ep->ws_l, stream));
    // b7 dWr = x^T . dlogits needs nothing else: side stream, beside the exchange and the expert products
    if (cudaEventRecord(ep->fork, s) != cudaSuccess || cudaStreamWaitEvent(ep->side, ep->fork, 0) != cudaSuccess)
      return set_error(MOE_ECUDA, "moe_ep_backward: fork failed");
    MOE_TRY(moe_router_dwr(&cl, x, ep->dlogits, g->dwr, ep->ws_l, ep->side));
    if (cudaEventRecord(ep->join, ep->side) != cudaSuccess)
      return set_error(MOE_ECUDA, "moe_ep_backward: join record failed");
    forked = true;
  } else {
    MOE_TRY(moe_unsort_rows_bwd(&cl, dy, y_sorted, &ep->topo_l, ep->gates, ep->dy_sorted, ep->dgates, stream));
  }
  // dY rows (already in expert order) to the owners' padded layouts
  MOE_TRY(moe_ep_dispatch_padded(&ep->ex, MOE_EP_RECV_DY, ep->dy_sorted, nullptr, 1, stream));
  MOE_TRY(moe_ep_wait(&ep->ex, MOE_EP_RECV_DY, stream));
  void* dy_g = win_region(ep, MOE_EP_RECV_DY);
  void* x_g = win_region(ep, MOE_EP_RECV_X);
  MOE_TRY(moe_zero_pad_rows(ce, &ep->topo_e, dy_g, stream));
  // b2 SDD^T (+act'), b3 DS^TD, b5 DD^TS, b4 DSD^T; experts without rows get exact zero columns
  MOE_TRY(moe_sdd_deriv(ce, dy_g, w->w2, 1, &ep->topo_e, ep->d.act, id ? nullptr : ep->act_deriv, ep->dh, nullptr,
                        stream));
  // dX rows back to the token owners first (fused: the DSD^T stores them there),
  // so their transfer overlaps the weight-gradient products below (NEXT-1)
  if (ep->fused_combine) {
    MOE_TRY(moe_ep_combine_dest(&ep->ex, MOE_EP_RET_DX, ep->dest_dx, ep->rows_e, stream));
    MOE_TRY(moe_dsd_rows(ce, ep->dh, w->w1, 1, &ep->topo_e, ep->dest_dx, stream));
    MOE_TRY(moe_ep_signal(&ep->ex, MOE_EP_RET_DX, stream));
  } else {
    MOE_TRY(moe_dsd(ce, ep->dh, 0, w->w1, 1, &ep->topo_e, ep->dx_g, stream));
    MOE_TRY(moe_ep_combine_padded(&ep->ex, MOE_EP_RET_DX, ep->dx_g, stream));
  }
  MOE_TRY(moe_dsd(ce, ep->a, 1, dy_g, 0, &ep->topo_e, g->dw2, stream));
  MOE_TRY(moe_dds(ce, x_g, 1, ep->dh, 0, &ep->topo_e, g->dw1, stream));
  // b6 (+ b7's dx += dlogits . Wr^T) once every source's dX rows arrived
  MOE_TRY(moe_ep_wait(&ep->ex, MOE_EP_RET_DX, stream));
  const void* dx_sorted = win_region(ep, MOE_EP_RET_DX);
  if (fused) {
    MOE_TRY(moe_sort_rows_bwd_router(&cl, dx_sorted, &ep->topo_l, ep->dlogits, w->wr, dx, stream));
  } else {
    MOE_TRY(moe_sort_rows_bwd(&cl, dx_sorted, &ep->topo_l, dx, stream));
    MOE_TRY(moe_router_bwd(&cl, x, w->wr, ep->logits, ep->idx, ep->dgates, g->dwr, dx, ep->ws_l, stream));
  }
  if (forked && cudaStreamWaitEvent(s, ep->join, 0) != cudaSuccess)
    return set_error(MOE_ECUDA, "moe_ep_backward: join failed");
  ep->bwd_of = ep->fwd_step;
  return MOE_OK;
}

void* moe_ep_tensor(const moe_ep* ep, int which) {
  if (!ep) return nullptr;
  switch (which) {
    case MOE_EP_T_LOGITS: return ep->logits;
    case MOE_EP_T_EXPERT_IDX: return ep->idx;
    case MOE_EP_T_GATES: return ep->gates;
    case MOE_EP_T_PLAN: return ep->ex.plan;
    case MOE_EP_T_AUX: return reinterpret_cast<char*>(ep->ws_l) + moe_workspace_offset(&ep->cfg_l, 5);
    case MOE_EP_T_X_G: return win_region(ep, MOE_EP_RECV_X);
    case MOE_EP_T_A: return ep->a;
    case MOE_EP_T_ACT_DERIV: return ep->act_deriv;
    default: return nullptr;
  }
}

moe_status moe_ep_state(const moe_ep* ep, int side, moe_config* cfg, moe_topology_t* topo) {
  MOE_CHECK_ARG(ep && (side == 0 || side == 1), "moe_ep_state: bad arguments");
  if (cfg) {
    *cfg = side == 0 ? ep->cfg_l : ep->cfg_e;
    if (side == 0 && ep->tokens > 0) cfg->tokens = ep->tokens;
  }
  if (topo) *topo = side == 0 ? ep->topo_l : ep->topo_e;
  return MOE_OK;
}

moe_status moe_ep_exchange_desc(const moe_ep* ep, moe_ep_t* out) {
  MOE_CHECK_ARG(ep && out, "moe_ep_exchange_desc: NULL pointer");
  *out = ep->ex;
  return MOE_OK;
}

moe_status moe_ep_destroy(moe_ep* ep) {
  if (!ep) return MOE_OK;
  int prev_device = 0;
  cudaGetDevice(&prev_device);
  cudaSetDevice(ep->device);
  cudaDeviceSynchronize();
  ep_free_all(ep);
  delete ep;
  cudaSetDevice(prev_device);
  return MOE_OK;
}

}  // extern "C"
