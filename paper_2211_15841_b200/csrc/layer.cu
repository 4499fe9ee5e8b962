// layer.cu — the dMoE layer as one stream-ordered sequence of the kernels
// above. Forward follows Fig. 5; backward follows the operation
// list of §5.1. No host synchronisation: data-dependent sizes live
// in saved->topo.sizes on the device.
#include <stdlib.h>

#include "bsgemm.cuh"
#include "common.cuh"
#include "permute.cuh"

using namespace moe;

namespace {
// Side stream (per thread and device) on which moe_backward runs the router's
// dWr while the SDD^T uses the remaining SMs; fork/join by events, so the
// whole backward stays one stream-ordered, graph-capturable call.
struct SideStream {
  int device = -1;
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
thread_local SideStream t_side;

moe_status side_stream(SideStream** out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return set_error(MOE_ECUDA, "cudaGetDevice failed");
  if (t_side.device != dev) {
    if (cudaStreamCreateWithFlags(&t_side.s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&t_side.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&t_side.join, cudaEventDisableTiming) != cudaSuccess)
      return set_error(MOE_ECUDA, "moe_backward: side stream creation failed");
    t_side.device = dev;
  }
  *out = &t_side;
  return MOE_OK;
}

// MOE_BWD_CONCURRENT=1: the backward's independent products run two at a time
// on split SM budgets (SDD^T beside dWr + DS^TD, then DD^TS beside DSD^T):
// experiment knob (the persistent kernels' ramps and tails overlap).
int bwd_concurrent() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MOE_BWD_CONCURRENT");
    v = e ? atoi(e) : 0;
  }
  return v;
}

// SMs given to the router dWr GEMM while the SDD^T runs beside it (MOE_DWR_SMS, 0 = serial).
// MOE_SAVE_PRE=1 (experiment): the forward saves H in the act_deriv buffer and
// the SDD^T evaluates act'(H) itself (the round-1 form before R18).
bool save_pre() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MOE_SAVE_PRE");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

int dwr_side_sms() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MOE_DWR_SMS");
    v = e ? atoi(e) : 8;
  }
  return v;
}
}  // namespace

extern "C" {

moe_status moe_forward(const moe_config* cfg, const moe_weights* w, const void* x, void* y, moe_saved* sv,
                       void* ws, void* stream) {
  reset_launch_count();
  MOE_TRY(moe_check_config(cfg));
  MOE_CHECK_ARG(w && w->wr && w->w1 && w->w2 && x && y && sv && ws, "moe_forward: NULL pointer");
  MOE_CHECK_ARG(sv->logits && sv->expert_idx && sv->gates && sv->x_g && sv->a && sv->y_g,
                "moe_forward: NULL saved tensor");
  const bool id = cfg->act == MOE_ACT_IDENTITY;
  // saved->act_deriv == NULL: the branch-coded activation (R24; an option that
  // saves the act'(H) buffer): only A is saved and the SDD^T decodes act'(H) from it
  const bool coded = !id && !sv->act_deriv;
  // (1) indices, weights = router(x)
  // (2) topology = make_topology(indices)
  //     (one launch with the router where possible: moe_router_topology)
  MOE_TRY(moe_router_topology(cfg, x, w->wr, sv->logits, sv->expert_idx, sv->gates, &sv->topo, ws, stream));
  //     + the auxiliary load-balancing loss into the workspace
  if (cfg->aux_loss_coeff > 0.f) MOE_TRY(moe_load_balance_loss(cfg, sv->logits, sv->expert_idx, ws, stream));
  // (3) x = padded_gather(x, indices)
  // (4) x = sdd(x, w1, topology) [+ act, act' saved]; x = dsd(x, w2)
  if (cfg->unpadded) {  // P:297 partial blocks at the fringe: X_g rows in expert order, no pad rows
    MOE_TRY(moe_sort_rows(cfg, x, &sv->topo, sv->x_g, stream));
    if (coded)
      MOE_TRY(moe_sdd_act_coded(cfg, sv->x_g, w->w1, 0, &sv->topo, cfg->act, nullptr, sv->a, stream));
    else
      MOE_TRY(save_pre() && !id
                  ? moe_sdd(cfg, sv->x_g, w->w1, 0, &sv->topo, cfg->act, nullptr, sv->a, sv->act_deriv, stream)
                  : moe_sdd_deriv(cfg, sv->x_g, w->w1, 0, &sv->topo, cfg->act, nullptr, sv->a,
                                  id ? nullptr : sv->act_deriv, stream));
  } else if (moe_gather_is_fused(cfg) && !coded) {  // the gather happens inside the SDD's loads (tile::gather4)
    MOE_TRY(moe_sdd_gather(cfg, x, w->w1, &sv->topo, cfg->act, sv->a, id ? nullptr : sv->act_deriv, sv->x_g, stream));
  } else {
    MOE_TRY(moe_gather(cfg, x, &sv->topo, sv->x_g, stream));
    if (coded)
      MOE_TRY(moe_sdd_act_coded(cfg, sv->x_g, w->w1, 0, &sv->topo, cfg->act, nullptr, sv->a, stream));
    else
      MOE_TRY(save_pre() && !id
                  ? moe_sdd(cfg, sv->x_g, w->w1, 0, &sv->topo, cfg->act, nullptr, sv->a, sv->act_deriv, stream)
                  : moe_sdd_deriv(cfg, sv->x_g, w->w1, 0, &sv->topo, cfg->act, nullptr, sv->a,
                                  id ? nullptr : sv->act_deriv, stream));
  }
  // (5) x = padded_scatter(x, indices) * weights            P:279-280 (fused into the DSD for top-1)
  MOE_TRY(moe_dsd_scatter(cfg, sv->a, w->w2, &sv->topo, sv->gates, sv->y_g, y, stream));
  return MOE_OK;
}

moe_status moe_backward(const moe_config* cfg, const moe_weights* w, const moe_saved* sv, const void* x,
                        const void* dy, void* dx, moe_grads* g, void* ws, void* stream) {
  reset_launch_count();
  MOE_TRY(moe_check_config(cfg));
  MOE_CHECK_ARG(w && sv && x && dy && dx && g && g->dwr && g->dw1 && g->dw2 && ws, "moe_backward: NULL pointer");
  const bool id = cfg->act == MOE_ACT_IDENTITY;
  const WsLayout L = ws_layout(cfg);
  char* wsb = reinterpret_cast<char*>(ws);
  void* dy_g = wsb + L.dy_g;
  void* dh = wsb + L.dh;
  void* dx_g = wsb + L.dx_g;
  float* dgates = reinterpret_cast<float*>(wsb + L.dgates);
  const moe_topology_t* topo = &sv->topo;
  const bool fused_router = router_on_tensor_cores(cfg);
  __nv_bfloat16* dl16 = reinterpret_cast<__nv_bfloat16*>(wsb + L.dlogits);
  // b1: dY_g = gates * dy (un-permuted rows), dgates = <Y_g, dy>
  //     [+ b7's dlogits = p * (dp - <p,dp>) in the same pass]
  if (cfg->unpadded && fused_router) {  // unpadded rows: the expert-order backward (+ softmax backward)
    MOE_TRY(moe_unsort_rows_bwd_router(cfg, dy, sv->y_g, topo, sv->gates, sv->logits, sv->expert_idx, dy_g, dgates,
                                       dl16, stream));
    MOE_TRY(moe_add_aux_dlogits(cfg, sv->logits, dl16, ws, stream));
  } else if (cfg->unpadded) {
    MOE_TRY(moe_unsort_rows_bwd(cfg, dy, sv->y_g, topo, sv->gates, dy_g, dgates, stream));
  } else if (fused_router) {
    const float* aux_c = cfg->aux_loss_coeff > 0.f ? reinterpret_cast<const float*>(wsb + L.aux) + 1 : nullptr;
    MOE_TRY(scatter_bwd_router_aux(cfg, dy, sv->y_g, topo, sv->gates, sv->logits, sv->expert_idx, dy_g, dgates,
                                   dl16, aux_c, as_stream(stream)));
  } else {
    MOE_TRY(moe_scatter_bwd(cfg, dy, sv->y_g, topo, sv->gates, dy_g, dgates, stream));
  }
  // b7 (dWr = x^T . dlogits) only needs the scatter backward's dlogits: it runs
  // on a side stream on dwr_side_sms() SMs while the SDD^T takes the others.
  const int side_sms = fused_router ? dwr_side_sms() : 0;
  SideStream* side = nullptr;
  if (side_sms > 0) {
    MOE_TRY(side_stream(&side));
    if (cudaEventRecord(side->fork, as_stream(stream)) != cudaSuccess ||
        cudaStreamWaitEvent(side->s, side->fork, 0) != cudaSuccess)
      return set_error(MOE_ECUDA, "moe_backward: fork failed");
    set_gemm_sm_budget(side_sms);
    const moe_status st = moe_router_dwr(cfg, x, dl16, g->dwr, ws, side->s);
    set_gemm_sm_budget(0);
    MOE_TRY(st);
    if (cudaEventRecord(side->join, side->s) != cudaSuccess)
      return set_error(MOE_ECUDA, "moe_backward: join record failed");
    set_gemm_sm_budget(moe_device_sm_count() - side_sms);
  }
  const int conc = side ? bwd_concurrent() : 0;
  const int all = moe_device_sm_count();
  if (conc) {
    // b3 on the side stream after dWr, beside the SDD^T (dY_g is all it needs)
    const int b3 = (int)(all * 0.42) & ~1;
    set_gemm_sm_budget(b3);
    const moe_status st = moe_dsd(cfg, sv->a, 1, dy_g, 0, topo, g->dw2, side->s);
    set_gemm_sm_budget(0);
    MOE_TRY(st);
    if (cudaEventRecord(side->join, side->s) != cudaSuccess)
      return set_error(MOE_ECUDA, "moe_backward: join record failed");
    set_gemm_sm_budget(all - b3 - side_sms);
  }
  // b2: SDD^T: dH = (dY_g . W2^T) * act'(H)                 "second layer data gradient"
  {
    const moe_status st =
        !id && !sv->act_deriv
            ? moe_sdd_act_coded(cfg, dy_g, w->w2, 1, topo, cfg->act, sv->a, dh, stream)  // act'(H) from A (R24)
            : save_pre() && !id
                  ? moe_sdd(cfg, dy_g, w->w2, 1, topo, cfg->act, sv->act_deriv, dh, nullptr, stream)  // act'(H) here
                  : moe_sdd_deriv(cfg, dy_g, w->w2, 1, topo, cfg->act, id ? nullptr : sv->act_deriv, dh, nullptr,
                                  stream);
    set_gemm_sm_budget(0);
    MOE_TRY(st);
  }
  if (conc) {
    // b5 on the side stream (after b3) beside b4 + b6 + b7 on the main stream; both need dH
    if (cudaEventRecord(side->fork, as_stream(stream)) != cudaSuccess ||
        cudaStreamWaitEvent(side->s, side->fork, 0) != cudaSuccess)
      return set_error(MOE_ECUDA, "moe_backward: fork failed");
    const int b5 = (all / 2) & ~1;
    set_gemm_sm_budget(b5);
    const moe_status st = moe_dds(cfg, sv->x_g, 1, dh, 0, topo, g->dw1, side->s);
    set_gemm_sm_budget(0);
    MOE_TRY(st);
    if (cudaEventRecord(side->join, side->s) != cudaSuccess)
      return set_error(MOE_ECUDA, "moe_backward: join record failed");
    set_gemm_sm_budget(all - b5);
    const moe_status st2 = moe_dsd_dx(cfg, dh, w->w1, topo, dl16, w->wr, dx, dx_g, stream);
    set_gemm_sm_budget(0);
    MOE_TRY(st2);
    if (cudaStreamWaitEvent(as_stream(stream), side->join, 0) != cudaSuccess)
      return set_error(MOE_ECUDA, "moe_backward: join failed");
    return MOE_OK;
  }
  // b3: DS^TD: dW2 = A^T . dY_g                              "second layer weight gradient"
  MOE_TRY(moe_dsd(cfg, sv->a, 1, dy_g, 0, topo, g->dw2, stream));
  if (fused_router) {
    // b5: DD^TS: dW1 = X_g^T . dH                            "first layer weight gradient"
    if (moe_gather_is_fused(cfg))
      MOE_TRY(moe_dds_gather(cfg, x, dh, topo, g->dw1, sv->x_g, stream));
    else
      MOE_TRY(moe_dds(cfg, sv->x_g, 1, dh, 0, topo, g->dw1, stream));
    // b7: dWr = x^T . dlogits (unless it already runs on the side stream)
    if (!side) MOE_TRY(moe_router_dwr(cfg, x, dl16, g->dwr, ws, stream));
    // b4 + b6 + b7: dx = sum_j (dH . W1^T)[pos[t*k+j]] + dlogits . Wr^T   "first layer data gradient"
    MOE_TRY(moe_dsd_dx(cfg, dh, w->w1, topo, dl16, w->wr, dx, dx_g, stream));
    if (side && cudaStreamWaitEvent(as_stream(stream), side->join, 0) != cudaSuccess)
      return set_error(MOE_ECUDA, "moe_backward: join failed");
    return MOE_OK;
  }
  // b4: DSD^T: dX_g = dH . W1^T                              "first layer data gradient"
  MOE_TRY(moe_dsd(cfg, dh, 0, w->w1, 1, topo, dx_g, stream));
  // b5: DD^TS: dW1 = X_g^T . dH                              "first layer weight gradient"
  if (moe_gather_is_fused(cfg))
    MOE_TRY(moe_dds_gather(cfg, x, dh, topo, g->dw1, sv->x_g, stream));
  else
    MOE_TRY(moe_dds(cfg, sv->x_g, 1, dh, 0, topo, g->dw1, stream));
  // b6: dx = sum_j dX_g[pos]
  if (cfg->unpadded)
    MOE_TRY(moe_sort_rows_bwd(cfg, dx_g, topo, dx, stream));
  else
    MOE_TRY(moe_gather_bwd(cfg, dx_g, topo, dx, stream));
  // b7: router backward (dWr, dx += dlogits . Wr^T)
  MOE_TRY(moe_router_bwd(cfg, x, w->wr, sv->logits, sv->expert_idx, dgates, g->dwr, dx, ws, stream));
  return MOE_OK;
}

}  // extern "C"
