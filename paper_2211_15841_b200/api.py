"""Thin Python binding of the C ABI (include/moe.h), same names as the C entry
points. Argument marshalling only: torch supplies device memory and the
current CUDA stream; every step runs in libmoe.so kernels.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from ._lib import (MoeConfig, MoeGrads, MoeSaved, MoeTopology, MoeWeights, TOPO_FIELDS, check, lib)

ACT_IDENTITY, ACT_GELU, ACT_RELU = 0, 1, 2


def make_config(tokens, hidden, num_experts, top_k, ffn_hidden, block_size=128, act=ACT_GELU,
                capacity=0, renormalize=False, aux_loss_coeff=0.0, unpadded=False) -> MoeConfig:
    """capacity = 0: dropless (the method). > 0: the token-dropping formulation
    with that many assignments kept per expert (moe_expert_capacity).
    renormalize: divide each token's k gates by their sum. aux_loss_coeff > 0:
    auxiliary load-balancing loss (moe_load_balance_loss)."""
    return MoeConfig(int(tokens), int(hidden), int(num_experts), int(top_k), int(ffn_hidden), int(block_size),
                     int(act), int(capacity), int(bool(renormalize)), float(aux_loss_coeff), int(bool(unpadded)))


def aux_region(cfg, ws) -> torch.Tensor:
    """float [1 + E] view of the workspace's auxiliary-loss region: {loss, coeff*E*f_e/T}."""
    off = int(lib.moe_workspace_offset(ctypes.byref(cfg), 5))
    return ws[off: off + 4 * (1 + cfg.num_experts)].view(torch.float32)


def moe_add_aux_dlogits(cfg, logits, dlogits, ws):
    """moe_add_aux_dlogits (include/moe.h): dlogits += the auxiliary loss's gradient, in place."""
    check("moe_add_aux_dlogits", lib.moe_add_aux_dlogits(ctypes.byref(cfg), _p(logits), _p(dlogits), _p(ws),
                                                         _stream()))
    return dlogits


def moe_load_balance_loss(cfg, logits, expert_idx, ws=None):
    """moe_load_balance_loss (include/moe.h): returns (loss [1] tensor view, the workspace)."""
    ws = ws if ws is not None else workspace(cfg, logits.device)
    check("moe_load_balance_loss", lib.moe_load_balance_loss(ctypes.byref(cfg), _p(logits), _p(expert_idx), _p(ws),
                                                             _stream()))
    return aux_region(cfg, ws)[:1], ws


def moe_expert_capacity(tokens, num_experts, capacity_factor) -> int:
    """ceil(tokens * capacity_factor / num_experts) (§2.2)."""
    return int(lib.moe_expert_capacity(int(tokens), int(num_experts), float(capacity_factor)))


def cfg_replace(cfg: MoeConfig, **kw) -> MoeConfig:
    d = {n: getattr(cfg, n) for n, _ in MoeConfig._fields_}
    d.update(kw)
    return MoeConfig(**d)


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def moe_check_config(cfg):
    return lib.moe_check_config(ctypes.byref(cfg))


def moe_max_padded_rows(cfg) -> int:
    return int(lib.moe_max_padded_rows(ctypes.byref(cfg)))


def moe_max_nnz_blocks(cfg) -> int:
    return int(lib.moe_max_nnz_blocks(ctypes.byref(cfg)))


def moe_workspace_bytes(cfg) -> int:
    return int(lib.moe_workspace_bytes(ctypes.byref(cfg)))


def workspace(cfg, device="cuda") -> torch.Tensor:
    return torch.empty(max(moe_workspace_bytes(cfg), 256), dtype=torch.uint8, device=device)


class Topology:
    """Device buffers of moe_topology_t, sized to the worst case."""

    def __init__(self, cfg, device="cuda"):
        E, bs = cfg.num_experts, cfg.block_size
        R = cfg.tokens * cfg.top_k
        rows, nnz = moe_max_padded_rows(cfg), moe_max_nnz_blocks(cfg)
        F = cfg.ffn_hidden // bs
        shapes = {"counts": E, "bins": E, "padded_bins": E, "sorted_idx": R, "pos": R, "sorted_pos": R,
                  "row_offsets": rows // bs + 1, "col_indices": nnz, "row_indices": nnz,
                  "t_col_offsets": E * F + 1, "t_block_offsets": nnz, "t_row_indices": nnz, "pair_bins": E,
                  "row_src": rows, "sizes": 3, "brow_start": rows // bs, "brow_rows": rows // bs}
        # one allocation, 16-byte aligned views (TMA / int4 loads read row_src)
        sizes = [((max(int(shapes[n]), 1) + 3) // 4) * 4 for n in TOPO_FIELDS]
        self.buf = torch.empty(sum(sizes), dtype=torch.int32, device=device)
        self.t, o = {}, 0
        for n, sz in zip(TOPO_FIELDS, sizes):
            self.t[n] = self.buf[o:o + max(int(shapes[n]), 1)]
            o += sz
        self.struct = MoeTopology(*[self.t[n].data_ptr() for n in TOPO_FIELDS])

    def __getitem__(self, name):
        return self.t[name]

    def sizes(self):
        """(Tp, nnz) — reads back from the device (tests / host orchestration only)."""
        s = self.t["sizes"].cpu()
        return int(s[0]), int(s[1])


def moe_topk(cfg, logits, expert_idx=None, gates=None):
    T, k = cfg.tokens, cfg.top_k
    expert_idx = expert_idx if expert_idx is not None else torch.empty(T, k, dtype=torch.int32, device=logits.device)
    gates = gates if gates is not None else torch.empty(T, k, dtype=torch.float32, device=logits.device)
    check("moe_topk", lib.moe_topk(ctypes.byref(cfg), _p(logits), _p(expert_idx), _p(gates), _stream()))
    return expert_idx, gates


def moe_router(cfg, x, wr, ws=None):
    T, E, k = cfg.tokens, cfg.num_experts, cfg.top_k
    dev = x.device
    logits = torch.empty(T, E, dtype=torch.float32, device=dev)
    idx = torch.empty(T, k, dtype=torch.int32, device=dev)
    gates = torch.empty(T, k, dtype=torch.float32, device=dev)
    ws = ws if ws is not None else workspace(cfg, dev)
    check("moe_router", lib.moe_router(ctypes.byref(cfg), _p(x), _p(wr), _p(logits), _p(idx), _p(gates), _p(ws),
                                       _stream()))
    return logits, idx, gates


def moe_topology(cfg, expert_idx, topo: Topology | None = None, ws=None) -> Topology:
    topo = topo if topo is not None else Topology(cfg, expert_idx.device)
    ws = ws if ws is not None else workspace(cfg, expert_idx.device)
    check("moe_topology", lib.moe_topology(ctypes.byref(cfg), _p(expert_idx), ctypes.byref(topo.struct), _p(ws),
                                           _stream()))
    return topo


def moe_router_topology(cfg, x, wr, ws=None, topo: Topology | None = None):
    """moe_router_topology (include/moe.h): router, top-k and topology, one
    launch where possible. Returns (logits, expert_idx, gates, topology)."""
    T, E, k = cfg.tokens, cfg.num_experts, cfg.top_k
    dev = x.device
    logits = torch.empty(T, E, dtype=torch.float32, device=dev)
    idx = torch.empty(T, k, dtype=torch.int32, device=dev)
    gates = torch.empty(T, k, dtype=torch.float32, device=dev)
    ws = ws if ws is not None else workspace(cfg, dev)
    topo = topo if topo is not None else Topology(cfg, dev)
    check("moe_router_topology", lib.moe_router_topology(ctypes.byref(cfg), _p(x), _p(wr), _p(logits), _p(idx),
                                                         _p(gates), ctypes.byref(topo.struct), _p(ws), _stream()))
    return logits, idx, gates, topo


def moe_topology_from_router(cfg, expert_idx, ws, topo: Topology | None = None) -> Topology:
    """moe_topology_from_router (include/moe.h): the topology from the per-tile
    histograms moe_router(cfg, ..., ws) left in ws (tensor-core router), else moe_topology."""
    topo = topo if topo is not None else Topology(cfg, expert_idx.device)
    check("moe_topology_from_router", lib.moe_topology_from_router(ctypes.byref(cfg), _p(expert_idx),
                                                                   ctypes.byref(topo.struct), _p(ws), _stream()))
    return topo


def moe_topology_counts(cfg, counts_per_source, topo: Topology | None = None) -> Topology:
    """moe_topology_counts (include/moe.h): topology of rows grouped by expert
    then source, from the [nsources, E] int32 device counts."""
    topo = topo if topo is not None else Topology(cfg, counts_per_source.device)
    check("moe_topology_counts", lib.moe_topology_counts(ctypes.byref(cfg), _p(counts_per_source),
                                                         int(counts_per_source.shape[0]), ctypes.byref(topo.struct),
                                                         _stream()))
    return topo


def moe_zero_pad_rows(cfg, topo: Topology, x_g):
    check("moe_zero_pad_rows", lib.moe_zero_pad_rows(ctypes.byref(cfg), ctypes.byref(topo.struct), _p(x_g), _stream()))
    return x_g


def moe_gather(cfg, x, topo: Topology, x_g=None):
    x_g = x_g if x_g is not None else torch.empty(moe_max_padded_rows(cfg), cfg.hidden, dtype=x.dtype,
                                                  device=x.device)
    check("moe_gather", lib.moe_gather(ctypes.byref(cfg), _p(x), ctypes.byref(topo.struct), _p(x_g), _stream()))
    return x_g


def moe_scatter(cfg, y_g, topo: Topology, gates=None, y=None):
    y = y if y is not None else torch.empty(cfg.tokens, cfg.hidden, dtype=y_g.dtype, device=y_g.device)
    check("moe_scatter", lib.moe_scatter(ctypes.byref(cfg), _p(y_g), ctypes.byref(topo.struct), _p(gates), _p(y),
                                         _stream()))
    return y


def moe_scatter_bwd(cfg, dy, y_g, topo: Topology, gates=None, want_dgates=True):
    dy_g = torch.empty(moe_max_padded_rows(cfg), cfg.hidden, dtype=dy.dtype, device=dy.device)
    dg = torch.empty(cfg.tokens, cfg.top_k, dtype=torch.float32, device=dy.device) if want_dgates else None
    check("moe_scatter_bwd", lib.moe_scatter_bwd(ctypes.byref(cfg), _p(dy), _p(y_g), ctypes.byref(topo.struct),
                                                 _p(gates), _p(dy_g), _p(dg), _stream()))
    return dy_g, dg


def moe_gather_bwd(cfg, dx_g, topo: Topology, dx=None):
    dx = dx if dx is not None else torch.empty(cfg.tokens, cfg.hidden, dtype=dx_g.dtype, device=dx_g.device)
    check("moe_gather_bwd", lib.moe_gather_bwd(ctypes.byref(cfg), _p(dx_g), ctypes.byref(topo.struct), _p(dx),
                                               _stream()))
    return dx


def moe_sort_rows(cfg, x, topo: Topology, out=None):
    out = out if out is not None else torch.empty(cfg.tokens * cfg.top_k, cfg.hidden, dtype=x.dtype, device=x.device)
    check("moe_sort_rows", lib.moe_sort_rows(ctypes.byref(cfg), _p(x), ctypes.byref(topo.struct), _p(out),
                                             _stream()))
    return out


def moe_unsort_rows(cfg, y_sorted, topo: Topology, gates=None, y=None):
    y = y if y is not None else torch.empty(cfg.tokens, cfg.hidden, dtype=y_sorted.dtype, device=y_sorted.device)
    check("moe_unsort_rows", lib.moe_unsort_rows(ctypes.byref(cfg), _p(y_sorted), ctypes.byref(topo.struct),
                                                 _p(gates), _p(y), _stream()))
    return y


def moe_unsort_rows_bwd(cfg, dy, y_sorted, topo: Topology, gates=None, want_dgates=True):
    dys = torch.empty(cfg.tokens * cfg.top_k, cfg.hidden, dtype=dy.dtype, device=dy.device)
    dg = torch.empty(cfg.tokens, cfg.top_k, dtype=torch.float32, device=dy.device) if want_dgates else None
    check("moe_unsort_rows_bwd", lib.moe_unsort_rows_bwd(ctypes.byref(cfg), _p(dy), _p(y_sorted),
                                                         ctypes.byref(topo.struct), _p(gates), _p(dys), _p(dg),
                                                         _stream()))
    return dys, dg


def moe_sort_rows_bwd(cfg, dx_sorted, topo: Topology, dx=None):
    dx = dx if dx is not None else torch.empty(cfg.tokens, cfg.hidden, dtype=dx_sorted.dtype, device=dx_sorted.device)
    check("moe_sort_rows_bwd", lib.moe_sort_rows_bwd(ctypes.byref(cfg), _p(dx_sorted), ctypes.byref(topo.struct),
                                                     _p(dx), _stream()))
    return dx


def router_on_tensor_cores(cfg) -> bool:
    """The fused tensor-core router path's condition (include/moe.h)."""
    return cfg.num_experts % 64 == 0 and cfg.num_experts <= 256 and cfg.top_k <= 8


def moe_unsort_rows_bwd_router(cfg, dy, y_sorted, topo: Topology, gates, logits, expert_idx, dy_sorted=None,
                               dgates=None, dlogits=None):
    """moe_unsort_rows_bwd_router (include/moe.h): dy_sorted, dgates and the bf16 dlogits [T,E]."""
    T, k = cfg.tokens, cfg.top_k
    dy_sorted = dy_sorted if dy_sorted is not None else torch.empty(T * k, cfg.hidden, dtype=dy.dtype, device=dy.device)
    dgates = dgates if dgates is not None else torch.empty(T, k, dtype=torch.float32, device=dy.device)
    dlogits = dlogits if dlogits is not None else torch.empty(T, cfg.num_experts, dtype=torch.bfloat16,
                                                              device=dy.device)
    check("moe_unsort_rows_bwd_router", lib.moe_unsort_rows_bwd_router(
        ctypes.byref(cfg), _p(dy), _p(y_sorted), ctypes.byref(topo.struct), _p(gates), _p(logits), _p(expert_idx),
        _p(dy_sorted), _p(dgates), _p(dlogits), _stream()))
    return dy_sorted, dgates, dlogits


def moe_sort_rows_bwd_router(cfg, dx_sorted, topo: Topology, dlogits, wr, dx=None):
    """moe_sort_rows_bwd_router (include/moe.h): dx = sum_j dx_sorted[sorted_pos] + dlogits . wr^T."""
    dx = dx if dx is not None else torch.empty(cfg.tokens, cfg.hidden, dtype=dx_sorted.dtype, device=dx_sorted.device)
    check("moe_sort_rows_bwd_router", lib.moe_sort_rows_bwd_router(
        ctypes.byref(cfg), _p(dx_sorted), ctypes.byref(topo.struct), _p(dlogits), _p(wr), _p(dx), _stream()))
    return dx


def moe_router_dwr(cfg, x, dlogits, dwr=None, ws=None):
    """moe_router_dwr (include/moe.h): dWr [h,E] fp32 = x^T . dlogits (tcgen05)."""
    dwr = dwr if dwr is not None else torch.empty(cfg.hidden, cfg.num_experts, dtype=torch.float32, device=x.device)
    ws = ws if ws is not None else workspace(cfg, x.device)
    check("moe_router_dwr", lib.moe_router_dwr(ctypes.byref(cfg), _p(x), _p(dlogits), _p(dwr), _p(ws), _stream()))
    return dwr


def moe_ep_recv_ids(counts_all, rank_e0, local_experts, n_rows, ids=None):
    """moe_ep_recv_ids (include/moe.h): local expert id of every received row, in
    arrival order (source, local expert, token), from the [P, E] int32 counts."""
    P, E = counts_all.shape
    ids = ids if ids is not None else torch.empty(max(int(n_rows), 1), dtype=torch.int32, device=counts_all.device)
    check("moe_ep_recv_ids", lib.moe_ep_recv_ids(_p(counts_all), int(P), int(E), int(rank_e0), int(local_experts),
                                                 _p(ids), int(n_rows), _stream()))
    return ids


def _nnz_values(cfg, device, dtype=torch.bfloat16):
    bs = cfg.block_size
    return torch.empty(moe_max_nnz_blocks(cfg), bs, bs, dtype=dtype, device=device)


def moe_sdd(cfg, a, b, trans_b, topo: Topology, act=ACT_IDENTITY, act_grad_src=None, want_pre=False, out=None):
    out = out if out is not None else _nnz_values(cfg, a.device)
    pre = _nnz_values(cfg, a.device) if want_pre else None
    check("moe_sdd", lib.moe_sdd(ctypes.byref(cfg), _p(a), _p(b), int(trans_b), ctypes.byref(topo.struct), int(act),
                                 _p(act_grad_src), _p(out), _p(pre), _stream()))
    return (out, pre) if want_pre else out


def moe_sdd_deriv(cfg, a, b, trans_b, topo: Topology, act=ACT_IDENTITY, deriv_src=None, want_deriv=False, out=None):
    """moe_sdd_deriv (include/moe.h): forward returns act(A.B) [and act'(A.B)];
    with deriv_src (the saved act'(H)) returns (A.B) * deriv_src (SDD^T)."""
    out = out if out is not None else _nnz_values(cfg, a.device)
    der = _nnz_values(cfg, a.device) if want_deriv else None
    check("moe_sdd_deriv", lib.moe_sdd_deriv(ctypes.byref(cfg), _p(a), _p(b), int(trans_b), ctypes.byref(topo.struct),
                                             int(act), _p(deriv_src), _p(out), _p(der), _stream()))
    return (out, der) if want_deriv else out


def moe_sdd_act_coded(cfg, a, b, trans_b, topo: Topology, act=ACT_IDENTITY, coded_src=None, out=None):
    """moe_sdd_act_coded (include/moe.h, reading R24): forward (coded_src None)
    returns the branch-coded act(A.B); with coded_src (the forward's output)
    returns (A.B) * act'(H) decoded from it (SDD^T)."""
    out = out if out is not None else _nnz_values(cfg, a.device)
    check("moe_sdd_act_coded", lib.moe_sdd_act_coded(ctypes.byref(cfg), _p(a), _p(b), int(trans_b),
                                                     ctypes.byref(topo.struct), int(act), _p(coded_src), _p(out),
                                                     _stream()))
    return out


def moe_act_code_decode_host(act, a_bits):
    """moe_act_code_decode_host (host only): act'(H) decoded from coded bf16 bit
    patterns (a numpy uint16 array) -> numpy float32."""
    import numpy as np
    a_bits = np.ascontiguousarray(a_bits, dtype=np.uint16)
    out = np.empty(a_bits.shape, dtype=np.float32)
    check("moe_act_code_decode_host", lib.moe_act_code_decode_host(int(act), a_bits.ctypes.data, out.ctypes.data,
                                                                   a_bits.size))
    return out


def moe_dsd(cfg, s, trans_s, b, trans_b, topo: Topology, out=None):
    rows = moe_max_padded_rows(cfg)
    n_out = cfg.num_experts * cfg.ffn_hidden if trans_s else rows
    out = out if out is not None else torch.empty(n_out, cfg.hidden, dtype=torch.bfloat16, device=s.device)
    check("moe_dsd", lib.moe_dsd(ctypes.byref(cfg), _p(s), int(trans_s), _p(b), int(trans_b),
                                 ctypes.byref(topo.struct), _p(out), _stream()))
    return out


def moe_dsd_rows(cfg, s, b, trans_b, topo: Topology, row_dst):
    """moe_dsd_rows (include/moe.h): DSD / DSD^T with output row p stored to the
    device address row_dst[p] (int64 tensor on the device; 0: not stored)."""
    check("moe_dsd_rows", lib.moe_dsd_rows(ctypes.byref(cfg), _p(s), _p(b), int(trans_b), ctypes.byref(topo.struct),
                                           _p(row_dst), _stream()))


def moe_gather_is_fused(cfg) -> bool:
    return bool(lib.moe_gather_is_fused(ctypes.byref(cfg)))


def moe_sdd_gather(cfg, x, w1, topo: Topology, act=ACT_IDENTITY, want_deriv=False, out=None, x_g=None):
    """moe_sdd_gather (include/moe.h): act(X_g . W1) [and act'] with X_g gathered from x inside the product."""
    out = out if out is not None else _nnz_values(cfg, x.device)
    der = _nnz_values(cfg, x.device) if want_deriv else None
    if x_g is None:   # scratch for configs the kernels cannot gather in
        x_g = torch.empty(moe_max_padded_rows(cfg), cfg.hidden, dtype=torch.bfloat16, device=x.device)
    check("moe_sdd_gather", lib.moe_sdd_gather(ctypes.byref(cfg), _p(x), _p(w1), ctypes.byref(topo.struct), int(act),
                                               _p(out), _p(der), _p(x_g), _stream()))
    return (out, der) if want_deriv else out


def moe_dds_gather(cfg, x, dh, topo: Topology, dw1=None, x_g=None):
    """moe_dds_gather (include/moe.h): dW1 = X_g^T . dH with X_g gathered from x inside the product."""
    dw1 = dw1 if dw1 is not None else torch.empty(cfg.hidden, cfg.num_experts * cfg.ffn_hidden, dtype=torch.bfloat16,
                                                  device=x.device)
    if x_g is None:
        x_g = torch.empty(moe_max_padded_rows(cfg), cfg.hidden, dtype=torch.bfloat16, device=x.device)
    check("moe_dds_gather", lib.moe_dds_gather(ctypes.byref(cfg), _p(x), _p(dh), ctypes.byref(topo.struct), _p(dw1),
                                               _p(x_g), _stream()))
    return dw1


def moe_dsd_scatter(cfg, s, w2, topo: Topology, gates, y_g=None, y=None):
    """moe_dsd_scatter (include/moe.h): Y_g = S . W2 and y = weighted un-permutation of Y_g."""
    rows = moe_max_padded_rows(cfg)
    y_g = y_g if y_g is not None else torch.empty(rows, cfg.hidden, dtype=torch.bfloat16, device=s.device)
    y = y if y is not None else torch.empty(cfg.tokens, cfg.hidden, dtype=torch.bfloat16, device=s.device)
    check("moe_dsd_scatter", lib.moe_dsd_scatter(ctypes.byref(cfg), _p(s), _p(w2), ctypes.byref(topo.struct),
                                                 _p(gates), _p(y_g), _p(y), _stream()))
    return y_g, y


def moe_dsd_dx(cfg, dh, w1, topo: Topology, dlogits_bf16=None, wr=None, dx=None, dx_g=None):
    """moe_dsd_dx (include/moe.h): dx = sum_j (dH . W1^T)[pos] (+ dlogits . Wr^T)."""
    dx = dx if dx is not None else torch.empty(cfg.tokens, cfg.hidden, dtype=torch.bfloat16, device=dh.device)
    if dx_g is None and (cfg.top_k > 1 or dlogits_bf16 is None):
        dx_g = torch.empty(moe_max_padded_rows(cfg), cfg.hidden, dtype=torch.bfloat16, device=dh.device)
    check("moe_dsd_dx", lib.moe_dsd_dx(ctypes.byref(cfg), _p(dh), _p(w1), ctypes.byref(topo.struct), _p(dlogits_bf16),
                                       _p(wr), _p(dx), _p(dx_g), _stream()))
    return dx


def moe_dds(cfg, a, trans_a, s, trans_s, topo: Topology, out=None):
    rows = moe_max_padded_rows(cfg)
    n_out = rows if trans_s else cfg.num_experts * cfg.ffn_hidden
    out = out if out is not None else torch.empty(cfg.hidden, n_out, dtype=torch.bfloat16, device=s.device)
    check("moe_dds", lib.moe_dds(ctypes.byref(cfg), _p(a), int(trans_a), _p(s), int(trans_s),
                                 ctypes.byref(topo.struct), _p(out), _stream()))
    return out


def moe_router_bwd(cfg, x, wr, logits, expert_idx, dgates, dx, ws=None):
    dwr = torch.empty(cfg.hidden, cfg.num_experts, dtype=torch.float32, device=x.device)
    ws = ws if ws is not None else workspace(cfg, x.device)
    check("moe_router_bwd", lib.moe_router_bwd(ctypes.byref(cfg), _p(x), _p(wr), _p(logits), _p(expert_idx),
                                               _p(dgates), _p(dwr), _p(dx), _p(ws), _stream()))
    return dwr


@dataclass
class Saved:
    logits: torch.Tensor
    expert_idx: torch.Tensor
    gates: torch.Tensor
    topo: Topology
    x_g: torch.Tensor
    act_deriv: torch.Tensor | None
    a: torch.Tensor
    y_g: torch.Tensor
    struct: MoeSaved = None
    ws: torch.Tensor | None = None   # the forward's workspace when it holds the auxiliary loss (aux_loss_coeff > 0)

    @staticmethod
    def allocate(cfg, device="cuda", save_deriv: bool = True) -> "Saved":
        """save_deriv=True (default): act'(H) is saved beside A (R18);
        False: act_deriv is None and the forward saves only the branch-coded A
        (R24: one [nnz, bs, bs] buffer less, measured slower at MoE-XS)."""
        T, E, k, h = cfg.tokens, cfg.num_experts, cfg.top_k, cfg.hidden
        rows = moe_max_padded_rows(cfg)
        s = Saved(torch.empty(T, E, dtype=torch.float32, device=device),
                  torch.empty(T, k, dtype=torch.int32, device=device),
                  torch.empty(T, k, dtype=torch.float32, device=device),
                  Topology(cfg, device),
                  torch.empty(rows, h, dtype=torch.bfloat16, device=device),
                  _nnz_values(cfg, device) if save_deriv and cfg.act != ACT_IDENTITY else None,
                  _nnz_values(cfg, device),
                  torch.empty(rows, h, dtype=torch.bfloat16, device=device))
        s.struct = MoeSaved(s.logits.data_ptr(), s.expert_idx.data_ptr(), s.gates.data_ptr(), s.topo.struct,
                            s.x_g.data_ptr(), None if s.act_deriv is None else s.act_deriv.data_ptr(), s.a.data_ptr(),
                            s.y_g.data_ptr())
        return s


def weights_struct(wr, w1, w2) -> MoeWeights:
    return MoeWeights(wr.data_ptr(), w1.data_ptr(), w2.data_ptr())


def moe_forward(cfg, wr, w1, w2, x, y=None, saved: Saved | None = None, ws=None):
    y = y if y is not None else torch.empty(cfg.tokens, cfg.hidden, dtype=torch.bfloat16, device=x.device)
    saved = saved if saved is not None else Saved.allocate(cfg, x.device)
    ws = ws if ws is not None else workspace(cfg, x.device)
    w = weights_struct(wr, w1, w2)
    check("moe_forward", lib.moe_forward(ctypes.byref(cfg), ctypes.byref(w), _p(x), _p(y), ctypes.byref(saved.struct),
                                         _p(ws), _stream()))
    if cfg.aux_loss_coeff > 0:
        saved.ws = ws   # its aux region (loss, gradient coefficients) is read by moe_backward
    return y, saved


def moe_backward(cfg, wr, w1, w2, saved: Saved, x, dy, dx=None, grads=None, ws=None):
    dev = x.device
    dx = dx if dx is not None else torch.empty(cfg.tokens, cfg.hidden, dtype=torch.bfloat16, device=dev)
    if grads is None:
        grads = (torch.empty(cfg.hidden, cfg.num_experts, dtype=torch.float32, device=dev),
                 torch.empty(cfg.hidden, cfg.num_experts * cfg.ffn_hidden, dtype=torch.bfloat16, device=dev),
                 torch.empty(cfg.num_experts * cfg.ffn_hidden, cfg.hidden, dtype=torch.bfloat16, device=dev))
    if ws is None:
        ws = saved.ws if saved.ws is not None else workspace(cfg, dev)
    w = weights_struct(wr, w1, w2)
    g = MoeGrads(grads[0].data_ptr(), grads[1].data_ptr(), grads[2].data_ptr())
    check("moe_backward", lib.moe_backward(ctypes.byref(cfg), ctypes.byref(w), ctypes.byref(saved.struct), _p(x),
                                           _p(dy), _p(dx), ctypes.byref(g), _p(ws), _stream()))
    return dx, grads


def moe_last_launch_count() -> int:
    return int(lib.moe_last_launch_count())
