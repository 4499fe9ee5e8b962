"""Test-only CPU stand-in for the C-ABI binding, built on the oracle, so the
expert-parallel orchestration (paper_2211_15841_b200.ep: split sizes, the
all-to-all exchange, the ordering contract) can run under torch.distributed
gloo with world_size 2 on a machine without GPUs. Never used by the product."""
import types

import numpy as np
import torch

from oracle import moe_oracle as O


def make_config(tokens, hidden, num_experts, top_k, ffn_hidden, block_size=4, act=1):
    return types.SimpleNamespace(tokens=tokens, hidden=hidden, num_experts=num_experts, top_k=top_k,
                                 ffn_hidden=ffn_hidden, block_size=4, act=act)


def _np(t):
    return t.detach().cpu().double().numpy()


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float64))


class Topo:
    def __init__(self, cfg, idx):
        self.k = idx.shape[1] if idx.ndim == 2 else 1
        self.plan = O.make_plan(idx.reshape(-1, self.k), cfg.num_experts, cfg.block_size)
        self.topo = O.make_topology(self.plan, cfg.block_size, cfg.ffn_hidden)
        R = self.plan.pos.size
        self.sorted_pos = np.empty(R, np.int64)
        self.sorted_pos[self.plan.sorted_idx] = np.arange(R)

    def __getitem__(self, name):
        return torch.from_numpy(getattr(self.plan, name).astype(np.int64))


def moe_router(cfg, x, wr):
    L = O.router_logits(_np(x), _np(wr))
    idx, g = O.topk(L, cfg.top_k, bool(getattr(cfg, "renormalize", 0)))
    return _t(L), torch.from_numpy(idx), _t(g)


def moe_topology(cfg, idx):
    i = idx.numpy().reshape(-1, cfg.top_k) if cfg.top_k > 1 or idx.ndim == 2 else idx.numpy().reshape(-1, 1)
    return Topo(cfg, i)


def moe_sort_rows(cfg, x, topo):
    return _t(_np(x)[topo.plan.sorted_idx // cfg.top_k])


def moe_gather(cfg, x, topo):
    return _t(O.padded_gather(_np(x), topo.plan, cfg.top_k))


def moe_sdd(cfg, a, b, trans_b, topo, act=0, act_grad_src=None, want_pre=False, out=None):
    H = O.sdd(_np(a), _np(b), topo.topo, trans_b=bool(trans_b))
    if act_grad_src is not None:
        return _t(H * O.act_grad(act, _np(act_grad_src)))
    A = O.act(act, H)
    return (_t(A), _t(H)) if want_pre else _t(A)


def moe_sdd_deriv(cfg, a, b, trans_b, topo, act=0, deriv_src=None, want_deriv=False, out=None):
    H = O.sdd(_np(a), _np(b), topo.topo, trans_b=bool(trans_b))
    if deriv_src is not None:
        return _t(H * _np(deriv_src))
    A = O.act(act, H)
    return (_t(A), _t(O.act_grad(act, H))) if want_deriv else _t(A)


def moe_dsd_scatter(cfg, s, w2, topo, gates, y_g=None, y=None):
    yg = O.dsd(_np(s), _np(w2), topo.topo)
    g = np.ones((cfg.tokens, cfg.top_k)) if gates is None else _np(gates).reshape(cfg.tokens, cfg.top_k)
    r = _t(O.padded_scatter(yg, topo.plan, g, cfg.tokens, cfg.top_k))
    if y is not None:
        y.copy_(r)
        return _t(yg), y
    return _t(yg), r


def moe_dsd_dx(cfg, dh, w1, topo, dlogits_bf16=None, wr=None, dx=None, dx_g=None):
    dxg = O.dsd(_np(dh), _np(w1), topo.topo, trans_b=True)
    T, k = cfg.tokens, cfg.top_k
    r = np.zeros((T, dxg.shape[1]))
    for t in range(T):
        for j in range(k):
            r[t] += dxg[topo.plan.pos[t * k + j]]
    if dlogits_bf16 is not None:
        r = r + _np(dlogits_bf16) @ _np(wr).T
    if dx is not None:
        dx.copy_(_t(r))
        return dx
    return _t(r)


def moe_dsd(cfg, s, trans_s, b, trans_b, topo, out=None):
    r = _t(O.dsd(_np(s), _np(b), topo.topo, trans_s=bool(trans_s), trans_b=bool(trans_b)))
    if out is not None:
        out.copy_(r)
        return out
    return r


def moe_dds(cfg, a, trans_a, s, trans_s, topo, out=None):
    r = _t(O.dds(_np(a), _np(s), topo.topo, trans_a=bool(trans_a), trans_s=bool(trans_s)))
    if out is not None:
        out.copy_(r)
        return out
    return r


def moe_scatter(cfg, y_g, topo, gates=None, y=None):
    g = np.ones((cfg.tokens, cfg.top_k)) if gates is None else _np(gates)
    r = _t(O.padded_scatter(_np(y_g), topo.plan, g, cfg.tokens, cfg.top_k))
    if y is not None:
        y.copy_(r)
        return y
    return r


def moe_unsort_rows(cfg, y_sorted, topo, gates=None):
    ys = _np(y_sorted)
    k = cfg.top_k
    g = np.ones((cfg.tokens, k)) if gates is None else _np(gates)
    y = np.zeros((cfg.tokens, ys.shape[1]))
    for t in range(cfg.tokens):
        for j in range(k):
            y[t] += g[t, j] * ys[topo.sorted_pos[t * k + j]]
    return _t(y)


def moe_unsort_rows_bwd(cfg, dy, y_sorted, topo, gates=None):
    ys, d = _np(y_sorted), _np(dy)
    k = cfg.top_k
    g = np.ones((cfg.tokens, k)) if gates is None else _np(gates)
    dys = np.zeros_like(ys)
    dg = np.zeros((cfg.tokens, k))
    for t in range(cfg.tokens):
        for j in range(k):
            u = topo.sorted_pos[t * k + j]
            dys[u] = g[t, j] * d[t]
            dg[t, j] = ys[u] @ d[t]
    return _t(dys), _t(dg)


def moe_gather_bwd(cfg, dx_g, topo, dx=None):
    dg = _np(dx_g)
    k = cfg.top_k
    r = np.zeros((cfg.tokens, dg.shape[1]))
    for i in range(cfg.tokens * k):
        r[i // k] += dg[topo.plan.pos[i]]
    if dx is not None:
        dx.copy_(_t(r))
        return dx
    return _t(r)


def moe_sort_rows_bwd(cfg, dx_sorted, topo):
    return moe_unsort_rows(cfg, dx_sorted, topo, None)


def moe_router_bwd(cfg, x, wr, logits, expert_idx, dgates, dx, ws=None):
    L, idx, dg = _np(logits), expert_idx.numpy(), _np(dgates)
    p = O.softmax(L)
    dp = np.zeros_like(p)
    for t in range(L.shape[0]):
        for j in range(cfg.top_k):
            dp[t, idx[t, j]] += dg[t, j]
    dl = p * (dp - (p * dp).sum(1, keepdims=True))
    dx += _t(dl @ _np(wr).T)
    return _t(_np(x).T @ dl)


# ---- fused tensor-core router forms (same arithmetic, unpadded expert order)

def router_on_tensor_cores(cfg):
    return True


def _dlogits(cfg, logits, expert_idx, dgates):
    L, idx, dg = _np(logits), expert_idx.numpy(), _np(dgates)
    p = O.softmax(L)
    dp = np.zeros_like(p)
    renorm = bool(getattr(cfg, "renormalize", 0))
    for t in range(L.shape[0]):
        S = sum(p[t, idx[t, i]] for i in range(cfg.top_k))
        gd = sum(dg[t, i] * p[t, idx[t, i]] / S for i in range(cfg.top_k))
        for j in range(cfg.top_k):
            dp[t, idx[t, j]] += (dg[t, j] - gd) / S if renorm else dg[t, j]
    return p * (dp - (p * dp).sum(1, keepdims=True))


def moe_unsort_rows_bwd_router(cfg, dy, y_sorted, topo, gates, logits, expert_idx):
    dys, dg = moe_unsort_rows_bwd(cfg, dy, y_sorted, topo, gates)
    return dys, dg, _t(_dlogits(cfg, logits, expert_idx, dg))


def moe_router_dwr(cfg, x, dlogits, ws=None):
    return _t(_np(x).T @ _np(dlogits))


def moe_sort_rows_bwd_router(cfg, dx_sorted, topo, dlogits, wr):
    return _t(_np(moe_sort_rows_bwd(cfg, dx_sorted, topo)) + _np(dlogits) @ _np(wr).T)


def moe_ep_recv_ids(counts_all, e0, local_experts, n_rows):
    c = counts_all.numpy()
    ids = np.concatenate([np.repeat(np.arange(local_experts), c[q, e0:e0 + local_experts]) for q in range(c.shape[0])])
    assert ids.size == n_rows
    return torch.from_numpy(ids.astype(np.int32))


# ---- auxiliary load-balancing loss (per rank's tokens; ws is a dict here)

def workspace(cfg, device=None):
    return {}


def moe_load_balance_loss(cfg, logits, expert_idx, ws=None):
    ws = ws if ws is not None else {}
    p = O.softmax(_np(logits))
    loss, dprobs = O.load_balance_loss(p, expert_idx.numpy(), cfg.aux_loss_coeff)
    ws["aux_c"] = dprobs[0] * 1.0      # the per-expert coefficient (same for every token)
    return torch.tensor([loss], dtype=torch.float64), ws


def moe_add_aux_dlogits(cfg, logits, dlogits, ws):
    p = O.softmax(_np(logits))
    c = ws["aux_c"][None, :]
    add = p * (c - (p * c).sum(1, keepdims=True))
    dlogits.copy_(_t(_np(dlogits) + add))
    return dlogits
