"""Expert parallelism for the dropless-MoE layer ("distributed training
of MoEs with both data and expert model parallelism"; "8-way expert
model parallelism for MoE layers and data parallelism for all other layers").

Rank r of P owns the contiguous experts [r*E/P, (r+1)*E/P) and their W1 / W2
slices; the router weights are replicated (data parallel). One process per
GPU; the token exchange is torch.distributed all_to_all_single over NCCL
(NVLink 5 / NVSwitch). Every compute step runs in libmoe.so kernels through
the binding (`backend`); this module is plumbing: split sizes, the exchange
and the ordering contract.

Ordering contract: the sender lists its assignments in
(global expert, flat id) order (moe_sort_rows over the local topology), so the
chunk for rank q is contiguous. The receiver gets rows ordered
(source rank, local expert, token); moe_topology's stable grouping by local
expert then yields (local expert, source rank, token) = ascending global token
id within each expert, i.e. each rank's expert topology is exactly the
single-device topology of the global batch restricted to its experts.

The host needs the per-rank counts to size the all-to-all (one small
all_gather + device->host copy per forward); the single-GPU path has no host
synchronisation at all.
"""
from __future__ import annotations

import sys
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


# ----------------------------------------------------------------------------- host logic (pure)

def local_expert_range(rank: int, world: int, num_experts: int):
    if num_experts % world:
        raise ValueError(f"num_experts={num_experts} not divisible by world size {world}")
    el = num_experts // world
    return rank * el, (rank + 1) * el


def send_splits(counts_row: np.ndarray, world: int) -> list[int]:
    """Rows this rank sends to each destination: its assignments to the
    destination's experts (counts_row = this rank's per-global-expert counts)."""
    E = counts_row.size
    el = E // world
    return [int(counts_row[q * el:(q + 1) * el].sum()) for q in range(world)]


def recv_plan(counts_all: np.ndarray, rank: int, world: int):
    """counts_all [P, E]: assignments of source rank q to global expert e.
    Returns (recv_splits per source, local expert id of every received row in
    arrival order (source, local expert, token))."""
    P, E = counts_all.shape
    e0, e1 = local_expert_range(rank, world, E)
    splits = [int(counts_all[q, e0:e1].sum()) for q in range(P)]
    ids = [np.repeat(np.arange(e1 - e0, dtype=np.int32), counts_all[q, e0:e1]) for q in range(P)]
    return splits, (np.concatenate(ids) if ids else np.zeros(0, np.int32))


# ----------------------------------------------------------------------------- layer

@dataclass
class EPState:
    cfg_local: object
    cfg_e: object
    logits: torch.Tensor
    expert_idx: torch.Tensor
    gates: torch.Tensor
    topo_local: object
    topo_e: object
    sends: list
    recvs: list
    x_g: torch.Tensor | None
    act_deriv: torch.Tensor | None
    a: torch.Tensor | None
    y_sorted: torch.Tensor
    n_recv: int
    step: int = 0     # which forward produced this state (one forward in flight per layer)


class ExpertParallelMoE:
    """Dropless MoE layer sharded by experts over a process group.

    backend: object exposing the C-ABI binding functions (paper_2211_15841_b200.api
    on GPUs). Weights: wr [h, E] (replicated), w1_local [h, E_l*f],
    w2_local [E_l*f, h] of this rank's experts.
    """

    def __init__(self, backend, group, hidden, num_experts, top_k, ffn_hidden, act=1, block_size=128,
                 transport="nccl", renormalize=False, aux_loss_coeff=0.0, max_tokens=None):
        """renormalize: top-k gates divided by their sum (the token owner's
        router and its backward; the expert side is unaffected).
        aux_loss_coeff > 0: the auxiliary load-balancing loss of this rank's
        tokens (f_e and P_e over the local batch, as data parallelism
        computes it per micro-batch), its value in `self.aux_loss` (device
        scalar) after each forward and its gradient added to the router's.
        max_tokens: the most tokens any rank will pass to one forward (p2p
        transport: the peer windows are sized once, collectively, for the
        maximum over ranks of this and of the first forward's token counts;
        a later forward with more tokens raises).

        One forward in flight: the state a forward returns refers to buffers
        the layer reuses (cached topologies, the peer windows), so each
        backward must follow its own forward before the next forward; a
        stale state raises instead of silently computing wrong gradients. With
        the p2p transport the state's logits / expert_idx / gates are views of
        the library layer's own buffers: valid until the next forward or
        `self.win.close()`."""
        if transport not in ("nccl", "p2p"):
            raise ValueError(f"transport must be 'nccl' or 'p2p', got {transport!r}")
        self.renormalize = bool(renormalize)
        self.aux_loss_coeff = float(aux_loss_coeff)
        self.aux_loss = None
        self.B = backend
        self.group = group
        self.transport = transport
        self.win = None
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.h, self.E, self.k, self.f, self.act, self.bs = hidden, num_experts, top_k, ffn_hidden, act, block_size
        self.e0, self.e1 = local_expert_range(self.rank, self.world, num_experts)
        self.El = self.e1 - self.e0
        self.max_tokens = int(max_tokens) if max_tokens else 0
        self.t_max = 0
        self._fwd_step = 0

    def _cfg(self, tokens, experts, k):
        cfg = self.B.make_config(max(int(tokens), 1), self.h, experts, k, self.f, self.bs, self.act)
        if experts == self.E:   # the token owner's (router) config
            cfg.renormalize = int(self.renormalize)
            cfg.aux_loss_coeff = self.aux_loss_coeff
        return cfg

    def _aux_ws(self, cfg_l, device):
        """The workspace holding the auxiliary loss between forward and backward:
        the local topology's cached one when there is one."""
        c = self.__dict__.get("_topo_cache", {})
        if "local" in c:
            return c["local"][3]
        if getattr(self, "_aux_ws_buf", None) is None:
            self._aux_ws_buf = self.B.workspace(cfg_l, device)
        return self._aux_ws_buf

    def _aux_forward(self, cfg_l, logits, idx):
        """The auxiliary loss of this rank's tokens (kept in the workspace until the backward)."""
        if self.aux_loss_coeff > 0:
            loss, _ = self.B.moe_load_balance_loss(cfg_l, logits, idx, ws=self._aux_ws(cfg_l, logits.device))
            self.aux_loss = loss

    def _aux_dlogits(self, cfg_l, logits, dlogits):
        if self.aux_loss_coeff > 0:
            self.B.moe_add_aux_dlogits(cfg_l, logits, dlogits, self._aux_ws(cfg_l, logits.device))

    def _router_bwd_ws(self, cfg_l, device):
        return self._aux_ws(cfg_l, device) if self.aux_loss_coeff > 0 else None

    def _topology(self, cfg, ids, slot):
        """moe_topology into device arrays and a workspace cached per slot. The
        expert side's row count changes every step, so its arrays are sized for
        a capacity (grown geometrically) rather than the exact count: the
        library only reads and writes the first R entries / device-side sizes."""
        if not hasattr(self.B, "Topology"):
            return self.B.moe_topology(cfg, ids)
        cache = self.__dict__.setdefault("_topo_cache", {})
        need = int(cfg.tokens) * int(cfg.top_k)
        ent = cache.get(slot)
        if ent is None or ent[0] < need or ent[1] != (cfg.num_experts, cfg.top_k):
            cap = max(need, int(ent[0] * 1.25) if ent is not None else need)
            cap = -(-cap // 1024) * 1024
            cap_cfg = self.B.cfg_replace(cfg, tokens=cap // int(cfg.top_k))
            ent = (cap, (cfg.num_experts, cfg.top_k), self.B.Topology(cap_cfg, ids.device),
                   self.B.workspace(cap_cfg, ids.device))
            cache[slot] = ent
        return self.B.moe_topology(cfg, ids, topo=ent[2], ws=ent[3])

    def _a2a(self, out, inp, out_splits, in_splits):
        dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)

    def _gather_counts(self, counts):
        """[P, E] int32 per-rank histograms on every rank (one collective)."""
        out = counts.new_empty(self.world, counts.numel())
        try:
            dist.all_gather_into_tensor(out, counts, group=self.group)
        except (RuntimeError, NotImplementedError, AttributeError):
            dist.all_gather(list(out.unbind(0)), counts, group=self.group)
        return out

    def _fused_router(self, cfg):
        f = getattr(self.B, "router_on_tensor_cores", None)
        return bool(f and f(cfg))

    def forward(self, x, wr, w1_local, w2_local):
        self._fwd_step += 1
        if self.transport == "p2p":
            y, st = self._forward_p2p(x, wr, w1_local, w2_local)
        else:
            y, st = self._forward_nccl(x, wr, w1_local, w2_local)
        st.step = self._fwd_step
        return y, st

    def _forward_nccl(self, x, wr, w1_local, w2_local):
        B = self.B
        T = x.shape[0]
        cfg_l = self._cfg(T, self.E, self.k)
        # (1) local router + top-k, grouped by GLOBAL expert
        logits, idx, gates = B.moe_router(cfg_l, x, wr)
        topo_l = self._topology(cfg_l, idx, "local")
        self._aux_forward(cfg_l, logits, idx)
        x_sorted = B.moe_sort_rows(cfg_l, x, topo_l)
        # (2) count exchange -> split sizes (the one host synchronisation)
        counts_dev = self._gather_counts(topo_l["counts"][: self.E].to(torch.int32).contiguous())
        counts_all = counts_dev.cpu().numpy()
        sends = send_splits(counts_all[self.rank], self.world)
        recvs = [int(counts_all[q, self.e0:self.e1].sum()) for q in range(self.world)]
        n_recv = int(sum(recvs))
        # (3) dispatch
        recv_x = x.new_empty(n_recv, self.h)
        self._a2a(recv_x, x_sorted, recvs, sends)
        # (4) local experts: topology over E_l experts, padded gather, SDD(+act), DSD, un-pad
        cfg_e = self._cfg(n_recv, self.El, 1)
        topo_e = x_g = act_deriv = a = None
        y_recv = x.new_empty(n_recv, self.h)
        if n_recv > 0:
            if hasattr(B, "moe_ep_recv_ids"):   # arrival-order expert ids built on the device
                ids = B.moe_ep_recv_ids(counts_dev, self.e0, self.El, n_recv)
            else:
                ids = torch.from_numpy(recv_plan(counts_all, self.rank, self.world)[1]).to(x.device)
            topo_e = self._topology(cfg_e, ids, "experts")
            x_g = B.moe_gather(cfg_e, recv_x, topo_e)
            if self.act != 0:
                a, act_deriv = B.moe_sdd_deriv(cfg_e, x_g, w1_local, 0, topo_e, act=self.act, want_deriv=True)
            else:
                a = B.moe_sdd(cfg_e, x_g, w1_local, 0, topo_e)
            B.moe_dsd_scatter(cfg_e, a, w2_local, topo_e, None, y=y_recv)   # DSD + un-pad in one kernel
        # (5) combine: reverse exchange, then gate-weighted sum in token order
        y_sorted = x.new_empty(T * self.k, self.h)
        self._a2a(y_sorted, y_recv, sends, recvs)
        y = B.moe_unsort_rows(cfg_l, y_sorted, topo_l, gates)
        st = EPState(cfg_l, cfg_e, logits, idx, gates, topo_l, topo_e, sends, recvs, x_g, act_deriv, a, y_sorted, n_recv)
        return y, st

    def backward(self, st: EPState, x, dy, wr, w1_local, w2_local, reduce_dwr=True):
        """reduce_dwr=False leaves the router gradient rank-local (the caller
        sums it, e.g. after replaying a captured step)."""
        if st.step != self._fwd_step:
            raise RuntimeError(f"ExpertParallelMoE: backward of forward #{st.step} after forward #{self._fwd_step}; "
                               "the layer reuses its topology and window buffers, so each backward must follow "
                               "its own forward (one forward in flight)")
        if self.transport == "p2p":
            return self._backward_p2p(st, x, dy, wr, w1_local, w2_local, reduce_dwr)
        B = self.B
        cfg_l, cfg_e = st.cfg_local, st.cfg_e
        fused = self._fused_router(cfg_l)
        side = None
        # b1 on the token owner: dY rows in expert order, dgates (+ the router's dlogits)
        if fused:
            dy_sorted, dgates, dlogits = B.moe_unsort_rows_bwd_router(cfg_l, dy, st.y_sorted, st.topo_local, st.gates,
                                                                      st.logits, st.expert_idx)
            self._aux_dlogits(cfg_l, st.logits, dlogits)
            # b7 dWr = x^T . dlogits needs nothing else: on a side stream beside the exchange
            if dy.is_cuda:
                side = self.__dict__.setdefault("_side", torch.cuda.Stream(device=dy.device))
                side.wait_stream(torch.cuda.current_stream(dy.device))
                dlogits.record_stream(side)
                ws_l = self._topo_cache["local"][3]      # the local topology's scratch: idle until the next step
                with torch.cuda.stream(side):
                    dwr = B.moe_router_dwr(cfg_l, x, dlogits, ws=ws_l)
            else:
                dwr = B.moe_router_dwr(cfg_l, x, dlogits)
        else:
            dy_sorted, dgates = B.moe_unsort_rows_bwd(cfg_l, dy, st.y_sorted, st.topo_local, st.gates)
        dy_recv = dy.new_empty(st.n_recv, self.h)
        self._a2a(dy_recv, dy_sorted, st.recvs, st.sends)
        # every column / row is written by the products (experts without tokens get exact zeros)
        dw1 = torch.empty(self.h, self.El * self.f, dtype=w1_local.dtype, device=dy.device)
        dw2 = torch.empty(self.El * self.f, self.h, dtype=w2_local.dtype, device=dy.device)
        if st.n_recv == 0:
            dw1.zero_()
            dw2.zero_()
        dx_recv = dy.new_empty(st.n_recv, self.h)
        if st.n_recv > 0:
            dy_g = B.moe_gather(cfg_e, dy_recv, st.topo_e)
            if self.act != 0:
                dh = B.moe_sdd_deriv(cfg_e, dy_g, w2_local, 1, st.topo_e, act=self.act, deriv_src=st.act_deriv)
            else:
                dh = B.moe_sdd(cfg_e, dy_g, w2_local, 1, st.topo_e)
            B.moe_dsd(cfg_e, st.a, 1, dy_g, 0, st.topo_e, out=dw2)
            B.moe_dds(cfg_e, st.x_g, 1, dh, 0, st.topo_e, out=dw1)
            B.moe_dsd_dx(cfg_e, dh, w1_local, st.topo_e, dx=dx_recv)          # DSD^T + un-pad in one kernel
        dx_sorted = dy.new_empty(cfg_l.tokens * self.k, self.h)
        self._a2a(dx_sorted, dx_recv, st.sends, st.recvs)
        if fused:   # b6 + b7: un-sort fused with dx += dlogits . Wr^T (tcgen05)
            dx = B.moe_sort_rows_bwd_router(cfg_l, dx_sorted, st.topo_local, dlogits, wr)
            if side is not None:
                torch.cuda.current_stream(dy.device).wait_stream(side)
                dwr.record_stream(torch.cuda.current_stream(dy.device))
        else:
            dx = B.moe_sort_rows_bwd(cfg_l, dx_sorted, st.topo_local)
            dwr = B.moe_router_bwd(cfg_l, x, wr, st.logits, st.expert_idx, dgates, dx, ws=self._router_bwd_ws(cfg_l, dy.device))
        if reduce_dwr:
            dist.all_reduce(dwr, op=dist.ReduceOp.SUM, group=self.group)   # data-parallel router grad
        return dx, dwr, dw1, dw2

    # ------------------------------------------------------------------ peer-memory transport (NEXT-1)
    # The whole step runs inside the library's expert-parallel layer object
    # (include/moe.h moe_ep_*, csrc/ep_layer.cu); this is argument marshalling.
    def _layer(self, T, device):
        """The C-ABI layer, created collectively at the first forward (every
        rank reaches it) with windows sized for t_max = the maximum over ranks
        of max_tokens and the first forward's token count: the peers write at
        offsets of their own window layout, so all layouts must agree."""
        from .ep_p2p import EpLayer
        if self.win is None:
            self.win = EpLayer(self.group, self.h, self.E, self.k, self.f, self.act, self.bs, self.renormalize,
                               self.aux_loss_coeff, max(int(T), self.max_tokens), device)
            self.t_max = self.win.t_max
        elif T > self.t_max:
            raise ValueError(f"ExpertParallelMoE: {T} tokens on rank {self.rank} exceed the {self.t_max} per rank the "
                             "peer windows were sized for at the first forward; pass max_tokens= to the constructor")
        return self.win

    def _forward_p2p(self, x, wr, w1_local, w2_local):
        from .ep_p2p import T_EXPERT_IDX, T_GATES, T_LOGITS
        T = int(x.shape[0])
        L = self._layer(T, x.device)
        y = L.forward(x, wr, w1_local, w2_local)
        if self.aux_loss_coeff > 0:
            self.aux_loss = L.aux[0:1]
        logits = L.tensor(T_LOGITS, (T, self.E), torch.float32)
        idx = L.tensor(T_EXPERT_IDX, (T, self.k), torch.int32)
        gates = L.tensor(T_GATES, (T, self.k), torch.float32)
        return y, EPState(None, None, logits, idx, gates, None, None, None, None, None, None, None, None, -1)

    def _backward_p2p(self, st: EPState, x, dy, wr, w1_local, w2_local, reduce_dwr=True):
        dx, dwr, dw1, dw2 = self.win.backward(x, dy, wr, w1_local, w2_local)
        if reduce_dwr:
            dist.all_reduce(dwr, op=dist.ReduceOp.SUM, group=self.group)   # data-parallel router grad
        return dx, dwr, dw1, dw2


# ----------------------------------------------------------------------------- bench (N > 1)

class _TimedBackend:
    """Wraps the binding: CUDA events around every moe_* call on the current
    stream (one extra eager EP step, outside the timed region)."""

    def __init__(self, mod):
        self.mod, self.marks = mod, []

    def __getattr__(self, name):
        f = getattr(self.mod, name)
        if not callable(f) or not name.startswith("moe_"):
            return f

        def w(*a, **k):
            self.marks.append((name, f, a, k))
            return f(*a, **k)
        return w


def _ep_roofline(layer, A, x, dy, wr, w1l, w2l, peaks, dev, shp):
    """Roofline of the expert side's dominant kernel (the SDD, act and act'
    written) in one extra eager step on this rank: algorithmic bytes of the
    rank's received rows (2(Rh + Rf + E_l h f) + 2 R f) / its
    event-timed duration; the max over ranks of the duration is reported."""
    torch.cuda.synchronize()
    y, st = layer.forward(x, wr, w1l, w2l)
    layer.backward(st, x, dy, wr, w1l, w2l)
    torch.cuda.synchronize()
    if layer.transport == "p2p":
        # the C layer's expert-side state of that step: re-issue its forward SDD
        import ctypes

        from ._lib import check, lib
        from .ep_p2p import T_A, T_ACT_DERIV, T_X_G
        cfg_e, topo_e = layer.win.state(1)
        ptr = {n: lib.moe_ep_tensor(layer.win.h_ep, n) for n in (T_X_G, T_A, T_ACT_DERIV)}

        def f():
            check("moe_sdd_deriv", lib.moe_sdd_deriv(
                ctypes.byref(cfg_e), ctypes.c_void_p(ptr[T_X_G]), ctypes.c_void_p(w1l.data_ptr()), 0,
                ctypes.byref(topo_e), int(layer.act), None, ctypes.c_void_p(ptr[T_A]),
                ctypes.c_void_p(ptr[T_ACT_DERIV]) if layer.act != 0 else None,
                ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
        a, k = (), {}
    else:
        B0 = layer.B
        tb = _TimedBackend(B0)
        layer.B = tb
        try:
            y, st = layer.forward(x, wr, w1l, w2l)
            layer.backward(st, x, dy, wr, w1l, w2l)
            torch.cuda.synchronize()
        finally:
            layer.B = B0
        calls = [(f, a, k) for n, f, a, k in tb.marks if n in ("moe_sdd_deriv", "moe_sdd")]
        if not calls:
            return None
        f, a, k = calls[0]          # the forward SDD, re-issued back to back on the same operands

    def timed_ms(fn, reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fn()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / reps
    sdd_ms = timed_ms(lambda: f(*a, **k), 10)
    ms = torch.tensor([sdd_ms, 1.0], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if layer.transport == "p2p":
        R = int(layer.win.n_recv().item())
    else:
        R = int(st.n_recv)
    Rmax = torch.tensor([R], dtype=torch.float64, device=dev)
    dist.all_reduce(Rmax, op=dist.ReduceOp.MAX)
    R = int(Rmax.item())
    h, f, El = layer.h, layer.f, layer.El
    bytes_ = 2 * (R * h + R * f + El * h * f)                     # one sparse output
    bytes2 = bytes_ + (2 * R * f if layer.act != 0 else 0)       # this design also writes act'(H) (R18)
    dur = float(ms[0].item()) * 1e-3
    ach = bytes_ / dur / 1e9
    return {"kernel": "sdd (expert side)", "launch_ms": round(float(ms[0].item()), 4), "bound": "hbm",
            "achieved": round(ach, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": round(ach / peaks["hbm_gbs"], 4), "peak_source": peaks.get("source", "measured") + " (burst)",
            "traffic": None, "rows_received_max": R, "alg_bytes": bytes_,
            "design_two_outputs": {"bytes": bytes2, "achieved": round(bytes2 / dur / 1e9, 1),
                                   "frac": round(bytes2 / dur / 1e9 / peaks["hbm_gbs"], 4)},
            "note": "after the timed region: the forward SDD of one extra eager step re-issued 10x back to back "
                    "on its operands, CUDA events on the launching stream, max over ranks"}


def bench_ep(args, peaks, clock_sampler=None):
    """Weak-scaling EP benchmark: T_local tokens per rank of the BASELINE
    config, experts split over ranks, NCCL all-to-all. Returns rank 0's JSON
    dict (others None). Timed on the device with CUDA events, max over ranks;
    e2e through the same public layer with pinned host inputs / outputs."""
    import os

    from . import api as A
    from synth import inputs as S

    os.environ.setdefault("RANK", "0")
    os.environ.setdefault("WORLD_SIZE", "1")
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29517")
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    # test hooks (not used by the driver): MOE_EP_SAME_DEVICE=1 puts every rank
    # on cuda:0 and MOE_EP_BACKEND=gloo replaces NCCL for the process group, so
    # the N > 1 bench flow (windows, graphs, e2e, max over ranks) can be run on
    # a one-GPU box; numbers from such a run are not measurements
    if os.environ.get("MOE_EP_SAME_DEVICE") == "1":
        local_rank = 0
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    backend = os.environ.get("MOE_EP_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(backend)
    rank, world = dist.get_rank(), dist.get_world_size()
    shp = S.CONFIGS[args.config]
    T, h, f, E, k = shp.tokens, shp.hidden, shp.ffn, shp.experts, shp.top_k
    wts = S.make_inputs(shp, seed=0, tokens=1)                 # identical global weights on every rank
    inp = S.make_inputs(shp, seed=100 + rank)                  # rank-local tokens
    e0, e1 = local_expert_range(rank, world, E)
    wr = wts["wr"].to(dev)
    w1l = wts["w1"][:, e0 * f:e1 * f].contiguous().to(dev)
    w2l = wts["w2"][e0 * f:e1 * f].contiguous().to(dev)
    x, dy = inp["x"].to(dev), inp["dy"].to(dev)
    del wts
    transport = getattr(args, "transport", "nccl")
    transport = "p2p" if transport == "auto" else transport
    l2 = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)
    note = None

    def make_layer(tr):
        return ExpertParallelMoE(A, dist.group.WORLD, h, E, k, f, act=shp.act, transport=tr)

    def warm(lay, n):
        for _ in range(n):
            l2.zero_()
            y_, st_ = lay.forward(x, wr, w1l, w2l)
            lay.backward(st_, x, dy, wr, w1l, w2l)
        torch.cuda.synchronize()

    layer = make_layer(transport)
    if transport == "p2p":   # fall back to NCCL, on every rank alike, if peer memory is unusable
        ok = torch.ones(1, device=dev)
        try:
            warm(layer, args.warmup)
            if layer.win.error_word() != 0:
                raise RuntimeError(f"exchange wait timed out (region {layer.win.error_word() - 1})")
        except RuntimeError as exc:
            ok.zero_()
            note = f"p2p unavailable ({exc}); NCCL all-to-all used"
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if ok.item() == 0:
            print(f"[bench] {note or 'p2p failed on a peer rank; NCCL all-to-all used'}", file=sys.stderr)
            transport = "nccl"
            layer = make_layer("nccl")
    warm(layer, args.warmup)
    launches0 = A.lib.moe_total_launch_count()
    warm(layer, 1)
    launches_per_step = A.lib.moe_total_launch_count() - launches0

    # the p2p step has no host synchronisation: capture forward + backward in a
    # CUDA graph (the router-gradient sum stays an eager NCCL all-reduce)
    graph = None
    if transport == "p2p" and not getattr(args, "no_graph", False):
        try:
            side = torch.cuda.Stream(device=dev)
            side.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(side):
                y_, st_ = layer.forward(x, wr, w1l, w2l)
                layer.backward(st_, x, dy, wr, w1l, w2l, reduce_dwr=False)
            torch.cuda.current_stream(dev).wait_stream(side)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                g_y, g_st = layer.forward(x, wr, w1l, w2l)
                g_dx, g_dwr, _, _ = layer.backward(g_st, x, dy, wr, w1l, w2l, reduce_dwr=False)
            torch.cuda.synchronize()
        except Exception as exc:  # noqa: BLE001 - eager launches are still correct
            print(f"[bench] graph capture unavailable ({exc}); timing eager launches", file=sys.stderr)
            graph = None

    def step(xd, dyd):
        if graph is not None:   # captured on the static x, dy
            if xd is not x:
                x.copy_(xd)
                dy.copy_(dyd)
            graph.replay()
            dist.all_reduce(g_dwr, op=dist.ReduceOp.SUM)
            return g_y, g_dx
        y, st = layer.forward(xd, wr, w1l, w2l)
        dx, _, _, _ = layer.backward(st, xd, dyd, wr, w1l, w2l)
        return y, dx

    def timed(fn, steps):
        total = 0.0
        for _ in range(steps):
            l2.zero_()
            dist.barrier()
            torch.cuda.synchronize()
            s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s_.record()
            fn()
            e_.record()
            torch.cuda.synchronize()
            total += s_.elapsed_time(e_)
        t = torch.tensor([total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(2):
        step(x, dy)
    torch.cuda.synchronize()
    clk = clock_sampler(dev.index) if clock_sampler else None
    if clk:
        clk.start()
    ms = timed(lambda: step(x, dy), args.steps)
    clocks = clk.stop() if clk else None
    launches = launches_per_step * args.steps
    if transport == "p2p" and layer.win.error_word() != 0:
        raise RuntimeError(f"p2p exchange wait timed out during the timed steps (region {layer.win.error_word() - 1})")
    roof = _ep_roofline(layer, A, x, dy, wr, w1l, w2l, peaks, dev, shp)
    # end to end: pinned host x, dy in; y, dx out, every step. Host->device
    # copies of step i+1 and device->host copies of step i-1 overlap step i's
    # compute (double-buffered device inputs / outputs, three streams), as in
    # bench.py's single-GPU e2e; with the p2p transport each buffer has its own
    # captured graph.
    hx, hdy = x.cpu().pin_memory(), dy.cpu().pin_memory()
    hy = [torch.empty(T, h, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    hdx = [torch.empty(T, h, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    xs, dys = [x, torch.empty_like(x)], [dy, torch.empty_like(dy)]
    graphs = [None, None]
    if graph is not None:
        graphs[0] = (graph, g_y, g_dx, g_dwr)
        try:
            g1 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g1):
                y1, st1 = layer.forward(xs[1], wr, w1l, w2l)
                dx1, dwr1, _, _ = layer.backward(st1, xs[1], dys[1], wr, w1l, w2l, reduce_dwr=False)
            graphs[1] = (g1, y1, dx1, dwr1)
        except Exception as exc:  # noqa: BLE001
            print(f"[bench] second graph unavailable ({exc}); e2e with eager launches", file=sys.stderr)
            graphs = [None, None]
    s_in, s_c, s_out = torch.cuda.Stream(device=dev), torch.cuda.current_stream(dev), torch.cuda.Stream(device=dev)
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_comp = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]
    for b_ in range(2):
        ev_comp[b_].record(s_c)
        ev_out[b_].record(s_out)

    def e2e_one(i):
        b_ = i & 1
        with torch.cuda.stream(s_in):
            s_in.wait_event(ev_comp[b_])            # step i-2 finished reading xs[b], dys[b]
            xs[b_].copy_(hx, non_blocking=True)
            dys[b_].copy_(hdy, non_blocking=True)
            ev_in[b_].record(s_in)
        with torch.cuda.stream(s_c):
            s_c.wait_event(ev_in[b_])
            s_c.wait_event(ev_out[b_])              # step i-2's results left the output buffers
            if graphs[b_] is not None:
                gr, y_, dx_, dwr_ = graphs[b_]
                gr.replay()
                dist.all_reduce(dwr_, op=dist.ReduceOp.SUM)
            else:
                y_, st_ = layer.forward(xs[b_], wr, w1l, w2l)
                dx_, _, _, _ = layer.backward(st_, xs[b_], dys[b_], wr, w1l, w2l)
            ev_comp[b_].record(s_c)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_comp[b_])
            hy[b_].copy_(y_, non_blocking=True)
            hdx[b_].copy_(dx_, non_blocking=True)
            ev_out[b_].record(s_out)

    ms_e2e = None
    if not getattr(args, "no_e2e", False):
        for i in range(2):
            e2e_one(i)
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        st_e, en_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st_e.record(s_in)
        for i in range(args.steps):
            e2e_one(i)
        s_out.wait_stream(s_c)
        en_e.record(s_out)
        torch.cuda.synchronize()
        te = torch.tensor([st_e.elapsed_time(en_e)], dtype=torch.float64, device=dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        ms_e2e = float(te.item())
    out = None
    if rank == 0:
        out = {"metric": "dropless MoE layer fwd+bwd tokens/s", "value": round(T * world * args.steps / (ms / 1e3), 1),
               "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded inputs, random-init weights)",
               "config": {"workload": shp.name, "tokens_per_rank": T, "hidden": h, "ffn_hidden": f,
                          "num_experts": E, "top_k": k, "parallelism": f"ep{world}", "transport": transport,
                          "launch_mode": "cuda_graph" if graph is not None else "eager",
                          **({"transport_note": note} if note else {}),
                          "l2": "flushed between timed steps (512 MiB memset, outside the events)"},
               "gpu_launches": int(launches), "clocks": clocks, "roofline": roof,
               "e2e": None if ms_e2e is None else {
                   "value": round(T * world * args.steps / (ms_e2e / 1e3), 1), "unit": "tokens/s",
                   "h2d_bytes_per_step": 2 * T * h * 2 * world, "d2h_bytes_per_step": 2 * T * h * 2 * world,
                   "ms_per_step": round(ms_e2e / args.steps, 4),
                   "api": "ExpertParallelMoE.forward/backward over the C ABI + "
                          + ("NCCL all_to_all" if transport == "nccl" else "peer-memory dispatch / combine")
                          + "; copies on separate streams overlapping the neighbouring steps' compute"}}
    dist.barrier()
    dist.destroy_process_group()
    return out
