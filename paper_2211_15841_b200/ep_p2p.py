"""Peer-memory transport for expert parallelism (
P:197): the token dispatch / combine of ExpertParallelMoE as kernels
that store rows straight into the owners' windows over NVLink (csrc/ep_p2p.cu,
include/moe.h "expert parallelism over peer memory"), with the per-rank
histograms exchanged the same way — no NCCL all-to-all and no host round
trip, so the host enqueues a whole step without waiting for the device.

Plumbing only: the layer object (moe_ep_init) allocates this rank's window
(cudaMalloc) and every buffer of the step, exports the window with CUDA IPC
and maps every peer's once (moe_ep_connect); the process group only carries
the agreed token maximum and the 64-byte handles at setup (all_gather_object)
and a barrier. Forward and backward are single library calls.
"""
from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

from ._lib import MoeConfig, MoeEpDesc, MoeGrads, MoeTopology, MoeWeights, check, lib


class _DevView:
    """Zero-copy torch view of library-owned device memory (CUDA array interface)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(int(v) for v in shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 2, "strides": None}


def dev_view(ptr: int, shape, dtype) -> torch.Tensor:
    typestr = {torch.int32: "<i4", torch.float32: "<f4"}[dtype]
    return torch.as_tensor(_DevView(ptr, shape, typestr), device="cuda")


T_LOGITS, T_EXPERT_IDX, T_GATES, T_PLAN, T_AUX, T_X_G, T_A, T_ACT_DERIV = range(8)   # MOE_EP_T_*


class EpLayer:
    """The C-ABI expert-parallel layer of this rank (include/moe.h moe_ep_*):
    the library owns the window, the buffers and the whole step (forward and
    backward run in library kernels, stream-ordered, no host synchronisation).
    This class is plumbing: the collective setup (max_tokens agreed over the
    group, the 64-byte window handles all-gathered) and argument marshalling."""

    def __init__(self, group, hidden: int, num_experts: int, top_k: int, ffn_hidden: int, act: int, block_size: int,
                 renormalize: bool, aux_loss_coeff: float, max_tokens: int, device, recv_rows_cap: int = 0):
        self.group = group
        self.P, self.rank = dist.get_world_size(group), dist.get_rank(group)
        self.E, self.h, self.k, self.device = num_experts, hidden, top_k, torch.device(device)
        ts = [None] * self.P
        dist.all_gather_object(ts, int(max_tokens), group=group)
        self.t_max = max(ts)                      # window layouts must agree on every rank
        desc = MoeEpDesc(self.P, self.rank, self.t_max, hidden, num_experts, top_k, ffn_hidden, block_size, int(act),
                         int(bool(renormalize)), float(aux_loss_coeff), int(recv_rows_cap))
        self.h_ep = ctypes.c_void_p()
        err, handle = None, None
        try:
            check("moe_ep_init", lib.moe_ep_init(ctypes.byref(self.h_ep), ctypes.byref(desc),
                                                 self.device.index if self.device.index is not None else 0))
            hb = (ctypes.c_char * 64)()
            check("moe_ep_get_handle", lib.moe_ep_get_handle(self.h_ep, hb))
            handle = bytes(hb)
        except Exception as exc:  # noqa: BLE001 - reported collectively below
            err = f"init: {exc}"
        handles = [None] * self.P
        dist.all_gather_object(handles, handle, group=group)
        uuids = [None] * self.P              # explicit peer-access check (NVLink / PCIe P2P) before mapping
        dist.all_gather_object(uuids, str(torch.cuda.get_device_properties(self.device).uuid), group=group)
        if err is None:
            try:
                if any(hq is None for hq in handles):
                    raise RuntimeError("a rank has no window")
                mine = self.device.index if self.device.index is not None else torch.cuda.current_device()
                local = {str(torch.cuda.get_device_properties(j).uuid): j for j in range(torch.cuda.device_count())}
                for q, u in enumerate(uuids):
                    j = local.get(u)
                    if j is not None and j != mine and not torch.cuda.can_device_access_peer(mine, j):
                        raise RuntimeError(f"GPU {mine} cannot access rank {q}'s GPU {j} (cudaDeviceCanAccessPeer)")
                buf = (ctypes.c_char * (64 * self.P)).from_buffer_copy(b"".join(handles))
                check("moe_ep_connect", lib.moe_ep_connect(self.h_ep, buf))
            except Exception as exc:  # noqa: BLE001
                err = f"connect: {exc}"
        errs = [None] * self.P
        dist.all_gather_object(errs, err, group=group)
        bad = [f"rank {q}: {e}" for q, e in enumerate(errs) if e]
        if bad:
            self.close()
            raise RuntimeError("expert-parallel layer unavailable: " + "; ".join(bad))
        self.plan_n = int(lib.moe_ep_plan_ints(self.P, self.E))
        self.plan = dev_view(lib.moe_ep_tensor(self.h_ep, T_PLAN), (self.plan_n,), torch.int32)
        self.aux = dev_view(lib.moe_ep_tensor(self.h_ep, T_AUX), (1 + self.E,), torch.float32)
        torch.cuda.synchronize(self.device)
        dist.barrier(group=group)

    @staticmethod
    def _s():
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def forward(self, x, wr, w1_local, w2_local, y=None):
        T = int(x.shape[0])
        if T > self.t_max:
            raise ValueError(f"{T} tokens on rank {self.rank} exceed max_tokens={self.t_max} the layer was built for")
        y = y if y is not None else torch.empty_like(x)
        w = MoeWeights(wr.data_ptr(), w1_local.data_ptr(), w2_local.data_ptr())
        check("moe_ep_forward", lib.moe_ep_forward(self.h_ep, T, ctypes.byref(w), ctypes.c_void_p(x.data_ptr()),
                                                   ctypes.c_void_p(y.data_ptr()), self._s()))
        return y

    def backward(self, x, dy, wr, w1_local, w2_local):
        dx = torch.empty_like(dy)
        dwr = torch.empty(wr.shape, dtype=torch.float32, device=dy.device)
        dw1, dw2 = torch.empty_like(w1_local), torch.empty_like(w2_local)
        w = MoeWeights(wr.data_ptr(), w1_local.data_ptr(), w2_local.data_ptr())
        g = MoeGrads(dwr.data_ptr(), dw1.data_ptr(), dw2.data_ptr())
        check("moe_ep_backward", lib.moe_ep_backward(self.h_ep, ctypes.byref(w), ctypes.c_void_p(x.data_ptr()),
                                                     ctypes.c_void_p(dy.data_ptr()), ctypes.c_void_p(dx.data_ptr()),
                                                     ctypes.byref(g), self._s()))
        return dx, dwr, dw1, dw2

    def tensor(self, which: int, shape, dtype) -> torch.Tensor:
        return dev_view(lib.moe_ep_tensor(self.h_ep, which), shape, dtype)

    def state(self, side: int):
        cfg, topo = MoeConfig(), MoeTopology()
        check("moe_ep_state", lib.moe_ep_state(self.h_ep, side, ctypes.byref(cfg), ctypes.byref(topo)))
        return cfg, topo

    def error_word(self) -> int:
        """0, 1 + the region whose wait timed out, or 100 (a receive bound was exceeded). Reads the device."""
        return int(self.plan[-1].item())

    def n_recv(self) -> torch.Tensor:
        return self.plan[self.P * self.E: self.P * self.E + 1]

    def close(self):
        if self.h_ep:
            lib.moe_ep_destroy(self.h_ep)
            self.h_ep = ctypes.c_void_p()
