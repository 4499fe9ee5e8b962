"""Peer-memory transport for expert parallelism (
P:197): the token dispatch / combine of ExpertParallelMoE as kernels
that store rows straight into the owners' windows over NVLink (csrc/ep_p2p.cu,
include/moe.h "expert parallelism over peer memory"), with the per-rank
histograms exchanged the same way — no NCCL all-to-all and no host round
trip, so the host enqueues a whole step without waiting for the device.

Plumbing only: the window is allocated by the library (cudaMalloc), exported
with CUDA IPC and mapped by every peer once; the process group only carries
the 64-byte handles at setup (all_gather_object) and a barrier.
"""
from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

from ._lib import MoeEp, check, lib

REGION = {"x": 3, "dy": 4, "y": 5, "dx": 6}   # MOE_EP_RECV_X, _RECV_DY, _RET_Y, _RET_DX
ERROR = 1


class RawRows:
    """A [rows, hidden] bf16 view of window memory for the binding (which only
    needs data_ptr / dtype / device / shape)."""

    def __init__(self, ptr: int, rows: int, hidden: int, device):
        self.ptr, self.shape, self.device, self.dtype = int(ptr), (int(rows), int(hidden)), device, torch.bfloat16

    def data_ptr(self) -> int:
        return self.ptr


class PeerWindows:
    """This rank's window, every peer's window mapped here and the device plan.
    Exchange epochs live in the window (device side), so these calls are
    graph-capturable."""

    def __init__(self, group, num_experts: int, hidden: int, cap_rows: int, owner_rows: int, device):
        self.group = group
        self.P, self.rank = dist.get_world_size(group), dist.get_rank(group)
        self.E, self.h, self.cap, self.owner, self.device = num_experts, hidden, int(cap_rows), int(owner_rows), device
        args = (self.P, self.E, self.h, self.cap, self.owner)
        self.win, self.mapped = 0, []
        # every rank reaches every collective below, failures included, and all
        # ranks agree on the outcome (so a caller can fall back consistently)
        err, handle = None, None
        try:
            win = ctypes.c_void_p()
            check("moe_ep_window_alloc", lib.moe_ep_window_alloc(lib.moe_ep_window_bytes(*args), ctypes.byref(win)))
            self.win = win.value
            hb = (ctypes.c_char * 64)()
            check("moe_ipc_get_handle", lib.moe_ipc_get_handle(ctypes.c_void_p(self.win), hb))
            handle = bytes(hb)
        except Exception as exc:  # noqa: BLE001 - reported collectively below
            err = f"window: {exc}"
        handles = [None] * self.P
        dist.all_gather_object(handles, handle, group=group)
        ptrs = []
        if err is None:
            try:
                for q, hq in enumerate(handles):
                    if q == self.rank:
                        ptrs.append(self.win)
                        continue
                    if hq is None:
                        raise RuntimeError(f"rank {q} has no window")
                    p = ctypes.c_void_p()
                    buf = (ctypes.c_char * 64).from_buffer_copy(hq)
                    check("moe_ipc_open_handle", lib.moe_ipc_open_handle(buf, ctypes.byref(p)))
                    self.mapped.append(p.value)
                    ptrs.append(p.value)
            except Exception as exc:  # noqa: BLE001
                err = f"peer mapping: {exc}"
        errs = [None] * self.P
        dist.all_gather_object(errs, err, group=group)
        bad = [f"rank {q}: {e}" for q, e in enumerate(errs) if e]
        if bad:
            self.close()
            raise RuntimeError("peer-memory windows unavailable: " + "; ".join(bad))
        self.peers = torch.tensor(ptrs, dtype=torch.int64, device=device)
        self.plan = torch.zeros(lib.moe_ep_plan_ints(self.P, self.E), dtype=torch.int32, device=device)
        self.ep = MoeEp(self.P, self.rank, self.E, self.h, self.cap, self.owner, self.peers.data_ptr(),
                        self.plan.data_ptr())
        self.off = {n: int(lib.moe_ep_window_offset(*args, r)) for n, r in REGION.items()}
        self.err_off = int(lib.moe_ep_window_offset(*args, ERROR))
        torch.cuda.synchronize(device)
        dist.barrier(group=group)

    # ---- views
    def counts_all(self) -> torch.Tensor:
        return self.plan[: self.P * self.E].view(self.P, self.E)

    def n_recv(self) -> torch.Tensor:
        return self.plan[self.P * self.E: self.P * self.E + 1]

    def rows(self, name: str) -> RawRows:
        # receive regions hold the padded layout: up to 127 pad rows per local expert
        n = self.cap + (self.E // self.P) * 128 if name in ("x", "dy") else self.owner
        return RawRows(self.win + self.off[name], n, self.h, self.device)

    def compact_counts(self) -> torch.Tensor:
        """[P, E/P] int32: rows of each of this rank's experts from each source (device)."""
        o = lib.moe_ep_plan_offset(self.P, self.E, 0)
        El = self.E // self.P
        return self.plan[o: o + self.P * El].view(self.P, El)

    def dispatch_padded(self, name: str, x: torch.Tensor, sorted_pos, top_k: int):
        """Rows straight into the owners' padded layouts: x [T, h] in token order
        sent to the sorted positions sorted_pos (input-driven), or, with
        sorted_pos None, rows already in expert order; waits for this rank's
        region (its pad rows still need zeroing)."""
        check("moe_ep_dispatch_padded", lib.moe_ep_dispatch_padded(
            ctypes.byref(self.ep), REGION[name], ctypes.c_void_p(x.data_ptr()),
            None if sorted_pos is None else ctypes.c_void_p(sorted_pos.data_ptr()), int(top_k), self._s()))
        check("moe_ep_wait", lib.moe_ep_wait(ctypes.byref(self.ep), REGION[name], self._s()))
        return self.rows(name)

    def combine_padded(self, name: str, rows_padded):
        """This rank's padded rows back to their sources' return regions; waits for this rank's."""
        check("moe_ep_combine_padded", lib.moe_ep_combine_padded(ctypes.byref(self.ep), REGION[name],
                                                                 ctypes.c_void_p(rows_padded.data_ptr()), self._s()))
        check("moe_ep_wait", lib.moe_ep_wait(ctypes.byref(self.ep), REGION[name], self._s()))
        return self.rows(name)

    # ---- exchanges (stream-ordered on the current stream)
    @staticmethod
    def _s():
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def exchange_counts(self, counts_local: torch.Tensor):
        check("moe_ep_exchange_counts", lib.moe_ep_exchange_counts(ctypes.byref(self.ep),
                                                                   ctypes.c_void_p(counts_local.data_ptr()), self._s()))

    def error_word(self) -> int:
        """0, or 1 + the arrival region whose wait timed out (the plan's last
        int, mirrored from the window's error word). Reads the device."""
        return int(self.plan[-1].item())

    def close(self):
        for p in self.mapped:
            lib.moe_ipc_close_handle(ctypes.c_void_p(p))
        self.mapped = []
        if self.win:
            torch.cuda.synchronize(self.device)
            lib.moe_ep_window_free(ctypes.c_void_p(self.win))
            self.win = 0
