"""ctypes loader for the in-tree C-ABI library libmoe.so (include/moe.h).

Argument marshalling only. There is no fallback: if the library is missing or
fails to load, importing the package raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmoe.so")

c_int32_p = ctypes.POINTER(ctypes.c_int32)
c_float_p = ctypes.POINTER(ctypes.c_float)


class MoeConfig(ctypes.Structure):
    _fields_ = [("tokens", ctypes.c_int64), ("hidden", ctypes.c_int64), ("num_experts", ctypes.c_int64),
                ("top_k", ctypes.c_int64), ("ffn_hidden", ctypes.c_int64), ("block_size", ctypes.c_int64),
                ("act", ctypes.c_int32), ("capacity", ctypes.c_int32),
                ("renormalize", ctypes.c_int32), ("aux_loss_coeff", ctypes.c_float), ("unpadded", ctypes.c_int32)]


TOPO_FIELDS = ["counts", "bins", "padded_bins", "sorted_idx", "pos", "sorted_pos", "row_offsets",
               "col_indices", "row_indices", "t_col_offsets", "t_block_offsets", "t_row_indices", "pair_bins", "row_src",
               "sizes", "brow_start", "brow_rows"]


class MoeTopology(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in TOPO_FIELDS]


class MoeWeights(ctypes.Structure):
    _fields_ = [("wr", ctypes.c_void_p), ("w1", ctypes.c_void_p), ("w2", ctypes.c_void_p)]


class MoeGrads(ctypes.Structure):
    _fields_ = [("dwr", ctypes.c_void_p), ("dw1", ctypes.c_void_p), ("dw2", ctypes.c_void_p)]


class MoeEp(ctypes.Structure):
    _fields_ = [("nranks", ctypes.c_int32), ("rank", ctypes.c_int32), ("num_experts", ctypes.c_int32),
                ("hidden", ctypes.c_int32), ("cap_rows", ctypes.c_int64), ("owner_rows", ctypes.c_int64),
                ("peers", ctypes.c_void_p), ("plan", ctypes.c_void_p)]


class MoeEpDesc(ctypes.Structure):
    _fields_ = [("nranks", ctypes.c_int32), ("rank", ctypes.c_int32), ("max_tokens", ctypes.c_int64),
                ("hidden", ctypes.c_int64), ("num_experts", ctypes.c_int64), ("top_k", ctypes.c_int64),
                ("ffn_hidden", ctypes.c_int64), ("block_size", ctypes.c_int64), ("act", ctypes.c_int32),
                ("renormalize", ctypes.c_int32), ("aux_loss_coeff", ctypes.c_float),
                ("recv_rows_cap", ctypes.c_int64)]


class MoeSaved(ctypes.Structure):
    _fields_ = [("logits", ctypes.c_void_p), ("expert_idx", ctypes.c_void_p), ("gates", ctypes.c_void_p),
                ("topo", MoeTopology), ("x_g", ctypes.c_void_p), ("act_deriv", ctypes.c_void_p),
                ("a", ctypes.c_void_p), ("y_g", ctypes.c_void_p)]


P = ctypes.c_void_p
CFG = ctypes.POINTER(MoeConfig)
TOPO = ctypes.POINTER(MoeTopology)
STATUS = ctypes.c_int

# name -> (restype, argtypes); mirrors include/moe.h exactly
SIGNATURES = {
    "moe_last_error": (ctypes.c_char_p, []),
    "moe_check_config": (STATUS, [CFG]),
    "moe_max_padded_rows": (ctypes.c_int64, [CFG]),
    "moe_max_nnz_blocks": (ctypes.c_int64, [CFG]),
    "moe_expert_capacity": (ctypes.c_int64, [ctypes.c_int64, ctypes.c_int64, ctypes.c_double]),
    "moe_workspace_bytes": (ctypes.c_size_t, [CFG]),
    "moe_device_sm_count": (ctypes.c_int, []),
    "moe_workspace_offset": (ctypes.c_size_t, [CFG, ctypes.c_int]),
    "moe_router": (STATUS, [CFG, P, P, P, P, P, P, P]),
    "moe_topk": (STATUS, [CFG, P, P, P, P]),
    "moe_topology": (STATUS, [CFG, P, TOPO, P, P]),
    "moe_topology_from_router": (STATUS, [CFG, P, TOPO, P, P]),
    "moe_router_topology": (STATUS, [CFG, P, P, P, P, P, TOPO, P, P]),
    "moe_gather": (STATUS, [CFG, P, TOPO, P, P]),
    "moe_scatter": (STATUS, [CFG, P, TOPO, P, P, P]),
    "moe_scatter_bwd": (STATUS, [CFG, P, P, TOPO, P, P, P, P]),
    "moe_gather_bwd": (STATUS, [CFG, P, TOPO, P, P]),
    "moe_sort_rows": (STATUS, [CFG, P, TOPO, P, P]),
    "moe_unsort_rows": (STATUS, [CFG, P, TOPO, P, P, P]),
    "moe_unsort_rows_bwd": (STATUS, [CFG, P, P, TOPO, P, P, P, P]),
    "moe_sort_rows_bwd": (STATUS, [CFG, P, TOPO, P, P]),
    "moe_unsort_rows_bwd_router": (STATUS, [CFG, P, P, TOPO, P, P, P, P, P, P, P]),
    "moe_sort_rows_bwd_router": (STATUS, [CFG, P, TOPO, P, P, P, P]),
    "moe_ep_window_bytes": (ctypes.c_size_t, [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                              ctypes.c_int64]),
    "moe_ep_window_offset": (ctypes.c_int64, [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                              ctypes.c_int64, ctypes.c_int]),
    "moe_ep_plan_ints": (ctypes.c_int, [ctypes.c_int, ctypes.c_int]),
    "moe_ep_window_alloc": (STATUS, [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]),
    "moe_ep_window_free": (STATUS, [P]),
    "moe_ipc_get_handle": (STATUS, [P, P]),
    "moe_ipc_open_handle": (STATUS, [P, ctypes.POINTER(ctypes.c_void_p)]),
    "moe_ipc_close_handle": (STATUS, [P]),
    "moe_ep_exchange_counts": (STATUS, [ctypes.POINTER(MoeEp), P, P]),
    "moe_ep_dispatch_padded": (STATUS, [ctypes.POINTER(MoeEp), ctypes.c_int, P, P, ctypes.c_int, P]),
    "moe_ep_combine_padded": (STATUS, [ctypes.POINTER(MoeEp), ctypes.c_int, P, P]),
    "moe_ep_plan_offset": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "moe_topology_counts": (STATUS, [CFG, P, ctypes.c_int, TOPO, P]),
    "moe_zero_pad_rows": (STATUS, [CFG, TOPO, P, P]),
    "moe_ep_wait": (STATUS, [ctypes.POINTER(MoeEp), ctypes.c_int, P]),
    "moe_ep_recv_ids": (STATUS, [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, ctypes.c_int64, P]),
    "moe_sdd": (STATUS, [CFG, P, P, ctypes.c_int, TOPO, ctypes.c_int32, P, P, P, P]),
    "moe_sdd_deriv": (STATUS, [CFG, P, P, ctypes.c_int, TOPO, ctypes.c_int32, P, P, P, P]),
    "moe_sdd_act_coded": (STATUS, [CFG, P, P, ctypes.c_int, TOPO, ctypes.c_int32, P, P, P]),
    "moe_act_code_decode_host": (STATUS, [ctypes.c_int32, P, P, ctypes.c_int64]),
    "moe_dsd": (STATUS, [CFG, P, ctypes.c_int, P, ctypes.c_int, TOPO, P, P]),
    "moe_dsd_rows": (STATUS, [CFG, P, P, ctypes.c_int, TOPO, P, P]),
    "moe_ep_combine_dest": (STATUS, [ctypes.POINTER(MoeEp), ctypes.c_int, P, ctypes.c_int64, P]),
    "moe_ep_signal": (STATUS, [ctypes.POINTER(MoeEp), ctypes.c_int, P]),
    "moe_dsd_scatter": (STATUS, [CFG, P, P, TOPO, P, P, P, P]),
    "moe_sdd_gather": (STATUS, [CFG, P, P, TOPO, ctypes.c_int32, P, P, P, P]),
    "moe_dds_gather": (STATUS, [CFG, P, P, TOPO, P, P, P]),
    "moe_gather_is_fused": (ctypes.c_int, [CFG]),
    "moe_dsd_dx": (STATUS, [CFG, P, P, TOPO, P, P, P, P, P]),
    "moe_dds": (STATUS, [CFG, P, ctypes.c_int, P, ctypes.c_int, TOPO, P, P]),
    "moe_router_bwd": (STATUS, [CFG, P, P, P, P, P, P, P, P, P]),
    "moe_scatter_bwd_router": (STATUS, [CFG, P, P, TOPO, P, P, P, P, P, P, P]),
    "moe_router_dwr": (STATUS, [CFG, P, P, P, P, P]),
    "moe_load_balance_loss": (STATUS, [CFG, P, P, P, P]),
    "moe_add_aux_dlogits": (STATUS, [CFG, P, P, P, P]),
    "moe_router_dx": (STATUS, [CFG, P, P, P, TOPO, P, P]),
    "moe_forward": (STATUS, [CFG, ctypes.POINTER(MoeWeights), P, P, ctypes.POINTER(MoeSaved), P, P]),
    "moe_backward": (STATUS, [CFG, ctypes.POINTER(MoeWeights), ctypes.POINTER(MoeSaved), P, P, P,
                              ctypes.POINTER(MoeGrads), P, P]),
    "moe_ep_init": (STATUS, [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(MoeEpDesc), ctypes.c_int]),
    "moe_ep_get_handle": (STATUS, [P, P]),
    "moe_ep_connect": (STATUS, [P, P]),
    "moe_ep_forward": (STATUS, [P, ctypes.c_int64, ctypes.POINTER(MoeWeights), P, P, P]),
    "moe_ep_backward": (STATUS, [P, ctypes.POINTER(MoeWeights), P, P, P, ctypes.POINTER(MoeGrads), P]),
    "moe_ep_tensor": (ctypes.c_void_p, [P, ctypes.c_int]),
    "moe_ep_state": (STATUS, [P, ctypes.c_int, CFG, TOPO]),
    "moe_ep_exchange_desc": (STATUS, [P, ctypes.POINTER(MoeEp)]),
    "moe_ep_destroy": (STATUS, [P]),
    "moe_last_launch_count": (ctypes.c_int, []),
    "moe_total_launch_count": (ctypes.c_int64, []),
}

STATUS_NAMES = {0: "MOE_OK", 1: "MOE_EINVAL", 2: "MOE_ESHAPE", 3: "MOE_EUNSUPPORTED", 4: "MOE_ECUDA",
                5: "MOE_ENCCL", 6: "MOE_EWORKSPACE"}


class MoeError(RuntimeError):
    def __init__(self, fn, status, msg):
        super().__init__(f"{fn} -> {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run `make` (or __graft_entry__.build()). "
                          "There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


def check(fn: str, status: int):
    if status != 0:
        raise MoeError(fn, status, lib.moe_last_error().decode())
