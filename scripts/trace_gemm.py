"""Timeline of the tcgen05 GEMM launches of one layer step (debug tool).

Run on the GPU box:  MOE_GEMM_TRACE=1 python scripts/trace_gemm.py [out.bin]
Every GEMM launch records %globaltimer per CTA and tile (bsgemm.cu trace_ev):
0 producer starts the tile, 1 MMA starts (accumulator free), 2 MMA done
(last commit), 3 epilogue has the accumulator, 4 epilogue done. Prints, per
launch, the kernel span and the mean per-tile phase times.
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("MOE_GEMM_TRACE", "1")

import bench  # noqa: E402

L, C, TT, EV = 16, 160, 32, 14


def main(out):
    from paper_2211_15841_b200 import api as A
    from paper_2211_15841_b200._lib import lib
    from synth import inputs as S
    lib.moe_debug_trace_dump.restype = ctypes.c_int
    lib.moe_debug_trace_dump.argtypes = [ctypes.c_char_p]
    dev = torch.device("cuda", 0)
    shp = S.CONFIGS["C1"]
    T, h, f, E, k = shp.tokens, shp.hidden, shp.ffn, shp.experts, shp.top_k
    inp = S.make_inputs(shp, seed=0)
    cfg = A.make_config(T, h, E, k, f, act=shp.act)
    x, dy = inp["x"].to(dev), inp["dy"].to(dev)
    wr, w1, w2 = (inp[n].to(dev) for n in ("wr", "w1", "w2"))
    saved = A.Saved.allocate(cfg, dev, save_deriv=os.environ.get("MOE_BENCH_ACT_SAVE", "deriv") == "deriv")
    ws = A.workspace(cfg, dev)
    t = {"x": x, "dy": dy, "wr": wr, "w1": w1, "w2": w2, "saved": saved, "ws": ws,
         "y": torch.empty(T, h, dtype=torch.bfloat16, device=dev),
         "dx": torch.empty(T, h, dtype=torch.bfloat16, device=dev),
         "dwr": torch.empty(h, E, dtype=torch.float32, device=dev),
         "dw1": torch.empty(h, E * f, dtype=torch.bfloat16, device=dev),
         "dw2": torch.empty(E * f, h, dtype=torch.bfloat16, device=dev)}
    t["ws_layout"] = bench.ws_views(A, cfg, ws)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    step = bench.Step(A, cfg, t, stream)
    l2 = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)
    for _ in range(3):
        l2.zero_()
        step.run()
    torch.cuda.synchronize()
    lib.moe_debug_trace_dump(out.encode())   # discard warm-up slots
    l2.zero_()
    torch.cuda.synchronize()
    step.run()
    n = lib.moe_debug_trace_dump(out.encode())
    tr = np.fromfile(out, dtype=np.uint64).reshape(n, C, TT, EV).astype(np.float64)
    gemm_names = [nm for nm in step.names if nm in ("router", "sdd", "sdd+gather", "dsd+scatter", "sddT", "dsTd", "dsdT",
                                                   "ddTs", "ddTs+gather", "dsdT+dx",
                                                   "router_dwr", "router_dx")]
    for li in range(n):
        a = tr[li]
        valid = a[..., 1] > 0
        if not valid.any():
            print(f"launch {li}: no 1-SM trace (CTA-pair kernel)")
            continue
        t0 = a[a > 0].min()
        span = (a.max() - t0) / 1e3
        mma = (a[..., 2] - a[..., 1])[valid] / 1e3
        epi = (a[..., 4] - a[..., 3])[valid & (a[..., 4] > 0)] / 1e3
        wait_acc = (a[..., 3] - a[..., 2])[valid & (a[..., 3] > 0)] / 1e3
        first = (a[:, 0, 1] - t0)[a[:, 0, 1] > 0] / 1e3
        # per tile: the MMA of tile i+1 may start only once the epilogue of tile i-1 freed its accumulator
        gap = (a[:, 1:, 1] - a[:, :-1, 2])[(a[:, 1:, 1] > 0) & (a[:, :-1, 2] > 0)] / 1e3
        last_end = (a[..., 4].max(axis=1) - t0) / 1e3
        ntile = valid.sum(axis=1)
        nm = gemm_names[li] if li < len(gemm_names) else "?"
        ent, ext = a[:, 0, 13], a[:, 1, 13]
        if (ent > 0).any():
            e0 = ent[ent > 0].min()
            first_ev = a[:, :, 0:13]
            fe = np.where(first_ev > 0, first_ev, np.inf).min(axis=(1, 2))
            print(f"   kernel entry spread {(ent[ent > 0].max() - e0) / 1e3:.2f} us | entry -> first tile event "
                  f"{np.mean((fe - ent)[(ent > 0) & np.isfinite(fe)]) / 1e3:.2f} us | last exit "
                  f"{(ext.max() - e0) / 1e3:.2f} us after the first entry | last tile event -> exit "
                  f"{np.mean((ext - a[:, :, 0:13].max(axis=(1, 2)))[ext > 0]) / 1e3:.2f} us")
        wend = a[..., 5:13]
        if (wend > 0).any():
            # CTA pairs (leader 2c, peer 2c+1): each epilogue warp's finish after the leader's accumulator-ready
            lead, peer = a[0::2], a[1::2]
            nt_ = min(lead.shape[0], peer.shape[0])
            r0 = lead[:nt_, :, 3:4]
            for nm_, src in (("leader", lead[:nt_, :, 5:13]), ("peer", peer[:nt_, :, 5:13])):
                ok = (src > 0) & (r0 > 0)
                rel = src - r0
                print(f"   epilogue warp done (us after acc ready), {nm_}:",
                      " ".join(f"{rel[..., w][ok[..., w]].mean() / 1e3:.2f}" for w in range(8)))
        print(f"launch {li} ({nm}): span {span:.1f} us | tiles/CTA {ntile.min()}-{ntile.max()} | "
              f"mainloop/tile {mma.mean():.2f} us (max {mma.max():.2f}) | epilogue/tile {epi.mean():.2f} us | "
              f"commit->epi {wait_acc.mean():.2f} us | first MMA start {first.mean():.2f} us (max {first.max():.2f}) | "
              f"CTA end min {last_end[last_end > 0].min():.1f} max {last_end.max():.1f} | "
              f"MMA idle between tiles {gap.mean() if gap.size else 0:.2f} us")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/trace.bin")
