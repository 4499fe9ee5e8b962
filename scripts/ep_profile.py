"""Per-phase device timeline of the expert-parallel layer at one rank (debug tool).

Run on the GPU box: python scripts/ep_profile.py [nccl|p2p] — prints ms per
phase of one eager forward + backward (CUDA events recorded between the phases
by monkey-patching the binding calls; the p2p exchanges are PeerWindows'
direct library calls and show up in the gaps before the call that follows)."""
import os
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("RANK", "0")
os.environ.setdefault("WORLD_SIZE", "1")
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29531")

from paper_2211_15841_b200 import api as A  # noqa: E402
from paper_2211_15841_b200 import ep  # noqa: E402
from synth import inputs as S  # noqa: E402


class Timed:
    def __init__(self, mod):
        self.mod, self.marks = mod, []

    def __getattr__(self, name):
        f = getattr(self.mod, name)
        if not callable(f) or not name.startswith("moe_"):
            return f

        def w(*a, **k):
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record()
            t0 = time.perf_counter()
            r = f(*a, **k)
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record()
            self.marks.append((name, e0, e1, time.perf_counter() - t0))
            return r
        return w


def main():
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    shp = S.CONFIGS["C1"]
    T, h, f, E, k = shp.tokens, shp.hidden, shp.ffn, shp.experts, shp.top_k
    inp = S.make_inputs(shp, seed=0)
    x, dy = inp["x"].to(dev), inp["dy"].to(dev)
    wr, w1, w2 = (inp[n].to(dev) for n in ("wr", "w1", "w2"))
    B = Timed(A)
    transport = sys.argv[1] if len(sys.argv) > 1 else "nccl"
    layer = ep.ExpertParallelMoE(B, dist.group.WORLD, h, E, k, f, act=shp.act, transport=transport)
    for it in range(4):
        B.marks.clear()
        torch.cuda.synchronize()
        s0 = torch.cuda.Event(enable_timing=True)
        s0.record()
        t0 = time.perf_counter()
        y, st = layer.forward(x, wr, w1, w2)
        layer.backward(st, x, dy, wr, w1, w2)
        s1 = torch.cuda.Event(enable_timing=True)
        s1.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    tot = s0.elapsed_time(s1)
    print(f"step: device {tot:.3f} ms, host wall {wall * 1e3:.3f} ms")
    busy = 0.0
    prev = s0
    for name, e0, e1, host in B.marks:
        gap = prev.elapsed_time(e0)
        dt = e0.elapsed_time(e1)
        busy += dt
        print(f"  {name:24s} gap {gap:7.3f}  kernel(s) {dt:7.3f} ms  host {host * 1e3:6.3f} ms")
        prev = e1
    print(f"  sum of call spans {busy:.3f} ms; rest (collectives, host syncs, glue) {tot - busy:.3f} ms")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
