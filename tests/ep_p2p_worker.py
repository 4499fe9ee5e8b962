"""Worker for the peer-memory expert-parallel GPU test (tests/test_gpu_parity.py):
one process per rank, all on cuda:0 (the only GPU a test box has), gloo for the
setup collectives (handle exchange, barrier) and the router-gradient sum; the
token exchange itself is the library's device-initiated peer stores through
CUDA IPC windows (paper_2211_15841_b200.ep_p2p)."""
import os
import sys


def make_global_inputs(shp, cfg, tokens):
    """The global batch; cfg["starve"] routes no token to the experts of the
    last rank (x[:, h-1] = 1, Wr[h-1, e] = -30 there), so that rank receives
    zero rows and its expert gradients must come out exactly zero."""
    from synth import inputs as S
    import torch
    inp = S.make_inputs(shp, seed=cfg["seed"], tokens=tokens)
    if cfg.get("starve"):
        E, h = shp.experts, shp.hidden
        world = cfg["world"]
        x = inp["x"].clone()
        wr = inp["wr"].clone()
        x[:, h - 1] = 1.0
        wr[h - 1, :] = 0.0
        wr[h - 1, E - E // world:] = -30.0
        inp["x"], inp["wr"] = x.to(torch.bfloat16), wr.to(torch.bfloat16)
    return inp


def rank_tokens(cfg, world):
    """Tokens of each rank: cfg["T"], minus cfg["uneven"] * rank (ranks with
    different batch sizes share one window layout sized for the largest)."""
    return [cfg["T"] - cfg.get("uneven", 0) * r for r in range(world)]


def run(rank, world, port, cfg, q):
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2211_15841_b200 import api as A
    from paper_2211_15841_b200 import ep
    from synth import inputs as S
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        d = torch.device("cuda", 0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        shp = S.CONFIGS[cfg["shape"]]
        Ts = rank_tokens(cfg, world)
        inp = make_global_inputs(shp, cfg, sum(Ts))
        E, f = shp.experts, shp.ffn
        e0, e1 = ep.local_expert_range(rank, world, E)
        sl = slice(sum(Ts[:rank]), sum(Ts[:rank + 1]))
        x, dy = inp["x"][sl].to(d), inp["dy"][sl].to(d)
        wr = inp["wr"].to(d)
        w1 = inp["w1"][:, e0 * f:e1 * f].contiguous().to(d)
        w2 = inp["w2"][e0 * f:e1 * f].contiguous().to(d)
        layer = ep.ExpertParallelMoE(A, dist.group.WORLD, shp.hidden, E, shp.top_k, f, act=shp.act, transport="p2p",
                                     renormalize=cfg.get("renorm", False))
        outs = []
        for _ in range(cfg.get("steps", 2)):   # repeated steps exercise the cumulative epochs
            y, st = layer.forward(x, wr, w1, w2)
            dx, dwr, dw1, dw2 = layer.backward(st, x, dy, wr, w1, w2)
            torch.cuda.synchronize()
            outs.append(y.float().cpu().numpy())
        err = layer.win.error_word()
        same = all(np.array_equal(outs[0], o) for o in outs[1:])
        res = (rank, err, same, y.float().cpu().numpy(), dx.float().cpu().numpy(), dwr.double().cpu().numpy(),
               dw1.float().cpu().numpy(), dw2.float().cpu().numpy(), st.expert_idx.cpu().numpy())
        layer.win.close()
        dist.barrier()
        dist.destroy_process_group()
        q.put(res)
    except Exception as exc:  # report instead of hanging the parent
        import traceback
        q.put((rank, "error", traceback.format_exc() + repr(exc)))
