"""Expert parallelism host logic under torch.distributed gloo, world_size 2,
on CPU: the EP layer (paper_2211_15841_b200.ep) with the test-only oracle
backend must reproduce the single-process oracle over the concatenated global
batch — outputs, input gradients, expert weight-gradient slices and the
all-reduced router gradient."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import moe_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(T, h, f, E, seed):
    rng = np.random.default_rng(seed)
    return (rng.normal(size=(T, h)), rng.normal(size=(h, E)) / np.sqrt(h), rng.normal(size=(h, E * f)) / np.sqrt(h),
            rng.normal(size=(E * f, h)) / np.sqrt(f), rng.normal(size=(T, h)))


def _worker(rank, world, port, cfgd, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import ep_cpu_backend as B
    from paper_2211_15841_b200 import ep   # host logic only; compute comes from the test backend
    T, h, f, E, k, act = cfgd["T"], cfgd["h"], cfgd["f"], cfgd["E"], cfgd["k"], cfgd["act"]
    x, wr, w1, w2, dy = _inputs(T * world, h, f, E, 0)
    sl = slice(rank * T, (rank + 1) * T)
    e0, e1 = ep.local_expert_range(rank, world, E)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a))  # noqa: E731
    layer = ep.ExpertParallelMoE(B, dist.group.WORLD, h, E, k, f, act=act, block_size=4,
                                 renormalize=cfgd.get("renorm", False), aux_loss_coeff=cfgd.get("aux", 0.0))
    xl, dyl = t(x[sl]), t(dy[sl])
    w1l, w2l = t(w1[:, e0 * f:e1 * f]), t(w2[e0 * f:e1 * f])
    y, st = layer.forward(xl, t(wr), w1l, w2l)
    dx, dwr, dw1, dw2 = layer.backward(st, xl, dyl, t(wr), w1l, w2l)
    aux = float(layer.aux_loss.item()) if layer.aux_loss is not None else 0.0
    q.put((rank, y.numpy(), dx.numpy(), dwr.numpy(), dw1.numpy(), dw2.numpy(), aux))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfgd", [dict(T=24, h=6, f=8, E=4, k=1, act=1), dict(T=17, h=4, f=4, E=6, k=2, act=2),
                                  dict(T=9, h=4, f=4, E=2, k=1, act=0), dict(T=15, h=4, f=4, E=4, k=2, act=1, renorm=True),
                                  dict(T=16, h=4, f=4, E=4, k=1, act=1, aux=0.05)])
def test_ep_world2_matches_global_oracle(cfgd):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfgd, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=120)
        res[r[0]] = r[1:]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    T, h, f, E, k, act = cfgd["T"], cfgd["h"], cfgd["f"], cfgd["E"], cfgd["k"], cfgd["act"]
    x, wr, w1, w2, dy = _inputs(T * world, h, f, E, 0)
    y, cache = O.dmoe_forward(x, wr, w1, w2, k, 4, f, act, renormalize=cfgd.get("renorm", False))
    g = O.dmoe_backward(cache, dy, wr, w1, w2)
    El = E // world
    coeff = cfgd.get("aux", 0.0)
    # the auxiliary loss is per rank's tokens (DP micro-batches): its router
    # gradient adds, per rank, p*(c - <p,c>) on that rank's rows; dWr sums them
    aux_dl = np.zeros_like(cache.logits)
    aux_loss = []
    if coeff:
        for r in range(world):
            sl = slice(r * T, (r + 1) * T)
            p = cache.probs[sl]
            loss_r, dprobs = O.load_balance_loss(p, cache.expert_idx[sl], coeff)
            aux_loss.append(loss_r)
            aux_dl[sl] = p * (dprobs - (p * dprobs).sum(1, keepdims=True))
    dx_want = g["dx"] + aux_dl @ wr.T
    dwr_want = g["dwr"] + x.T @ aux_dl
    for r in range(world):
        yr, dxr, dwrr, dw1r, dw2r, auxr = res[r]
        if coeff:
            assert abs(auxr - aux_loss[r]) < 1e-10
        sl = slice(r * T, (r + 1) * T)
        np.testing.assert_allclose(yr, y[sl], atol=1e-10)
        np.testing.assert_allclose(dxr, dx_want[sl], atol=1e-10)
        np.testing.assert_allclose(dwrr, dwr_want, atol=1e-10)
        np.testing.assert_allclose(dw1r, g["dw1"][:, r * El * f:(r + 1) * El * f], atol=1e-10)
        np.testing.assert_allclose(dw2r, g["dw2"][r * El * f:(r + 1) * El * f], atol=1e-10)


def test_split_helpers():
    from paper_2211_15841_b200 import ep
    counts = np.array([[3, 0, 2, 1], [1, 4, 0, 0]])
    assert ep.send_splits(counts[0], 2) == [3, 3]
    assert ep.send_splits(counts[1], 2) == [5, 0]
    splits, ids = ep.recv_plan(counts, 1, 2)
    assert splits == [3, 0]
    assert ids.tolist() == [0, 0, 1]
    splits, ids = ep.recv_plan(counts, 0, 2)
    assert splits == [3, 5] and ids.tolist() == [0, 0, 0, 0, 1, 1, 1, 1]
    with pytest.raises(ValueError):
        ep.local_expert_range(0, 3, 4)
