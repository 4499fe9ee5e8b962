"""Pins for the CPU oracle (oracle/moe_oracle.py) — no GPU needed.

Each test pins the oracle to something other than itself: the paper's / SPEC's
worked examples (tests/golden/*, each citing its source), closed forms,
invariants, brute force on tiny inputs, and three independent formulations of
the layer written here in plain torch float64 (dense all-experts-then-mask,
token dropping at capacity factor E with batched matmul, per-expert loop),
plus finite differences and torch.autograd for the backward pass.
"""
import itertools
import math

import numpy as np
import pytest
import torch

from conftest import golden_kv, read_golden
from oracle import moe_oracle as O
from synth import inputs as S


def nums(vals, t=float):
    return [t(v) for v in vals]


# ---------------------------------------------------------------- golden pins

def test_softmax_golden():
    g = golden_kv("softmax_S49.txt")
    p = O.softmax(np.array([nums(g["input"])]))
    np.testing.assert_allclose(p[0], nums(g["output"]), atol=1e-8)


def test_softmax_shift_invariance_and_rows_sum_to_one():
    rng = np.random.default_rng(0)
    L = rng.normal(size=(16, 7))
    p = O.softmax(L)
    np.testing.assert_allclose(p.sum(1), 1.0, atol=1e-12)
    np.testing.assert_allclose(O.softmax(L + 3.5), p, atol=1e-12)
    assert (p >= 0).all()


def test_router_golden():
    for line in read_golden("router_S267.txt"):
        logits, k, idx, gate = [s.strip() for s in line.split("|")]
        L = np.array([nums(logits.split())])
        i, g = O.topk(L, int(k))
        assert i[0, 0] == int(idx)
        assert abs(g[0, 0] - float(gate)) < 1e-8


def test_topk_brute_force_with_ties():
    # brute force: enumerate all k-subsets ordered by (-score, index) lexicographically
    rng = np.random.default_rng(1)
    for trial in range(200):
        E = int(rng.integers(1, 7))
        k = int(rng.integers(1, E + 1))
        L = rng.integers(0, 3, size=(1, E)).astype(np.float64)  # many exact ties
        best = None
        for combo in itertools.permutations(range(E), k):
            key = [(-L[0, e], e) for e in combo]
            if key != sorted(key):
                continue
            score = sorted(((-L[0, e], e) for e in combo))
            rest = sorted((-L[0, e], e) for e in range(E) if e not in combo)
            if rest and score[-1] > rest[0]:
                continue  # a better candidate was left out
            best = list(combo)
        idx, gates = O.topk(L, k)
        assert list(idx[0]) == best, (L, k)
        np.testing.assert_allclose(gates[0], O.softmax(L)[0, best], atol=0)


def test_topk_single_expert_gate_is_one():
    idx, g = O.topk(np.random.default_rng(2).normal(size=(5, 1)), 1)
    assert (idx == 0).all() and np.allclose(g, 1.0)


def test_plan_golden():
    g = golden_kv("plan_S287.txt")
    counts, bs = nums(g["counts"], int), int(g["block"][0])
    idx = np.repeat(np.arange(len(counts)), counts).astype(np.int32)
    plan = O.make_plan(idx, len(counts), bs)
    assert list(plan.padded_counts) == nums(g["padded_counts"], int)
    assert plan.Tp == int(g["total"][0])
    assign = np.array(nums(g["assign"], int), np.int32)
    p2 = O.make_plan(assign, 2, 4)
    assert list(p2.sorted_idx) == nums(g["gather_order"], int)


def test_bcsr_golden():
    g = golden_kv("bcsr_S114.txt")
    nbr, nbc = nums(g["grid"], int)
    blocks = [tuple(map(int, b.split(","))) for b in g["blocks"]]
    t = O.topology_from_blocks(blocks, nbr, nbc, 1)
    for key in ["row_offsets", "col_indices", "row_indices", "t_col_offsets",
                "t_block_offsets", "t_row_indices"]:
        assert list(getattr(t, key)) == nums(g[key], int), key


def test_bcsr_empty():
    t = O.topology_from_blocks([], 3, 2, 4)
    assert t.nnz == 0 and list(t.row_offsets) == [0, 0, 0, 0] and list(t.t_col_offsets) == [0, 0, 0]


def test_moe_topology_golden():
    g = golden_kv("moe_topology_S317.txt")
    counts = nums(g["counts"], int)
    bs, ffn = int(g["block"][0]), int(g["ffn"][0])
    idx = np.repeat(np.arange(len(counts)), counts).astype(np.int32)
    plan = O.make_plan(idx, len(counts), bs)
    blocks = sorted(tuple(map(int, b.split(","))) for b in g["blocks"])
    assert sorted(O.moe_topology_blocks(plan, bs, ffn)) == blocks
    for topo in (O.make_topology(plan, bs, ffn), O.make_topology_closed_form(plan, bs, ffn)):
        for key in ["row_offsets", "col_indices", "row_indices", "t_col_offsets",
                    "t_block_offsets", "t_row_indices"]:
            assert list(getattr(topo, key)) == nums(g[key], int), key


def test_gelu_golden_and_derivative():
    for line in read_golden("gelu_S58.txt"):
        kind, x, want, tol = line.split()
        kid = {"gelu": O.ACT_GELU, "relu": O.ACT_RELU}[kind]
        assert abs(O.act(kid, np.array([float(x)]))[0] - float(want)) <= float(tol)
    xs = np.array([-1.0, 0.5, 2.0, -3.0, 0.1])
    eps = 1e-6
    for kid in (O.ACT_IDENTITY, O.ACT_GELU, O.ACT_RELU):
        fd = (O.act(kid, xs + eps) - O.act(kid, xs - eps)) / (2 * eps)
        np.testing.assert_allclose(O.act_grad(kid, xs), fd, rtol=1e-6, atol=1e-8)


def test_capacity_golden():
    for line in read_golden("capacity_P115.txt"):
        T, E, cf, cap = line.split()
        assert O.expert_capacity(int(T), int(E), float(cf)) == int(cap)


# ---------------------------------------------------------------- invariants

def to_dense(vals, topo):
    bs = topo.bs
    d = np.zeros((topo.n_block_rows * bs, topo.n_block_cols * bs))
    for s in range(topo.nnz):
        r, c = topo.row_indices[s], topo.col_indices[s]
        d[r * bs:(r + 1) * bs, c * bs:(c + 1) * bs] = vals[s]
    return d


def mask_of(topo):
    return to_dense(np.ones((topo.nnz, topo.bs, topo.bs)), topo)


def random_topology(rng, max_grid=6, bs=None):
    nbr, nbc = int(rng.integers(1, max_grid + 1)), int(rng.integers(1, max_grid + 1))
    bs = bs or int(rng.choice([1, 2, 3, 4]))
    dens = rng.uniform(0, 1)
    coords = [(r, c) for r in range(nbr) for c in range(nbc) if rng.uniform() < dens]
    return O.topology_from_blocks(coords, nbr, nbc, bs)


def test_transpose_index_equals_explicit_transpose_200_topologies():
    rng = np.random.default_rng(3)
    for _ in range(200):
        t = random_topology(rng)
        vals = rng.normal(size=(t.nnz, t.bs, t.bs))
        dense_t = to_dense(vals, t).T
        # rebuild the transposed matrix only through the transpose index
        bs = t.bs
        d2 = np.zeros((t.n_block_cols * bs, t.n_block_rows * bs))
        for c in range(t.n_block_cols):
            for i in range(t.t_col_offsets[c], t.t_col_offsets[c + 1]):
                b, r = t.t_block_offsets[i], t.t_row_indices[i]
                d2[c * bs:(c + 1) * bs, r * bs:(r + 1) * bs] = vals[b].T
        np.testing.assert_array_equal(d2, dense_t)
        assert sorted(t.t_block_offsets.tolist()) == list(range(t.nnz))
        assert t.row_offsets[-1] == t.nnz == t.t_col_offsets[-1]


def test_moe_closed_form_equals_generic_random_plans():
    rng = np.random.default_rng(4)
    for _ in range(200):
        E = int(rng.integers(1, 7))
        bs = int(rng.choice([1, 2, 4]))
        F = int(rng.integers(1, 4))
        T = int(rng.integers(0, 30))
        k = int(rng.integers(1, E + 1))
        idx = np.stack([rng.permutation(E)[:k] for _ in range(T)]) if T else np.zeros((0, k), np.int32)
        plan = O.make_plan(idx, E, bs)
        a = O.make_topology(plan, bs, F * bs)
        b = O.make_topology_closed_form(plan, bs, F * bs)
        for key in ["row_offsets", "col_indices", "row_indices", "t_col_offsets",
                    "t_block_offsets", "t_row_indices"]:
            np.testing.assert_array_equal(getattr(a, key), getattr(b, key), err_msg=key)
        # plan invariants
        assert plan.counts.sum() == T * k
        assert plan.Tp == plan.padded_bins[-1]
        assert a.nnz == (plan.Tp // bs) * F
        assert (plan.padded_counts % bs == 0).all()
        assert ((plan.padded_counts == 0) == (plan.counts == 0)).all()
        assert plan.Tp <= O.max_padded_rows(T, k, E, bs) or T == 0


def test_plan_positions_stable_and_padding_at_tail():
    rng = np.random.default_rng(5)
    idx = rng.integers(0, 5, size=(40, 1)).astype(np.int32)
    plan = O.make_plan(idx, 5, 4)
    start = plan.padded_bins - plan.padded_counts
    for e in range(5):
        ids = [i for i in range(40) if idx[i, 0] == e]
        assert [plan.pos[i] for i in ids] == list(range(start[e], start[e] + len(ids)))
    x = rng.normal(size=(40, 3))
    xg = O.padded_gather(x, plan, 1)
    real = set(plan.pos.tolist())
    for p in range(plan.Tp):
        if p not in real:
            assert (xg[p] == 0).all()          # pad rows exactly zero
    y = O.padded_scatter(xg, plan, np.ones((40, 1)), 40, 1)
    np.testing.assert_array_equal(y, x)        # round trip with unit gates


def test_scatter_topk2_weighted_sum():
    # S:308 / P:157: g1*y1 + g2*y2
    idx = np.array([[0, 1]], np.int32)
    plan = O.make_plan(idx, 2, 1)
    yg = np.array([[1.0, 2.0], [10.0, 20.0]])
    y = O.padded_scatter(yg, plan, np.array([[0.25, 0.75]]), 1, 2)
    np.testing.assert_allclose(y, [[0.25 * 1 + 0.75 * 10, 0.25 * 2 + 0.75 * 20]])


# ---------------------------------------------------------------- products vs densify

@pytest.mark.parametrize("seed", range(60))
def test_products_match_densify_oracle(seed):
    rng = np.random.default_rng(100 + seed)
    t = random_topology(rng, max_grid=5)
    bs = t.bs
    M, N = t.n_block_rows * bs, t.n_block_cols * bs
    K = int(rng.integers(1, 7))
    vals = rng.normal(size=(t.nnz, bs, bs))
    S_d = to_dense(vals, t)
    mask = mask_of(t)
    a, b = rng.normal(size=(M, K)), rng.normal(size=(K, N))
    # SDD, with transposed operands
    np.testing.assert_allclose(to_dense(O.sdd(a, b, t), t), (a @ b) * mask, atol=1e-12)
    np.testing.assert_allclose(to_dense(O.sdd(a.T.copy(), b, t, trans_a=True), t), (a @ b) * mask, atol=1e-12)
    np.testing.assert_allclose(to_dense(O.sdd(a, b.T.copy(), t, trans_b=True), t), (a @ b) * mask, atol=1e-12)
    # DSD, DSD^T-style (dense operand transposed), DS^TD
    bn = rng.normal(size=(N, K))
    np.testing.assert_allclose(O.dsd(vals, bn, t), S_d @ bn, atol=1e-12)
    np.testing.assert_allclose(O.dsd(vals, bn.T.copy(), t, trans_b=True), S_d @ bn, atol=1e-12)
    bm = rng.normal(size=(M, K))
    np.testing.assert_allclose(O.dsd(vals, bm, t, trans_s=True), S_d.T @ bm, atol=1e-12)
    # DDS, DD^TS, DDS^T
    am = rng.normal(size=(K, M))
    np.testing.assert_allclose(O.dds(am, vals, t), am @ S_d, atol=1e-12)
    np.testing.assert_allclose(O.dds(am.T.copy(), vals, t, trans_a=True), am @ S_d, atol=1e-12)
    an = rng.normal(size=(K, N))
    np.testing.assert_allclose(O.dds(an, vals, t, trans_s=True), an @ S_d.T, atol=1e-12)


def test_sdd_dense_limit_and_work_count():
    rng = np.random.default_rng(6)
    bs, nbr, nbc, K = 2, 3, 4, 5
    t = O.topology_from_blocks([(r, c) for r in range(nbr) for c in range(nbc)], nbr, nbc, bs)
    a, b = rng.normal(size=(nbr * bs, K)), rng.normal(size=(K, nbc * bs))
    np.testing.assert_allclose(to_dense(O.sdd(a, b, t), t), a @ b, atol=1e-12)


# ---------------------------------------------------------------- independent layer formulations (torch fp64)

def t64(a):
    return torch.tensor(np.asarray(a), dtype=torch.float64)


def torch_act(kind, h):
    if kind == O.ACT_IDENTITY:
        return h
    if kind == O.ACT_RELU:
        return torch.relu(h)
    return torch.nn.functional.gelu(h, approximate="tanh")


def dense_masked_moe(x, wr, w1, w2, k, f, act_kind):
    """Formulation (i): every expert computes every token, then mask by routing."""
    L = x @ wr
    p = torch.softmax(L, dim=1)
    idx = torch.topk(L, k, dim=1).indices
    E = wr.shape[1]
    y = torch.zeros_like(x)
    for e in range(E):
        ye = torch_act(act_kind, x @ w1[:, e * f:(e + 1) * f]) @ w2[e * f:(e + 1) * f]
        sel = (idx == e).any(dim=1).to(x.dtype)
        y = y + (sel * p[:, e])[:, None] * ye
    return y, idx


def dropping_moe_cf(x, wr, w1, w2, k, f, act_kind, cf):
    """Formulation (ii): token-dropping MoE with capacity
    num_tokens/num_experts*cf, keep-earliest, batched matmul over experts
    (Fig. 3A). With cf = E nothing is dropped."""
    T, h = x.shape
    E = wr.shape[1]
    C = O.expert_capacity(T, E, cf)
    L = x @ wr
    p = torch.softmax(L, dim=1)
    idx = torch.topk(L, k, dim=1).indices
    xb = torch.zeros(E, C, h, dtype=x.dtype)
    slot = {}
    fill = [0] * E
    for t in range(T):
        for j in range(k):
            e = int(idx[t, j])
            if fill[e] < C:
                slot[(t, j)] = (e, fill[e])
                xb[e, fill[e]] = x[t]
                fill[e] += 1
    W1 = torch.stack([w1[:, e * f:(e + 1) * f] for e in range(E)])
    W2 = torch.stack([w2[e * f:(e + 1) * f] for e in range(E)])
    yb = torch.bmm(torch_act(act_kind, torch.bmm(xb, W1)), W2)
    y = torch.zeros_like(x)
    for (t, j), (e, c) in slot.items():
        y[t] += p[t, e] * yb[e, c]
    return y, len(slot)


def per_expert_loop(x, wr, w1, w2, k, f, act_kind):
    """Formulation (iii): loop over experts, each on exactly its own tokens."""
    L = x @ wr
    p = torch.softmax(L, dim=1)
    idx = torch.topk(L, k, dim=1).indices
    y = torch.zeros_like(x)
    for e in range(wr.shape[1]):
        rows, slots = torch.nonzero(idx == e, as_tuple=True)
        if rows.numel() == 0:
            continue
        ye = torch_act(act_kind, x[rows] @ w1[:, e * f:(e + 1) * f]) @ w2[e * f:(e + 1) * f]
        y.index_add_(0, rows, p[rows, e][:, None] * ye)
    return y


SMALL = [
    # T, h, f, E, k, bs, act
    (40, 8, 8, 4, 1, 4, O.ACT_GELU),
    (33, 6, 6, 3, 2, 2, O.ACT_RELU),
    (25, 4, 8, 5, 3, 4, O.ACT_IDENTITY),
    (64, 16, 8, 8, 2, 8, O.ACT_GELU),
    (7, 4, 4, 1, 1, 4, O.ACT_GELU),
]


def small_inputs(T, h, f, E, seed):
    rng = np.random.default_rng(seed)
    return (rng.normal(size=(T, h)), rng.normal(size=(h, E)) / math.sqrt(h),
            rng.normal(size=(h, E * f)) / math.sqrt(h), rng.normal(size=(E * f, h)) / math.sqrt(f),
            rng.normal(size=(T, h)))


@pytest.mark.parametrize("cfg", SMALL)
def test_layer_forward_three_formulations(cfg):
    T, h, f, E, k, bs, a = cfg
    x, wr, w1, w2, _ = small_inputs(T, h, f, E, 7)
    y, cache = O.dmoe_forward(x, wr, w1, w2, k, bs, f, a)
    y_i, idx_i = dense_masked_moe(t64(x), t64(wr), t64(w1), t64(w2), k, f, a)
    assert (idx_i.numpy() == cache.expert_idx).all()
    np.testing.assert_allclose(y, y_i.numpy(), atol=1e-11)
    y_ii, kept = dropping_moe_cf(t64(x), t64(wr), t64(w1), t64(w2), k, f, a, cf=E)
    assert kept == T * k                         # cf = E drops nothing
    np.testing.assert_allclose(y, y_ii.numpy(), atol=1e-11)
    y_iii = per_expert_loop(t64(x), t64(wr), t64(w1), t64(w2), k, f, a)
    np.testing.assert_allclose(y, y_iii.numpy(), atol=1e-11)


def test_dropping_cf1_drops_one_minus_one_over_E():
    # 8 tokens all to expert 0 of 4 experts, cf 1 -> capacity 2, drop 6/8
    T, h, f, E = 8, 4, 4, 4
    x = np.ones((T, h))
    wr = np.zeros((h, E)); wr[:, 0] = 1.0
    w1 = np.random.default_rng(0).normal(size=(h, E * f))
    w2 = np.random.default_rng(1).normal(size=(E * f, h))
    _, kept = dropping_moe_cf(t64(x), t64(wr), t64(w1), t64(w2), 1, f, O.ACT_GELU, cf=1.0)
    assert 1 - kept / T == 1 - 1 / E


def test_single_expert_is_dense_mlp():
    T, h, f = 9, 4, 8
    x, wr, w1, w2, _ = small_inputs(T, h, f, 1, 8)
    y, _ = O.dmoe_forward(x, wr, w1, w2, 1, 4, f, O.ACT_IDENTITY)
    np.testing.assert_allclose(y, (x @ w1) @ w2, atol=1e-12)


def test_uniform_routing_equals_bmm():
    # exact-uniform routing, count multiple of bs -> block-sparse == batched matmul (A5)
    T, h, f, E, bs = 32, 8, 8, 4, 4
    x, wr, w1, w2, _ = small_inputs(T, h, f, E, 9)
    idx = S.uniform_expert_idx(T, E, 1).numpy()
    plan = O.make_plan(idx, E, bs)
    topo = O.make_topology(plan, bs, f)
    xg = O.padded_gather(x, plan, 1)
    assert plan.Tp == T                          # no padding under exact-uniform routing
    hs = O.sdd(xg, w1, topo)
    xb = t64(xg).reshape(E, T // E, h)
    W1 = torch.stack([t64(w1)[:, e * f:(e + 1) * f] for e in range(E)])
    hb = torch.bmm(xb, W1).numpy()
    # block (r, e*F+j) of the SDD = rows r*bs.. of expert e's batched product, cols j*bs..
    F = f // bs
    for s in range(topo.nnz):
        r, c = topo.row_indices[s], topo.col_indices[s]
        e, j = c // F, c % F
        rr = r * bs - e * (T // E)
        np.testing.assert_allclose(hs[s], hb[e, rr:rr + bs, j * bs:(j + 1) * bs], atol=1e-12)


@pytest.mark.parametrize("cfg", SMALL)
def test_layer_backward_vs_autograd(cfg):
    T, h, f, E, k, bs, a = cfg
    x, wr, w1, w2, dy = small_inputs(T, h, f, E, 10)
    y, cache = O.dmoe_forward(x, wr, w1, w2, k, bs, f, a)
    g = O.dmoe_backward(cache, dy, wr, w1, w2)
    tx, twr, tw1, tw2 = (t64(v).requires_grad_() for v in (x, wr, w1, w2))
    yt, _ = dense_masked_moe(tx, twr, tw1, tw2, k, f, a)
    (yt * t64(dy)).sum().backward()
    np.testing.assert_allclose(g["dx"], tx.grad.numpy(), atol=1e-10)
    np.testing.assert_allclose(g["dwr"], twr.grad.numpy(), atol=1e-10)
    np.testing.assert_allclose(g["dw1"], tw1.grad.numpy(), atol=1e-10)
    np.testing.assert_allclose(g["dw2"], tw2.grad.numpy(), atol=1e-10)


def test_layer_backward_finite_differences():
    T, h, f, E, k, bs, a = 12, 4, 4, 3, 2, 2, O.ACT_GELU
    x, wr, w1, w2, dy = small_inputs(T, h, f, E, 11)
    _, cache = O.dmoe_forward(x, wr, w1, w2, k, bs, f, a)
    g = O.dmoe_backward(cache, dy, wr, w1, w2)
    eps = 1e-6

    def loss(x_, wr_, w1_, w2_):
        y_, c_ = O.dmoe_forward(x_, wr_, w1_, w2_, k, bs, f, a)
        assert (c_.expert_idx == cache.expert_idx).all()
        return float((y_ * dy).sum())

    rng = np.random.default_rng(12)
    for name, arr, pos in [("dw1", w1, 0), ("dw2", w2, 1), ("dwr", wr, 2), ("dx", x, 3)]:
        for _ in range(6):
            i = tuple(int(rng.integers(0, n)) for n in arr.shape)
            args = [w1, w2, wr, x]
            plus = [v.copy() for v in args]; plus[pos][i] += eps
            minus = [v.copy() for v in args]; minus[pos][i] -= eps
            fd = (loss(plus[3], plus[2], plus[0], plus[1]) - loss(minus[3], minus[2], minus[0], minus[1])) / (2 * eps)
            assert abs(fd - g[name][i]) < 1e-6 * max(1.0, abs(fd)), (name, i, fd, g[name][i])


def test_max_padded_rows_bound_is_tight():
    # all experts get exactly one assignment -> every group pads to bs
    T, k, E, bs = 8, 1, 8, 4
    idx = np.arange(8).reshape(8, 1).astype(np.int32)
    plan = O.make_plan(idx, E, bs)
    assert plan.Tp == O.max_padded_rows(T, k, E, bs) == 32


def test_product_sweep_layout_conversion():
    """scripts/product_sweep.py compares the library's BCSR values with torch.bmm
    through blocks_to_dense / dense_to_blocks; pin both against the oracle's SDD
    under exact-uniform routing (block (r, e*F+j) = rows r*bs.. of expert e's
    batched product, columns j*bs..)."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "product_sweep", os.path.join(os.path.dirname(__file__), "..", "scripts", "product_sweep.py"))
    ps = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(ps)
    T, h, f, E, bs = 512, 8, 256, 2, 128
    x, wr, w1, w2, _ = small_inputs(T, h, f, E, 5)
    idx = S.uniform_expert_idx(T, E, 1).numpy()
    plan = O.make_plan(idx, E, bs)
    topo = O.make_topology(plan, bs, f)
    hs = O.sdd(O.padded_gather(x, plan, 1), w1, topo)
    dense = ps.blocks_to_dense(torch.from_numpy(hs), E, T // E, f, bs)
    want = torch.bmm(t64(x).reshape(E, T // E, h), torch.stack([t64(w1)[:, e * f:(e + 1) * f] for e in range(E)]))
    np.testing.assert_allclose(dense.numpy(), want.numpy(), atol=1e-12)
    np.testing.assert_array_equal(ps.dense_to_blocks(dense, E, T // E, f, bs).numpy(), hs)


# ------------------------------------------------------------------ token-dropping formulation (NEXT-4)

def test_capacity_plan_spec_example_keep_earliest():
    # 8 tokens all to expert 0 of 4 experts, cf 1 -> capacity 2: tokens 2..7 dropped
    idx = np.zeros((8, 1), np.int64)
    C = O.expert_capacity(8, 4, 1.0)
    assert C == 2
    plan = O.make_plan(idx, 4, 4, capacity=C)
    assert plan.dropped.tolist() == [False, False] + [True] * 6
    assert plan.counts.tolist() == [2, 0, 0, 0] and plan.Tp == 4
    assert plan.pos.tolist() == [0, 1] + [-1] * 6
    assert plan.sorted_idx.tolist() == [0, 1]


def test_capacity_large_enough_equals_dropless():
    # no expert overflows -> identical to the dropless plan and layer, bit for bit
    T, h, f, E, k = 40, 8, 8, 4, 2
    x, wr, w1, w2, dy = small_inputs(T, h, f, E, 11)
    y0, c0 = O.dmoe_forward(x, wr, w1, w2, k, 4, f, O.ACT_GELU)
    y1, c1 = O.dmoe_forward(x, wr, w1, w2, k, 4, f, O.ACT_GELU, capacity=int(c0.plan.counts.max()))
    np.testing.assert_array_equal(c0.plan.pos, c1.plan.pos)
    np.testing.assert_array_equal(y0, y1)
    g0, g1 = O.dmoe_backward(c0, dy, wr, w1, w2), O.dmoe_backward(c1, dy, wr, w1, w2)
    for n in ("dx", "dwr", "dw1", "dw2"):
        np.testing.assert_array_equal(g0[n], g1[n])


@pytest.mark.parametrize("T,h,f,E,k,cf", [(32, 6, 8, 4, 1, 1.0), (30, 4, 8, 4, 2, 1.5), (24, 8, 4, 3, 1, 0.5)])
def test_capacity_layer_equals_batched_dropping_moe_and_autograd(T, h, f, E, k, cf):
    """The block-sparse layer with a capacity (make_plan keep-earliest, pos = -1
    for dropped slots) against formulation (ii), the batched-matmul token-dropping
    MoE (Fig. 3A), forward and — through torch autograd of (ii) —
    every gradient."""
    x, wr, w1, w2, dy = small_inputs(T, h, f, E, 13)
    C = O.expert_capacity(T, E, cf)
    y, cache = O.dmoe_forward(x, wr, w1, w2, k, 4, f, O.ACT_GELU, capacity=C)
    assert cache.plan.dropped.any()                      # the case really drops
    tx, twr, tw1, tw2 = (t64(a).requires_grad_(True) for a in (x, wr, w1, w2))
    yt, kept = dropping_moe_cf(tx, twr, tw1, tw2, k, f, O.ACT_GELU, cf)
    assert kept == int((~cache.plan.dropped).sum())
    np.testing.assert_allclose(y, yt.detach().numpy(), atol=1e-10)
    (yt * t64(dy)).sum().backward()
    g = O.dmoe_backward(cache, dy, wr, w1, w2)
    np.testing.assert_allclose(g["dx"], tx.grad.numpy(), atol=1e-10)
    np.testing.assert_allclose(g["dwr"], twr.grad.numpy(), atol=1e-10)
    np.testing.assert_allclose(g["dw1"], tw1.grad.numpy(), atol=1e-10)
    np.testing.assert_allclose(g["dw2"], tw2.grad.numpy(), atol=1e-10)


# ------------------------------------------------------------------ top-k gate renormalisation (NEXT-4)

def test_renormalized_gates_invariants():
    # gates in (0, 1]; k = E with renormalisation -> each token's gates sum to 1; k = 1 -> gate 1
    rng = np.random.default_rng(5)
    L = rng.normal(size=(50, 6))
    _, g = O.topk(L, 6, renormalize=True)
    np.testing.assert_allclose(g.sum(axis=1), 1.0, atol=1e-12)
    _, g1 = O.topk(L, 1, renormalize=True)
    np.testing.assert_array_equal(g1, np.ones((50, 1)))
    idx, g3 = O.topk(L, 3, renormalize=True)
    _, raw = O.topk(L, 3)
    np.testing.assert_allclose(g3, raw / raw.sum(axis=1, keepdims=True), atol=1e-15)
    assert (g3 > 0).all() and (g3 <= 1).all()


@pytest.mark.parametrize("T,h,f,E,k", [(20, 6, 8, 4, 2), (17, 4, 4, 5, 3), (12, 5, 8, 3, 1)])
def test_renormalized_layer_backward_vs_autograd(T, h, f, E, k):
    """Formulation (i) with renormalised gates (every expert on every token,
    masked, weight p_e / sum of the chosen p) under torch autograd against the
    oracle layer with renormalize=True, forward and every gradient."""
    x, wr, w1, w2, dy = small_inputs(T, h, f, E, 17)
    y, cache = O.dmoe_forward(x, wr, w1, w2, k, 4, f, O.ACT_GELU, renormalize=True)
    g = O.dmoe_backward(cache, dy, wr, w1, w2)
    tx, twr, tw1, tw2 = (t64(a).requires_grad_(True) for a in (x, wr, w1, w2))
    L = tx @ twr
    p = torch.softmax(L, dim=1)
    idx = torch.topk(L, k, dim=1).indices
    sel = torch.zeros_like(p).scatter(1, idx, 1.0)
    wsel = p * sel
    wsel = wsel / wsel.sum(dim=1, keepdim=True)
    yt = torch.zeros_like(tx)
    for e in range(E):
        ye = torch_act(O.ACT_GELU, tx @ tw1[:, e * f:(e + 1) * f]) @ tw2[e * f:(e + 1) * f]
        yt = yt + wsel[:, e:e + 1] * ye
    np.testing.assert_allclose(y, yt.detach().numpy(), atol=1e-10)
    (yt * t64(dy)).sum().backward()
    np.testing.assert_allclose(g["dx"], tx.grad.numpy(), atol=1e-10)
    np.testing.assert_allclose(g["dwr"], twr.grad.numpy(), atol=1e-10)
    np.testing.assert_allclose(g["dw1"], tw1.grad.numpy(), atol=1e-10)
    np.testing.assert_allclose(g["dw2"], tw2.grad.numpy(), atol=1e-10)


# ------------------------------------------------------------------ auxiliary load-balancing loss (NEXT-4)

def test_load_balance_loss_closed_forms():
    # uniform f and P -> loss = coefficient; all tokens to one expert with prob 1 -> coefficient * E
    E, T = 4, 8
    p = np.full((T, E), 1.0 / E)
    idx = np.array([[t % E] for t in range(T)])
    assert abs(O.load_balance_loss(p, idx, 0.3)[0] - 0.3) < 1e-15
    p1 = np.zeros((T, E)); p1[:, 2] = 1.0
    assert abs(O.load_balance_loss(p1, np.full((T, 1), 2), 0.3)[0] - 0.3 * E) < 1e-15


def test_load_balance_loss_grad_finite_differences_and_layer_autograd():
    # d loss / d probs by finite differences (f held fixed); then the layer's
    # dlogits / dWr / dx with the aux term against torch autograd of the masked formulation
    rng = np.random.default_rng(3)
    T, E = 6, 5
    p = rng.random((T, E)); p /= p.sum(1, keepdims=True)
    idx = p.argmax(1)[:, None]
    loss, g = O.load_balance_loss(p, idx, 0.7)
    eps = 1e-6
    for t in range(T):
        for e in range(E):
            q = p.copy(); q[t, e] += eps
            fd = (O.load_balance_loss(q, idx, 0.7)[0] - loss) / eps
            assert abs(fd - g[t, e]) <= 1e-6 * max(1.0, abs(g[t, e]))
    T, h, f, E, k = 16, 6, 8, 4, 2
    x, wr, w1, w2, dy = small_inputs(T, h, f, E, 23)
    y, cache = O.dmoe_forward(x, wr, w1, w2, k, 4, f, O.ACT_GELU, aux_coeff=0.05)
    gr = O.dmoe_backward(cache, dy, wr, w1, w2)
    tx, twr, tw1, tw2 = (t64(a).requires_grad_(True) for a in (x, wr, w1, w2))
    L = tx @ twr
    pt = torch.softmax(L, dim=1)
    ti = torch.topk(L, k, dim=1).indices
    fe = torch.bincount(ti[:, 0], minlength=E).double() / T           # constant (no gradient)
    aux = 0.05 * E * (fe * pt.mean(0)).sum()
    assert abs(aux.item() - cache.aux_loss) < 1e-12
    yt = torch.zeros_like(tx)
    for e in range(E):
        ye = torch_act(O.ACT_GELU, tx @ tw1[:, e * f:(e + 1) * f]) @ tw2[e * f:(e + 1) * f]
        sel = (ti == e).any(dim=1).double()
        yt = yt + (sel * pt[:, e])[:, None] * ye
    ((yt * t64(dy)).sum() + aux).backward()
    np.testing.assert_allclose(gr["dx"], tx.grad.numpy(), atol=1e-10)
    np.testing.assert_allclose(gr["dwr"], twr.grad.numpy(), atol=1e-10)


@pytest.mark.parametrize("T,h,f,E,k,renorm", [(24, 6, 8, 4, 2, False), (19, 4, 4, 5, 3, True), (16, 5, 8, 3, 1, False)])
def test_forward_given_expert_idx_vs_autograd(T, h, f, E, k, renorm):
    """dmoe_forward(expert_idx=...) (R6: a test resolving a near-tie token the
    other valid way) with an arbitrary, non-greedy choice of distinct experts:
    y[t] = sum_j g[t,j] act(x_t W1_e) W2_e with g = softmax(x Wr)[t, e_j]
    (renormalised over the k if asked), written per token in torch; and its
    backward against torch autograd of that formulation (the routing is a
    constant, the gates carry the router gradient)."""
    x, wr, w1, w2, dy = small_inputs(T, h, f, E, 13)
    rng = np.random.default_rng(5)
    idx = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
    y, cache = O.dmoe_forward(x, wr, w1, w2, k, 4, f, O.ACT_GELU, renormalize=renorm, expert_idx=idx)
    assert (cache.expert_idx == idx).all()
    g = O.dmoe_backward(cache, dy, wr, w1, w2)
    tx, twr, tw1, tw2 = (t64(v).requires_grad_() for v in (x, wr, w1, w2))
    p = torch.softmax(tx @ twr, dim=1)
    rows = []
    for t in range(T):
        gs = torch.stack([p[t, int(e)] for e in idx[t]])
        if renorm:
            gs = gs / gs.sum()
        yt = torch.zeros(h, dtype=torch.float64)
        for j, e in enumerate(idx[t]):
            e = int(e)
            yt = yt + gs[j] * (torch_act(O.ACT_GELU, tx[t] @ tw1[:, e * f:(e + 1) * f]) @ tw2[e * f:(e + 1) * f])
        rows.append(yt)
    yt = torch.stack(rows)
    np.testing.assert_allclose(y, yt.detach().numpy(), atol=1e-12)
    (yt * t64(dy)).sum().backward()
    np.testing.assert_allclose(g["dx"], tx.grad.numpy(), atol=1e-10)
    np.testing.assert_allclose(g["dwr"], twr.grad.numpy(), atol=1e-10)
    np.testing.assert_allclose(g["dw1"], tw1.grad.numpy(), atol=1e-10)
    np.testing.assert_allclose(g["dw2"], tw2.grad.numpy(), atol=1e-10)


@pytest.mark.parametrize("seed", range(40))
def test_fringe_rows_link_padded_and_unpadded_layouts(seed):
    """fringe_rows (P:297 partial blocks at the fringe; R23): every assignment
    at padded row p = pos[i] sits in block-row r = p // bs at offset p % bs;
    in the unpadded layout it is dense row sorted_pos[i] = brow_start[r] +
    p % bs, inside the block's valid rows; each expert's block-rows hold
    exactly its counts (only the last one partial) and tile [bins-counts, bins)."""
    rng = np.random.default_rng(seed)
    E, bs = int(rng.integers(1, 9)), int(rng.choice([2, 4, 8]))
    T, k = int(rng.integers(1, 60)), int(rng.integers(1, min(E, 3) + 1))
    idx = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
    plan = O.make_plan(idx, E, bs)
    bst, brows = O.fringe_rows(plan, bs)
    assert bst.size == plan.Tp // bs
    sorted_pos = np.empty(T * k, np.int64)
    sorted_pos[plan.sorted_idx] = np.arange(T * k)
    for i in range(T * k):
        p = plan.pos[i]
        r, off = p // bs, p % bs
        assert off < brows[r]
        assert sorted_pos[i] == bst[r] + off
    for e in range(E):
        r0 = (plan.padded_bins[e] - plan.padded_counts[e]) // bs
        nr = plan.padded_counts[e] // bs
        assert brows[r0:r0 + nr].sum() == plan.counts[e]
        if nr:
            assert (brows[r0:r0 + nr - 1] == bs).all()
            assert bst[r0] == plan.bins[e] - plan.counts[e]
            assert bst[r0 + nr - 1] + brows[r0 + nr - 1] == plan.bins[e]
