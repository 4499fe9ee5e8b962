"""CPU checks of the parity helpers (tests/parity_util.py): the near-tie band
and the top-k validity test on hand-made logits, and the per-row / per-block
error measures on planted errors."""
import numpy as np

from parity_util import (block_max_rel, check_routing, logit_error_bound, near_tie_band, resolved_routing,
                         row_max_rel, valid_topk)


def test_near_tie_band_and_validity():
    L = np.array([[3.0, 1.0, 0.0, -1.0],      # clear winner
                  [1.0, 1.0 - 1e-6, 0.0, 0.0],  # top-1 tie within the bound
                  [2.0, 1.0, 1.0 - 1e-6, 0.0]])  # top-2 tie at the boundary of k=2
    b = np.full_like(L, 1e-5)
    assert near_tie_band(L, b, 1).tolist() == [False, True, False]
    assert near_tie_band(L, b, 2).tolist() == [False, True, True]
    assert valid_topk(L[1], b[1], [1]) and valid_topk(L[1], b[1], [0])
    assert not valid_topk(L[0], b[0], [1])
    assert valid_topk(L[2], b[2], [0, 2]) and not valid_topk(L[2], b[2], [2, 0])
    assert not valid_topk(L[2], b[2], [0, 0])


def test_check_routing_accepts_valid_flip_and_rejects_wrong_one():
    L = np.array([[1.0, 1.0 - 1e-6, 0.0], [2.0, 0.0, 1.0]])
    b = np.full_like(L, 1e-5)
    want = np.array([[0], [0]])
    flips = check_routing(L, b, np.array([[1], [0]]), want, max_frac=1.0)
    assert flips.tolist() == [True, False]
    idx, _ = resolved_routing(L, b, np.array([[1], [0]]), want, max_frac=1.0)
    assert idx.tolist() == [[1], [0]]
    try:
        check_routing(L, b, np.array([[0], [2]]), want, max_frac=1.0)
    except AssertionError:
        pass
    else:
        raise AssertionError("a flip outside the near-tie band must fail")


def test_logit_error_bound_covers_fp32_accumulation():
    rng = np.random.default_rng(0)
    x = rng.normal(size=(64, 512)).astype(np.float32)
    w = (rng.normal(size=(512, 8)) / 22.6).astype(np.float32)
    exact = x.astype(np.float64) @ w.astype(np.float64)
    f32 = np.zeros((64, 8), np.float32)
    for i in range(512):                        # naive fp32 accumulation, the worst order
        f32 += x[:, i:i + 1] * w[i:i + 1, :]
    assert (np.abs(f32 - exact) <= logit_error_bound(x, w)).all()


def test_row_and_block_measures_find_a_planted_error():
    rng = np.random.default_rng(1)
    want = rng.normal(size=(300, 64))
    got = want * (1 + 1e-3 * rng.normal(size=want.shape))
    assert row_max_rel(got, want) < 1e-2
    got[123] = 0.0                               # one row lost: whole-tensor error only ~6e-2
    assert row_max_rel(got, want) > 0.99
    W = rng.normal(size=(256, 384))
    G = W.copy()
    G[128:256, 256:384] *= 1.05                  # one tile off by 5%
    assert block_max_rel(G, W) > 0.04 and np.linalg.norm(G - W) / np.linalg.norm(W) < 0.03
