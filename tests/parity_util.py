"""Parity helpers shared by the GPU tests and `__graft_entry__.smoke()`.

Test infrastructure: compares the CUDA path's outputs with the oracle's. Holds
no arithmetic of the method; the only model here is the error bound of the
GPU's fp32 router logits, used to decide where two routings may both be right
(reading R6).

Bars (BASELINE.json north_star):
* bf16 outputs and gradients: relative Frobenius error <= 1e-2 per tensor, and
  per row (y, dx) / per 128 x 128 block (dW1, dW2) <= ROW_TOL, so an error
  confined to a few rows or one tail tile cannot hide inside a whole-tensor norm.
* routing: bit-exact for every token outside the near-tie band; inside it the
  GPU's choice must be a valid top-k of the oracle's exact logits within the
  fp32 accumulation bound (`check_routing`).
"""
from __future__ import annotations

import numpy as np

FRO_TOL = 1e-2
# Per row / per block. A bf16 row's error is an average of independent
# per-element roundings (2^-9 relative, ~1.1e-3 rms, plus the bf16-rounded
# intermediate A): rows sit near the whole-tensor figure (2-4e-3). 2e-2 is 5x
# that and still catches a wrong, dropped or stale row or tile (error ~1).
ROW_TOL = 2e-2
U32 = 2.0 ** -24


def f64(t):
    return t.detach().float().cpu().double().numpy()


def rel_fro(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    den = np.linalg.norm(want)
    return float(np.linalg.norm(got - want) / (den if den > 0 else 1.0))


def row_max_rel(got, want, floor_frac=1e-2):
    """max over rows of ||got_r - want_r|| / max(||want_r||, floor_frac * rms row norm)."""
    got = np.asarray(got, np.float64).reshape(len(want), -1)
    want = np.asarray(want, np.float64).reshape(len(want), -1)
    if want.size == 0:
        return 0.0
    n = np.linalg.norm(want, axis=1)
    rms = float(np.sqrt((n ** 2).mean()))
    den = np.maximum(n, floor_frac * rms if rms > 0 else 1.0)
    return float((np.linalg.norm(got - want, axis=1) / den).max())


def block_max_rel(got, want, bs=128, floor_frac=1e-2):
    """max over bs x bs blocks of the block's relative Frobenius error (dW tiles)."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    R, C = want.shape
    errs, norms = [], []
    for r in range(0, R, bs):
        for c in range(0, C, bs):
            w = want[r:r + bs, c:c + bs]
            norms.append(np.linalg.norm(w))
            errs.append(np.linalg.norm(got[r:r + bs, c:c + bs] - w))
    norms, errs = np.array(norms), np.array(errs)
    rms = float(np.sqrt((norms ** 2).mean())) if norms.size else 0.0
    den = np.maximum(norms, floor_frac * rms if rms > 0 else 1.0)
    return float((errs / den).max()) if errs.size else 0.0


def assert_close(name, got, want, rows=None, per="row", tol=FRO_TOL, row_tol=ROW_TOL):
    """Whole-tensor relative Frobenius <= tol and per-row (per='row') or
    per-128x128-block (per='block') <= row_tol. `rows` selects rows to compare
    (e.g. tokens routed identically on both sides)."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    if rows is not None:
        got, want = got[rows], want[rows]
    e = rel_fro(got, want)
    assert e < tol, f"{name}: relative Frobenius error {e:.3e} >= {tol}"
    if per == "row":
        m = row_max_rel(got, want)
    elif per == "block":
        m = block_max_rel(got, want)
    else:
        m = 0.0
    assert m < row_tol, f"{name}: worst {per} relative error {m:.3e} >= {row_tol}"
    return e, m


# ------------------------------------------------------------------ routing (R6)

def logit_error_bound(x64, wr64, c=2.0):
    """Worst-case |L_fp32 - L_exact| per (token, expert): the bf16 products are
    exact in fp32, so only the h-term fp32 accumulation errs, by at most
    gamma_h * sum_i |x_ti Wr_ie| with gamma_h ~ h * u (Higham, Thm 3.1);
    c = 2 covers the tensor core's accumulation order."""
    x64 = np.asarray(x64, np.float64)
    h = x64.shape[1]
    return c * h * U32 * (np.abs(x64) @ np.abs(np.asarray(wr64, np.float64)))


def near_tie_band(L, bound, k):
    """Tokens whose ordered top-k (set or slot order) could change if every
    logit moved by up to its bound: some rank a < k whose lower end does not
    clear the upper end of a lower-ranked expert."""
    L = np.asarray(L, np.float64)
    T, E = L.shape
    order = np.argsort(-L, axis=1, kind="stable")
    lo = np.take_along_axis(L - bound, order, axis=1)
    hi = np.take_along_axis(L + bound, order, axis=1)
    near = np.zeros(T, bool)
    if E == 1:
        return near
    suf = np.maximum.accumulate(hi[:, ::-1], axis=1)[:, ::-1]  # suf[:, b] = max hi over ranks >= b
    for a in range(min(k, E - 1)):
        near |= lo[:, a] <= suf[:, a + 1]
    return near


def valid_topk(Lt, bt, sel):
    """Is the ordered selection `sel` the greedy top-k of some logits within
    +-bt of Lt? Every chosen expert must be able to outrank every unchosen one,
    and each slot the slots after it."""
    sel = [int(e) for e in sel]
    if len(set(sel)) != len(sel):
        return False
    lo, hi = Lt - bt, Lt + bt
    rest = np.setdiff1d(np.arange(len(Lt)), sel)
    if rest.size and min(hi[e] for e in sel) < lo[rest].max():
        return False
    return all(hi[sel[a]] >= lo[sel[b]] for a in range(len(sel)) for b in range(a + 1, len(sel)))


def check_routing(L, bound, got_idx, want_idx, max_frac=1e-2):
    """Bit-exact routing outside the near-tie band; inside it, the GPU's choice
    must be a valid top-k within the bound. Returns the mask of flipped tokens
    (rows whose y / dx are not comparable to the oracle's)."""
    got_idx = np.asarray(got_idx).reshape(len(L), -1)
    want_idx = np.asarray(want_idx).reshape(len(L), -1)
    k = got_idx.shape[1]
    flips = (got_idx != want_idx).any(axis=1)
    near = near_tie_band(L, bound, k)
    bad = flips & ~near
    assert not bad.any(), f"routing differs outside the near-tie band at tokens {np.nonzero(bad)[0][:10]}"
    for t in np.nonzero(flips)[0]:
        assert valid_topk(L[t], bound[t], got_idx[t]), f"token {t}: {got_idx[t]} is not a valid top-{k}"
    assert flips.mean() <= max_frac, f"{flips.sum()} routing flips"
    return flips


def resolved_routing(L, bound, got_idx, want_idx, max_frac=1e-2):
    """The oracle's routing with each validated near-tie token resolved the way
    the GPU resolved it (R6; both are correct there). Lets a test compare
    downstream state that depends on every token's routing (capacity drops,
    weight gradients) without feeding the oracle any GPU floating-point value."""
    flips = check_routing(L, bound, got_idx, want_idx, max_frac)
    idx = np.array(want_idx, np.int32, copy=True).reshape(len(L), -1)
    idx[flips] = np.asarray(got_idx).reshape(len(L), -1)[flips]
    return idx, flips
