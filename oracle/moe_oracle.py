"""CPU oracle for MegaBlocks' dropless-MoE layer (arXiv 2211.15841).

TEST INFRASTRUCTURE ONLY. Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s cpu_baseline / `--impl reference` legs may import this module.
The product path (`paper_2211_15841_b200`) never imports it and shares no code
with it (no kernels, headers, helpers or constants).

Plain, slow, obviously-correct numpy in float64. Every function follows the
paper's description step by step, in the paper's order and notation; a library
primitive (matmul, stable argsort, cumsum) serves as a step where noted.
Citations: `P:n` = PAPER.md line n (section / figure named), `S:n` = SPEC.md
line n (used for interfaces and worked examples only). Readings of points the
paper leaves open are numbered R1..R16 and listed in DESIGN.md §3.

Parity pins: every function here is pinned by a `-m "not gpu"` test in
tests/test_oracle.py (golden fixtures, closed forms, independent formulations,
finite differences). No function is "parity unpinned".

Layout conventions (shared with the C ABI by *specification*, not by code):
  x      [T, h]          tokens x hidden
  wr     [h, E]          router projection
  w1     [h, E*f]        first expert layer, expert e = columns e*f:(e+1)*f
  w2     [E*f, h]        second expert layer, expert e = rows e*f:(e+1)*f (R1)
  sparse values [nnz, bs, bs], blocks in BCSR (row-major block) order, each block
                  row-major (Fig. 4)
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

ACT_IDENTITY, ACT_GELU, ACT_RELU = 0, 1, 2
_GELU_C = math.sqrt(2.0 / math.pi)


# ----------------------------------------------------------------------------
# Router: §2.1 Routing. "the tokens are projected from hidden_size
# elements to num_experts scores by multiplying with a weight matrix ... The
# scores are normalized with a softmax and the routing decisions are made by
# greedily selecting the top_k scoring experts for each token."
# ----------------------------------------------------------------------------

def router_logits(x: np.ndarray, wr: np.ndarray) -> np.ndarray:
    """L = x . Wr  (P:98 'projected ... by multiplying with a weight matrix')."""
    return np.asarray(x, np.float64) @ np.asarray(wr, np.float64)


def softmax(logits: np.ndarray) -> np.ndarray:
    """Row softmax with max subtraction (P:98 'normalized with a softmax')."""
    L = np.asarray(logits, np.float64)
    z = L - L.max(axis=1, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=1, keepdims=True)


def topk(logits: np.ndarray, k: int, renormalize: bool = False):
    """Greedy top-k (P:98 'greedily selecting the top_k scoring experts').

    R6: selection is made on the logits (softmax is monotone, so this is the
    same set as selecting on the probabilities in exact arithmetic); slots are
    in descending score order; exact ties go to the lower expert index.
    Gates are the softmax probabilities of the chosen experts, not
    renormalised (R4, P:96 'probabilities for each assignment'); with
    `renormalize` each token's k gates are divided by
    their sum.
    Returns (expert_idx [T,k] int32, gates [T,k] float64).
    """
    L = np.asarray(logits, np.float64)
    T, E = L.shape
    if not 1 <= k <= E:
        raise ValueError(f"top_k={k} must be in [1, num_experts={E}]")
    idx = np.empty((T, k), np.int32)
    for t in range(T):
        # stable sort on descending score: equal scores keep ascending index order
        order = np.argsort(-L[t], kind="stable")
        idx[t] = order[:k]
    p = softmax(L)
    gates = np.take_along_axis(p, idx.astype(np.int64), axis=1)
    if renormalize:
        gates = gates / gates.sum(axis=1, keepdims=True)
    return idx, gates


def load_balance_loss(probs: np.ndarray, expert_idx: np.ndarray, coeff: float):
    """Auxiliary load-balancing loss (§2.2 P:118 names it without a formula;
    SURVEY NEXT-4 takes S:354's): loss = coeff * E * sum_e f_e * P_e, f_e = the
    fraction of tokens whose top-1 choice is e (treated as a constant), P_e =
    the mean router probability of e. Returns (loss, dloss/dprobs [T,E])."""
    p = np.asarray(probs, np.float64)
    T, E = p.shape
    top1 = np.asarray(expert_idx).reshape(T, -1)[:, 0]
    f = np.zeros(E, np.float64)
    for t in range(T):
        f[top1[t]] += 1.0
    f /= T
    P = p.sum(axis=0) / T
    loss = coeff * E * float((f * P).sum())
    dprobs = np.broadcast_to(coeff * E * f / T, (T, E)).copy()
    return loss, dprobs


# ----------------------------------------------------------------------------
# Permutation plan: §2.2 + §5.2 "we pad each group of tokens with zeros
# to the nearest multiple of 128" + Fig. 5 padded_gather.
# ----------------------------------------------------------------------------

@dataclass
class Plan:
    counts: np.ndarray          # [E] assignments per expert (kept ones, with a capacity)
    bins: np.ndarray            # [E] inclusive cumsum of counts
    padded_counts: np.ndarray   # [E] counts rounded up to a multiple of bs
    padded_bins: np.ndarray     # [E] inclusive cumsum of padded_counts
    sorted_idx: np.ndarray      # [R_kept] kept flat ids i = t*k + j in expert order (stable)
    pos: np.ndarray             # [R] padded row of flat id i; -1 for a dropped assignment
    Tp: int                     # total padded rows
    dropped: np.ndarray = None  # [R] bool, assignment i dropped by the capacity (all False dropless)


def make_plan(expert_idx: np.ndarray, num_experts: int, bs: int, capacity: int | None = None) -> Plan:
    """Histogram, bins, stable expert-grouped order and padded positions.

    counts[e] = #{(t,j): idx[t,j] = e}; bins = inclusive cumsum (R7: grouping is
    stable by flat id t*k+j); padded_counts = ceil(counts/bs)*bs, pad rows at the
    tail of each expert's group and zero-token experts get zero rows (R8).

    capacity (the token-dropping formulation the paper compares against, §2.2
    P:112-116): each expert keeps at most `capacity`
    assignments, the earliest in flat-id order (S:284 keep-earliest); the others
    are dropped (pos = -1) and contribute nothing ("tokens are dropped").
    None = dropless, the method of the paper."""
    flat = np.asarray(expert_idx, np.int64).reshape(-1)
    R = flat.size
    order = np.argsort(flat, kind="stable")         # stable: ascending flat id within expert
    rank_all = np.zeros(R, np.int64)
    seen = np.zeros(num_experts, np.int64)
    for i in order:                                  # rank of each assignment within its expert
        rank_all[i] = seen[flat[i]]
        seen[flat[i]] += 1
    dropped = np.zeros(R, bool) if capacity is None else rank_all >= capacity
    counts = np.zeros(num_experts, np.int64)
    for i in range(R):                               # histogram of the kept assignments
        if not dropped[i]:
            counts[flat[i]] += 1
    bins = np.cumsum(counts)
    padded_counts = ((counts + bs - 1) // bs) * bs
    padded_bins = np.cumsum(padded_counts)
    sorted_idx = np.array([i for i in order if not dropped[i]], np.int64)
    pos = np.full(R, -1, np.int64)
    for i in sorted_idx:
        e = flat[i]
        pos[i] = (padded_bins[e] - padded_counts[e]) + rank_all[i]
    Tp = int(padded_bins[-1]) if num_experts > 0 else 0
    return Plan(counts, bins, padded_counts, padded_bins, sorted_idx, pos, Tp, dropped)


def padded_gather(x: np.ndarray, plan: Plan, k: int) -> np.ndarray:
    """Fig. 5 line 15 'x = padded_gather(x, indices)': group tokens by
    expert, pad each group with zero rows to a multiple of bs."""
    x = np.asarray(x, np.float64)
    xg = np.zeros((plan.Tp, x.shape[1]), np.float64)
    for i in range(plan.pos.size):
        if plan.pos[i] >= 0:                        # dropped assignments are not gathered
            xg[plan.pos[i]] = x[i // k]
    return xg


def padded_scatter(yg: np.ndarray, plan: Plan, gates: np.ndarray, T: int, k: int) -> np.ndarray:
    """Fig. 5 lines 26-27 'padded_scatter' then 'x * weights' and
    §2.4 'weighted results are summed'. R5: weight each slot then
    sum in ascending slot order."""
    yg = np.asarray(yg, np.float64)
    g = np.asarray(gates, np.float64).reshape(T, k)
    y = np.zeros((T, yg.shape[1]), np.float64)
    for t in range(T):
        for j in range(k):
            if plan.pos[t * k + j] >= 0:            # a dropped slot contributes zero
                y[t] += g[t, j] * yg[plan.pos[t * k + j]]
    return y


# ----------------------------------------------------------------------------
# Hybrid blocked-CSR-COO topology with transpose indices (§5.1.3 P:235-242,
# §5.1.4, Fig. 4).
# ----------------------------------------------------------------------------

@dataclass
class Topology:
    bs: int
    n_block_rows: int
    n_block_cols: int
    row_offsets: np.ndarray     # [n_block_rows+1]  BCSR
    col_indices: np.ndarray     # [nnz]             BCSR
    row_indices: np.ndarray     # [nnz]             COO rows, 'materialize the row indices'
    t_col_offsets: np.ndarray   # [n_block_cols+1]  transposed offsets (R9)
    t_block_offsets: np.ndarray # [nnz]             'offset of each nonzero block in memory',
                                #                   'stored in transposed order', block units
    t_row_indices: np.ndarray   # [nnz]             row of each block in transposed order (R9)
    extra: dict = field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(self.col_indices.size)


def topology_from_blocks(coords, n_block_rows: int, n_block_cols: int, bs: int) -> Topology:
    """Generic construction from a set of nonzero block coordinates.

    BCSR: blocks sorted row-major; row_offsets from per-row counts; COO
    row_indices kept in the same row-wise order (P:242 'we maintain the row-wise
    ordering of nonzero blocks so the matrix can be operated on as either BCSR
    or blocked coordinate format'). Transpose index: storage indices of the
    blocks listed in (column, row) order, with per-column offsets.
    """
    coords = sorted(set((int(r), int(c)) for r, c in coords))
    for r, c in coords:
        if not (0 <= r < n_block_rows and 0 <= c < n_block_cols):
            raise ValueError(f"block ({r},{c}) outside {n_block_rows}x{n_block_cols} grid")
    nnz = len(coords)
    row_indices = np.array([r for r, _ in coords], np.int64)
    col_indices = np.array([c for _, c in coords], np.int64)
    row_counts = np.zeros(n_block_rows, np.int64)
    for r in row_indices:
        row_counts[r] += 1
    row_offsets = np.concatenate([[0], np.cumsum(row_counts)]).astype(np.int64)
    # transposed order: sort storage indices by (col, row)
    storage = list(range(nnz))
    storage.sort(key=lambda s: (col_indices[s], row_indices[s]))
    t_block_offsets = np.array(storage, np.int64)
    col_counts = np.zeros(n_block_cols, np.int64)
    for c in col_indices:
        col_counts[c] += 1
    t_col_offsets = np.concatenate([[0], np.cumsum(col_counts)]).astype(np.int64)
    t_row_indices = row_indices[t_block_offsets] if nnz else np.zeros(0, np.int64)
    return Topology(bs, n_block_rows, n_block_cols, row_offsets, col_indices, row_indices,
                    t_col_offsets, t_block_offsets, t_row_indices)


def moe_topology_blocks(plan: Plan, bs: int, ffn: int):
    """The nonzero blocks of Fig. 3C: expert e owns the dense
    rectangle of padded_counts[e]/bs block-rows starting at its padded offset
    and the block-columns [e*F, (e+1)*F), F = ffn/bs."""
    F = ffn // bs
    coords = []
    for e in range(plan.counts.size):
        r0 = (plan.padded_bins[e] - plan.padded_counts[e]) // bs
        for r in range(plan.padded_counts[e] // bs):
            for j in range(F):
                coords.append((r0 + r, e * F + j))
    return coords


def make_topology(plan: Plan, bs: int, ffn: int) -> Topology:
    """Fig. 5 line 12 'topology = make_topology(indices)', with the
    transposed metadata built at the same time. Generic sort-based
    construction over the MoE block pattern."""
    if ffn % bs:
        raise ValueError(f"ffn_hidden_size={ffn} not a multiple of block_size={bs}")
    E = plan.counts.size
    return topology_from_blocks(moe_topology_blocks(plan, bs, ffn), plan.Tp // bs, E * ffn // bs, bs)


def make_topology_closed_form(plan: Plan, bs: int, ffn: int) -> Topology:
    """Closed form of the MoE topology, an independent
    derivation asserted equal to make_topology() by the tests:
      row_offsets[r] = r*F; row_indices[s] = s // F; col_indices[s] = e(r)*F + s % F
      t_col_offsets[e*F+j] = F*start_e/bs + j*padded_counts[e]/bs
      t_block_offsets lists (start_e/bs + i)*F + j for i over the expert's rows.
    """
    F = ffn // bs
    E = plan.counts.size
    nbr = plan.Tp // bs
    start = plan.padded_bins - plan.padded_counts
    row_expert = np.empty(nbr, np.int64)
    for e in range(E):
        row_expert[start[e] // bs:(start[e] + plan.padded_counts[e]) // bs] = e
    nnz = nbr * F
    s = np.arange(nnz, dtype=np.int64)
    row_offsets = np.arange(nbr + 1, dtype=np.int64) * F
    row_indices = s // F
    col_indices = row_expert[row_indices] * F + s % F if nnz else np.zeros(0, np.int64)
    t_col_offsets = np.zeros(E * F + 1, np.int64)
    t_block_offsets = np.zeros(nnz, np.int64)
    t_row_indices = np.zeros(nnz, np.int64)
    for e in range(E):
        nr = plan.padded_counts[e] // bs
        for j in range(F):
            c = e * F + j
            off = F * start[e] // bs + j * nr
            t_col_offsets[c] = off
            for i in range(nr):
                t_block_offsets[off + i] = (start[e] // bs + i) * F + j
                t_row_indices[off + i] = start[e] // bs + i
    t_col_offsets[E * F] = nnz
    return Topology(bs, nbr, E * F, row_offsets, col_indices, row_indices,
                    t_col_offsets, t_block_offsets, t_row_indices)


def fringe_rows(plan: Plan, bs: int):
    """Partial blocks at the fringe ('We could remove this constraint
    [padding to a multiple of 128] by supporting partial blocks at the fringe
    of the problem', DESIGN reading R23): the dense
    expert-grouped rows are NOT padded — row u holds assignment sorted_idx[u],
    expert e's rows are [bins[e] - counts[e], bins[e]) — while the block
    structure (BCSR over the padded block-rows) is unchanged. Block-row r, the
    i-th of expert e, covers the dense rows [brow_start[r], brow_start[r] +
    brow_rows[r]) with brow_start = bins[e] - counts[e] + bs*i and brow_rows =
    min(bs, counts[e] - bs*i); rows of its blocks at or beyond brow_rows are
    the fringe (zero in the sparse values). Returns (brow_start, brow_rows),
    int64 [Tp / bs]."""
    nbr = plan.Tp // bs
    brow_start = np.zeros(nbr, np.int64)
    brow_rows = np.zeros(nbr, np.int64)
    for e in range(plan.counts.size):
        r0 = (plan.padded_bins[e] - plan.padded_counts[e]) // bs
        u0 = plan.bins[e] - plan.counts[e]
        for i in range(plan.padded_counts[e] // bs):
            brow_start[r0 + i] = u0 + bs * i
            brow_rows[r0 + i] = min(bs, plan.counts[e] - bs * i)
    return brow_start, brow_rows


# ----------------------------------------------------------------------------
# Block-sparse products, Triton notation (§4 'Preliminaries'): output,
# left input, right input; superscript T transposes an input. §5.1:
# forward SDD then DSD; backward SDD^T, DS^TD, DSD^T, DD^TS.
# ----------------------------------------------------------------------------

def _eff(m: np.ndarray, trans: bool) -> np.ndarray:
    m = np.asarray(m, np.float64)
    return m.T if trans else m


def sdd(a: np.ndarray, b: np.ndarray, topo: Topology, trans_a: bool = False,
        trans_b: bool = False) -> np.ndarray:
    """SDD (P:177 'sampled dense-dense'): for every nonzero block (r,c) located
    through the COO row index, block = A[r-block, :] . B[:, c-block].
    Returns values [nnz, bs, bs]."""
    A, B, bs = _eff(a, trans_a), _eff(b, trans_b), topo.bs
    out = np.zeros((topo.nnz, bs, bs), np.float64)
    for s in range(topo.nnz):
        r, c = topo.row_indices[s], topo.col_indices[s]
        out[s] = A[r * bs:(r + 1) * bs, :] @ B[:, c * bs:(c + 1) * bs]
    return out


def dsd(vals: np.ndarray, b: np.ndarray, topo: Topology, trans_s: bool = False,
        trans_b: bool = False) -> np.ndarray:
    """DSD: dense = sparse . dense.
    Not transposed: out[r-block] = sum over blocks s of row r (BCSR walk)
    of S_s . B[c_s-block, :].
    Transposed (DS^TD): out[c-block] = sum over blocks of column c walked
    through the transpose index (no value copy) of S_b^T . B[r_b-block, :].
    """
    B, bs = _eff(b, trans_b), topo.bs
    V = np.asarray(vals, np.float64)
    if not trans_s:
        out = np.zeros((topo.n_block_rows * bs, B.shape[1]), np.float64)
        for r in range(topo.n_block_rows):
            for s in range(topo.row_offsets[r], topo.row_offsets[r + 1]):
                c = topo.col_indices[s]
                out[r * bs:(r + 1) * bs] += V[s] @ B[c * bs:(c + 1) * bs, :]
    else:
        out = np.zeros((topo.n_block_cols * bs, B.shape[1]), np.float64)
        for c in range(topo.n_block_cols):
            for i in range(topo.t_col_offsets[c], topo.t_col_offsets[c + 1]):
                blk, r = topo.t_block_offsets[i], topo.t_row_indices[i]
                out[c * bs:(c + 1) * bs] += V[blk].T @ B[r * bs:(r + 1) * bs, :]
    return out


def dds(a: np.ndarray, vals: np.ndarray, topo: Topology, trans_a: bool = False,
        trans_s: bool = False) -> np.ndarray:
    """DDS: dense = dense . sparse.
    Not transposed (DD^TS with trans_a): out[:, c-block] = sum over the
    blocks of column c (transpose index) of A[:, r_b-block] . S_b.
    Transposed sparse: out[:, r-block] = sum over blocks s of row r of
    A[:, c_s-block] . S_s^T.
    """
    A, bs = _eff(a, trans_a), topo.bs
    V = np.asarray(vals, np.float64)
    if not trans_s:
        out = np.zeros((A.shape[0], topo.n_block_cols * bs), np.float64)
        for c in range(topo.n_block_cols):
            for i in range(topo.t_col_offsets[c], topo.t_col_offsets[c + 1]):
                blk, r = topo.t_block_offsets[i], topo.t_row_indices[i]
                out[:, c * bs:(c + 1) * bs] += A[:, r * bs:(r + 1) * bs] @ V[blk]
    else:
        out = np.zeros((A.shape[0], topo.n_block_rows * bs), np.float64)
        for r in range(topo.n_block_rows):
            for s in range(topo.row_offsets[r], topo.row_offsets[r + 1]):
                c = topo.col_indices[s]
                out[:, r * bs:(r + 1) * bs] += A[:, c * bs:(c + 1) * bs] @ V[s].T
    return out


# ----------------------------------------------------------------------------
# Expert activation. The paper never names it ('iterate between SDD and DSD',
# P:182); R2: gelu with the tanh approximation, identity and relu also.
# ----------------------------------------------------------------------------

def act(kind: int, h: np.ndarray) -> np.ndarray:
    h = np.asarray(h, np.float64)
    if kind == ACT_IDENTITY:
        return h.copy()
    if kind == ACT_RELU:
        return np.maximum(h, 0.0)
    if kind == ACT_GELU:
        return 0.5 * h * (1.0 + np.tanh(_GELU_C * (h + 0.044715 * h ** 3)))
    raise ValueError(f"unknown activation {kind}")


def act_grad(kind: int, h: np.ndarray) -> np.ndarray:
    """d act / d h at the pre-activation h."""
    h = np.asarray(h, np.float64)
    if kind == ACT_IDENTITY:
        return np.ones_like(h)
    if kind == ACT_RELU:
        return (h > 0).astype(np.float64)
    if kind == ACT_GELU:
        u = _GELU_C * (h + 0.044715 * h ** 3)
        t = np.tanh(u)
        du = _GELU_C * (1.0 + 3.0 * 0.044715 * h ** 2)
        return 0.5 * (1.0 + t) + 0.5 * h * (1.0 - t * t) * du
    raise ValueError(f"unknown activation {kind}")


# ----------------------------------------------------------------------------
# The dMoE layer: Fig. 5 forward; §5.1 backward.
# ----------------------------------------------------------------------------

@dataclass
class Cache:
    x: np.ndarray
    logits: np.ndarray
    probs: np.ndarray
    expert_idx: np.ndarray
    gates: np.ndarray
    plan: Plan
    topo: Topology
    xg: np.ndarray
    h_pre: np.ndarray
    a: np.ndarray
    yg: np.ndarray
    k: int
    act: int
    renormalize: bool = False
    aux_coeff: float = 0.0
    aux_loss: float = 0.0


def dmoe_forward(x, wr, w1, w2, top_k: int, bs: int, ffn: int, act_kind: int = ACT_GELU,
                 logits: np.ndarray | None = None, capacity: int | None = None, renormalize: bool = False,
                 aux_coeff: float = 0.0, expert_idx: np.ndarray | None = None):
    """Fig. 5 'dmoe_forward', step by step:
    (1) indices, weights = router(x)
    (2) topology = make_topology(indices)
    (3) x = padded_gather(x, indices)
    (4) x = sdd(x, w1, topology); act; dsd(x, w2) P:275-276 (+ R2 activation)
    (5) padded_scatter(x, indices) * weights
    `logits` may be given to route from a fixed score matrix (tests of the
    routing-independent part). `capacity` selects the token-dropping
    formulation (make_plan); None = dropless. `expert_idx` [T, k] replaces
    the greedy selection of step (1) (R6: a test resolving a near-tie token
    the other valid way); the gates are still this oracle's softmax
    probabilities of the given experts (renormalised if asked)."""
    x = np.asarray(x, np.float64)
    T = x.shape[0]
    E = np.asarray(wr).shape[1]
    L = router_logits(x, wr) if logits is None else np.asarray(logits, np.float64)
    if expert_idx is None:
        idx, gates = topk(L, top_k, renormalize)
    else:
        idx = np.asarray(expert_idx, np.int32).reshape(T, top_k)
        gates = np.take_along_axis(softmax(L), idx.astype(np.int64), axis=1)
        if renormalize:
            gates = gates / gates.sum(axis=1, keepdims=True)
    plan = make_plan(idx, E, bs, capacity)
    topo = make_topology(plan, bs, ffn)
    xg = padded_gather(x, plan, top_k)
    h_pre = sdd(xg, w1, topo)
    a = act(act_kind, h_pre)
    yg = dsd(a, w2, topo)
    y = padded_scatter(yg, plan, gates, T, top_k)
    aux = load_balance_loss(softmax(L), idx, aux_coeff)[0] if aux_coeff else 0.0
    cache = Cache(x, L, softmax(L), idx, gates, plan, topo, xg, h_pre, a, yg, top_k, act_kind, renormalize,
                  aux_coeff, aux)
    return y, cache


def dmoe_backward(cache: Cache, dy, wr, w1, w2):
    """Backward of Fig. 5 through the ops §5.1 names:
    b1 scatter backward: dYg[pos] = gate*dy; dgate = <Yg[pos], dy>   (chain rule of P:280)
    b2 SDD^T  : dA = dYg . W2^T on the topology, dH = dA * act'(H)     'second layer data gradient'
    b3 DS^TD  : dW2 = A^T . dYg  (transpose index)                     'second layer weight gradient'
    b4 DSD^T  : dXg = dH . W1^T                                       'first layer data gradient'
    b5 DD^TS  : dW1 = Xg^T . dH  (transpose index)                     'first layer weight gradient'
    b6 gather backward: dx[t] = sum_j dXg[pos[t*k+j]]
    b7 router backward through softmax: dlogits = p*(dp - <p,dp>),
       dWr = x^T dlogits, dx += dlogits Wr^T
    Returns dict dx, dwr, dw1, dw2, dgates, dlogits.
    """
    c = cache
    dy = np.asarray(dy, np.float64)
    T, h = dy.shape
    k = c.k
    plan, topo = c.plan, c.topo
    # b1
    dyg = np.zeros((plan.Tp, h), np.float64)
    dgates = np.zeros((T, k), np.float64)
    for t in range(T):
        for j in range(k):
            p = plan.pos[t * k + j]
            if p < 0:                               # dropped: y does not depend on it, dgate = 0
                continue
            dyg[p] = c.gates[t, j] * dy[t]
            dgates[t, j] = float(c.yg[p] @ dy[t])
    # b2
    da = sdd(dyg, w2, topo, trans_b=True)
    dh = da * act_grad(c.act, c.h_pre)
    # b3
    dw2 = dsd(c.a, dyg, topo, trans_s=True)
    # b4
    dxg = dsd(dh, w1, topo, trans_b=True)
    # b5
    dw1 = dds(c.xg, dh, topo, trans_a=True)
    # b6
    dx = np.zeros((T, h), np.float64)
    for t in range(T):
        for j in range(k):
            if plan.pos[t * k + j] >= 0:
                dx[t] += dxg[plan.pos[t * k + j]]
    # b7
    E = c.logits.shape[1]
    dp = np.zeros((T, E), np.float64)
    p = c.probs
    for t in range(T):
        if c.renormalize:
            # g_j = p_j / S, S = sum_i p_i over the chosen: dL/dp_j = (dg_j - sum_i dg_i g_i) / S
            S = sum(p[t, c.expert_idx[t, i]] for i in range(k))
            gd = sum(dgates[t, i] * c.gates[t, i] for i in range(k))
            for j in range(k):
                dp[t, c.expert_idx[t, j]] += (dgates[t, j] - gd) / S
        else:
            for j in range(k):
                dp[t, c.expert_idx[t, j]] += dgates[t, j]
    if c.aux_coeff:                                 # + the auxiliary loss's gradient (d total / d aux = 1)
        dp = dp + load_balance_loss(p, c.expert_idx, c.aux_coeff)[1]
    dlogits = p * (dp - (p * dp).sum(axis=1, keepdims=True))
    dwr = c.x.T @ dlogits
    dx = dx + dlogits @ np.asarray(wr, np.float64).T
    return {"dx": dx, "dwr": dwr, "dw1": dw1, "dw2": dw2, "dgates": dgates,
            "dlogits": dlogits, "dyg": dyg, "dh": dh, "dxg": dxg}


# ----------------------------------------------------------------------------
# Sizes: worst-case padded rows / blocks.
# ----------------------------------------------------------------------------

def max_padded_rows(T: int, k: int, E: int, bs: int) -> int:
    """Tp = sum_e bs*ceil(c_e/bs) <= R + min(E, R)*(bs-1), rounded down to bs."""
    R = T * k
    return bs * ((R + min(E, R) * (bs - 1)) // bs)


def expert_capacity(num_tokens: int, num_experts: int, capacity_factor: float) -> int:
    """§2.2 displayed formula: num_tokens/num_experts * capacity_factor,
    rounded up (S:270s). Used only by the token-dropping cross-check."""
    return int(math.ceil(num_tokens * capacity_factor / num_experts - 1e-12))
