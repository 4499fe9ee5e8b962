#!/usr/bin/env python
"""E4-style block-sparse product sweep (SURVEY.md §8(d) "E4-style sweep";
BASELINE.json configs[4] "block-sparse GEMM sweep vs dense batched GEMM").

The paper benchmarks each of the six products of the dMoE layer (SDD, DSD,
SDD^T, DS^TD, DSD^T, DD^TS; §5.1 / Fig. "block-sparse matmul
benchmarks") against cuBLAS batched GEMM on the per-GPU problems of
its expert-parallel MoE-XS / Small / Medium runs, with the topology built
outside the timed region and an exactly uniform expert load (so the
block-diagonal problem is exactly a batched GEMM). This script does the same
on one B200: each product through the library's C ABI (moe_sdd / moe_dsd /
moe_dds, tcgen05 kernels) against torch.bmm (cuBLAS strided-batched bf16) on
the identical operands, L2 flushed before every timed launch (outside the
events), CUDA events on the launching stream.

It also checks that the two agree (relative Frobenius error ≤ 1e-2, the
north-star tolerance): with exact-uniform routing the block-diagonal product
IS the batched GEMM (SURVEY §8(c) pin "exact-uniform routing equals
torch.bmm").

Prints one JSON line per problem and a summary line; `--out FILE` also writes
them as a JSON list.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

# per-GPU problems at EP8 (SURVEY §8(d) sweep table): E local experts, n tokens per expert
PROBLEMS = {
    "XS": dict(E=8, n=8192, h=512, f=2048, k=1),
    "Small": dict(E=8, n=4096, h=768, f=3072, k=1),
    "Medium": dict(E=8, n=1024, h=1024, f=4096, k=1),
    "Medium-top2": dict(E=8, n=2048, h=1024, f=4096, k=2),   # C4 per-GPU: T=8192 tokens, k=2
    # bench.py's N = 8 weak-scaling run: 32768 tokens per rank of C1, 8 local experts
    "C1-EP8": dict(E=8, n=4096, h=512, f=2048, k=1),
}
PRODUCTS = ["sdd", "dsd", "sddT", "dsTd", "dsdT", "ddTs"]


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["bf16_tflops"]), float(p.get("bf16_tflops_sustained", p["bf16_tflops"])), "measured"
    except Exception:
        return 1590.0, 1400.0, "fallback"


def rel_fro(a, b):
    a = a.double()
    b = b.double()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


def blocks_to_dense(s, E, n, f, bs=128):
    """BCSR values [nnz, bs, bs] (block (r, e*F+j) at r*F+j) -> [E, n, f]."""
    F = f // bs
    return s.view(E, n // bs, F, bs, bs).permute(0, 1, 3, 2, 4).reshape(E, n, f)


def dense_to_blocks(d, E, n, f, bs=128):
    F = f // bs
    return d.view(E, n // bs, bs, F, bs).permute(0, 1, 3, 2, 4).reshape(E * (n // bs) * F, bs, bs).contiguous()


def time_launches(fn, reps, flush, stream):
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts), statistics.mean(ts)


def run_problem(name, pr, reps, warmup, flush):
    from paper_2211_15841_b200 import api as A
    d = torch.device("cuda:0")
    E, n, h, f, k = pr["E"], pr["n"], pr["h"], pr["f"], pr["k"]
    R = E * n                       # assignments = padded rows (exact-uniform, n % 128 == 0)
    T = R // k
    g = torch.Generator().manual_seed(11)
    # exact-uniform routing: expert_idx[t, j] = (floor(t*E/T) + j*E/2) mod E
    t_ = torch.arange(T)
    idx = torch.stack([((t_ * E) // T + j * (E // 2)) % E for j in range(k)], 1).to(torch.int32)
    cfg = A.make_config(T, h, E, k, f, act=A.ACT_IDENTITY)
    tg = A.moe_topology(cfg, idx.to(d))
    Tp, nnz = tg.sizes()
    assert Tp == R and nnz == R // 128 * (f // 128), (Tp, nnz)
    bf = torch.bfloat16
    rnd = lambda *s, std=1.0: (torch.randn(*s, generator=g) * std).to(bf).to(d)  # noqa: E731
    xg = rnd(R, h)                       # X_g (rows grouped by expert: rows [e*n, (e+1)*n))
    dyg = rnd(R, h)
    w1 = rnd(h, E * f, std=h ** -0.5)
    w2 = rnd(E * f, h, std=f ** -0.5)
    # batched-GEMM operands in the natural contiguous batched layout
    X3 = xg.view(E, n, h)
    dY3 = dyg.view(E, n, h)
    W1b = w1.view(h, E, f).permute(1, 0, 2).contiguous()       # [E, h, f]
    W2b = w2.view(E, f, h).contiguous()                         # [E, f, h]
    s_a = A.moe_sdd(cfg, xg, w1, 0, tg)                         # S operands of the later products
    s_dh = A.moe_sdd(cfg, dyg, w2, 1, tg)
    S3_a = blocks_to_dense(s_a[:nnz], E, n, f).contiguous()
    S3_dh = blocks_to_dense(s_dh[:nnz], E, n, f).contiguous()
    out_s = torch.empty_like(s_a)
    out_rows = torch.empty(A.moe_max_padded_rows(cfg), h, dtype=bf, device=d)
    out_w2 = torch.empty(E * f, h, dtype=bf, device=d)
    out_w1 = torch.empty(h, E * f, dtype=bf, device=d)
    ob_nf = torch.empty(E, n, f, dtype=bf, device=d)
    ob_nh = torch.empty(E, n, h, dtype=bf, device=d)
    ob_fh = torch.empty(E, f, h, dtype=bf, device=d)
    ob_hf = torch.empty(E, h, f, dtype=bf, device=d)

    ours = {
        "sdd": (lambda: A.moe_sdd(cfg, xg, w1, 0, tg, out=out_s), lambda: blocks_to_dense(out_s[:nnz], E, n, f)),
        "dsd": (lambda: A.moe_dsd(cfg, s_a, 0, w2, 0, tg, out=out_rows), lambda: out_rows[:R].view(E, n, h)),
        "sddT": (lambda: A.moe_sdd(cfg, dyg, w2, 1, tg, out=out_s), lambda: blocks_to_dense(out_s[:nnz], E, n, f)),
        "dsTd": (lambda: A.moe_dsd(cfg, s_a, 1, dyg, 0, tg, out=out_w2), lambda: out_w2.view(E, f, h)),
        "dsdT": (lambda: A.moe_dsd(cfg, s_dh, 0, w1, 1, tg, out=out_rows), lambda: out_rows[:R].view(E, n, h)),
        "ddTs": (lambda: A.moe_dds(cfg, xg, 1, s_dh, 0, tg, out=out_w1),
                 lambda: out_w1.view(h, E, f).permute(1, 0, 2)),
    }
    dense = {
        "sdd": (lambda: torch.bmm(X3, W1b, out=ob_nf), ob_nf),
        "dsd": (lambda: torch.bmm(S3_a, W2b, out=ob_nh), ob_nh),
        "sddT": (lambda: torch.bmm(dY3, W2b.transpose(1, 2), out=ob_nf), ob_nf),
        "dsTd": (lambda: torch.bmm(S3_a.transpose(1, 2), dY3, out=ob_fh), ob_fh),
        "dsdT": (lambda: torch.bmm(S3_dh, W1b.transpose(1, 2), out=ob_nh), ob_nh),
        "ddTs": (lambda: torch.bmm(X3.transpose(1, 2), S3_dh, out=ob_hf), ob_hf),
    }
    st = torch.cuda.current_stream()
    flop = 2.0 * R * h * f
    pk, pk_sus, src = peaks()
    rows = []
    for p in PRODUCTS:
        fo, get = ours[p]
        fd, od = dense[p]
        for _ in range(warmup):
            fo()
            fd()
        torch.cuda.synchronize()
        err = rel_fro(get().float(), od.float())
        mo, ao = time_launches(fo, reps, flush, st)
        md, ad = time_launches(fd, reps, flush, st)
        tf_o = flop / (mo * 1e-3) / 1e12
        tf_d = flop / (md * 1e-3) / 1e12
        rows.append({"problem": name, "product": p, "E": E, "tokens_per_expert": n, "hidden": h, "ffn": f,
                     "top_k": k, "gflop": round(flop / 1e9, 2), "ours_ms": round(mo, 4), "ours_ms_mean": round(ao, 4),
                     "bmm_ms": round(md, 4), "bmm_ms_mean": round(ad, 4),
                     "ours_tflops": round(tf_o, 1), "bmm_tflops": round(tf_d, 1),
                     "ours_frac_of_bf16_peak": round(tf_o / pk, 4), "bmm_frac_of_bf16_peak": round(tf_d / pk, 4),
                     "ours_frac_of_sustained": round(tf_o / pk_sus, 4),
                     "ours_over_bmm": round(md / mo, 4), "rel_fro_vs_bmm": err, "peak_source": src,
                     "peak_tflops": pk})
        assert err < 1e-2, (name, p, err)
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--problems", default=",".join(PROBLEMS))
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda:0")   # > 126 MB L2
    allrows = []
    for name in args.problems.split(","):
        rows = run_problem(name, PROBLEMS[name], args.reps, args.warmup, flush)
        for r in rows:
            print(json.dumps(r), flush=True)
        allrows += rows
        tot_o = sum(r["ours_ms"] for r in rows)
        tot_d = sum(r["bmm_ms"] for r in rows)
        print(json.dumps({"problem": name, "summary": True, "six_products_ours_ms": round(tot_o, 4),
                          "six_products_bmm_ms": round(tot_d, 4), "ours_over_bmm": round(tot_d / tot_o, 4),
                          "ours_tflops": round(6 * rows[0]["gflop"] / tot_o, 1),
                          "ours_frac_of_bf16_peak": round(6 * rows[0]["gflop"] / tot_o / rows[0]["peak_tflops"], 4)}),
              flush=True)
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(allrows, fh, indent=1)


if __name__ == "__main__":
    main()
