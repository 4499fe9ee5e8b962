"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NO arithmetic of the method (no routing, no topology, no
products). It only draws random tensors with the distributions stated in
DESIGN.md ("Input recipe", after SURVEY.md §8(d)) and rounds them to bf16 once,
so that both sides consume the very same bytes.

Configurations follow BASELINE.json `configs` and the paper's tables:
  Table 1: hidden sizes 512/768/1024, ffn = 4*hidden.
  Table 2: 64 experts, top_k = 1.
  Table 3: micro-batch 64/32/8 sequences of 1024 tokens.
"""
from __future__ import annotations

import dataclasses
import math

import torch


@dataclasses.dataclass(frozen=True)
class MoEShape:
    name: str
    tokens: int
    hidden: int
    ffn: int
    experts: int
    top_k: int
    block: int = 128
    routing: str = "natural"     # natural | uniform | skew
    skew: float = 0.0            # Zipf exponent s for routing == "skew"
    act: int = 1                 # 0 identity, 1 gelu(tanh), 2 relu

    def replace(self, **kw) -> "MoEShape":
        return dataclasses.replace(self, **kw)


# BASELINE.json configs[0..4]; token counts = Table 3 micro-batch x seq 1024
# where BASELINE leaves them open (SURVEY.md §8(d) "Configs, restated").
CONFIGS = {
    "C0": MoEShape("C0-tiny", 1024, 256, 512, 4, 1),
    "C1": MoEShape("C1-MoE-XS", 32768, 512, 2048, 64, 1),
    "C2": MoEShape("C2-MoE-Small-skew", 32768, 768, 3072, 64, 1, routing="skew", skew=0.5),
    "C3": MoEShape("C3-MoE-Medium", 8192, 1024, 4096, 64, 1),
    "C4": MoEShape("C4-MoE-Medium-top2", 8192, 1024, 4096, 64, 2),
    # "also report C3 at T_local = 32768 (it fits in B200 memory)"
    "C3L": MoEShape("C3-MoE-Medium-T32k", 32768, 1024, 4096, 64, 1),
}

# tensor ids used to derive per-tensor seeds: seed = base * 1000 + id
_X, _WR, _W1, _W2, _DY = 1, 2, 3, 4, 5


def _gen(base: int, tid: int) -> torch.Generator:
    g = torch.Generator()
    g.manual_seed(base * 1000 + tid)
    return g


def _normal(shape, std: float, base: int, tid: int) -> torch.Tensor:
    t = torch.randn(*shape, generator=_gen(base, tid), dtype=torch.float32)
    if std != 1.0:
        t.mul_(std)
    return t


def make_inputs(shape: MoEShape, seed: int = 0, tokens: int | None = None) -> dict:
    """Draw x, wr, w1, w2, dy as bf16 CPU tensors (RNE rounding from fp32).

    x  ~ N(0,1)        [T, h]
    wr ~ N(0, 1/h)     [h, E]      so logits ~ N(0,1): near-uniform routing
    w1 ~ N(0, 1/h)     [h, E*f]    (w1 (hidden, inner_dim))
    w2 ~ N(0, 1/f)     [E*f, h]    (PAPER.md:274 is garbled; reading R1)
    dy ~ N(0,1)        [T, h]
    routing == "skew": x[:, h-1] = 1 and wr[h-1, e] = log p_e, p_e ∝ (e+1)^-s,
    which biases the learned router toward low expert ids.
    """
    T = shape.tokens if tokens is None else tokens
    h, f, E = shape.hidden, shape.ffn, shape.experts
    x = _normal((T, h), 1.0, seed, _X)
    wr = _normal((h, E), 1.0 / math.sqrt(h), seed, _WR)
    if shape.routing == "skew":
        x[:, h - 1] = 1.0
        w = torch.tensor([(e + 1) ** (-shape.skew) for e in range(E)], dtype=torch.float64)
        wr[h - 1, :] = torch.log(w / w.sum()).to(torch.float32)
    w1 = _normal((h, E * f), 1.0 / math.sqrt(h), seed, _W1)
    w2 = _normal((E * f, h), 1.0 / math.sqrt(f), seed, _W2)
    dy = _normal((T, h), 1.0, seed, _DY)
    bf = torch.bfloat16
    return {"x": x.to(bf), "wr": wr.to(bf), "w1": w1.to(bf), "w2": w2.to(bf), "dy": dy.to(bf)}


def uniform_expert_idx(tokens: int, experts: int, top_k: int) -> torch.Tensor:
    """Exact-uniform assignment for the product sweep ("uniform
    distribution of tokens to experts"): idx[t, j] = (floor(t*E/T) + j*E/2) mod E.
    Slots of one token hit distinct experts when E >= 2."""
    t = torch.arange(tokens, dtype=torch.int64)
    base = (t * experts) // tokens
    cols = [(base + j * (experts // 2 if experts > 1 else 0)) % experts for j in range(top_k)]
    return torch.stack(cols, dim=1).to(torch.int32)


def random_expert_idx(tokens: int, experts: int, top_k: int, seed: int = 0,
                      zipf: float = 0.0) -> torch.Tensor:
    """Random distinct-per-token expert ids (Gumbel-top-k over log p_e with
    p_e ∝ (e+1)^-zipf). Used to feed topology/permutation tests directly."""
    g = _gen(seed, 11)
    logp = torch.tensor([-zipf * math.log(e + 1) for e in range(experts)], dtype=torch.float64)
    u = torch.rand(tokens, experts, generator=g, dtype=torch.float64).clamp_(1e-300, 1.0)
    gumbel = -torch.log(-torch.log(u))
    return torch.topk(logp + gumbel, top_k, dim=1).indices.to(torch.int32)


def random_logits(tokens: int, experts: int, seed: int = 0, ties: bool = False) -> torch.Tensor:
    """fp32 logits for top-k tests. With ties=True values are drawn from a tiny
    set so exact ties occur often (exercises the lower-index tie rule)."""
    g = _gen(seed, 12)
    if ties:
        return torch.randint(0, 4, (tokens, experts), generator=g).to(torch.float32) * 0.5
    return torch.randn(tokens, experts, generator=g, dtype=torch.float32)


def to_f64(t: torch.Tensor):
    """bf16/fp32 torch tensor -> numpy float64 (exact widening)."""
    return t.detach().to("cpu").to(torch.float64).numpy()
