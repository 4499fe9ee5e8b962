"""torch.autograd wrapper of the C-ABI layer (SURVEY §8(b) "Python layer: a
torch.autograd.Function calls moe_forward / moe_backward and owns the
moe_saved tensors").

`DroplessMoEFunction` is argument marshalling only: the forward is one
`moe_forward` call (router, topology, padded gather, SDD + act, DSD, weighted
scatter: Fig. 5), the backward one `moe_backward` call (the §5.1
operation list). Both run in libmoe.so's kernels; the saved
tensors (`api.Saved`) live on the autograd context between the two.
`DroplessMoE` is the module holding the three weights (router Wr [h, E],
W1 [h, E*f], W2 [E*f, h] in bf16, P:272-276 with reading R1).
"""
from __future__ import annotations

import math

import torch

from . import api


class DroplessMoEFunction(torch.autograd.Function):
    """y = dMoE(x; wr, w1, w2) on x [T, h] bf16 (contiguous, CUDA).

    Gradients: dx, dWr (computed in fp32 by the library, returned in wr's
    dtype), dW1, dW2. With aux_loss_coeff > 0 the forward also computes the
    auxiliary load-balancing loss into the workspace and the
    backward adds its router gradient as if that loss were added to the
    objective (d objective / d aux = 1, the usual way it is trained); its
    value is returned through `stats["aux_loss"]` (a detached device scalar)."""

    @staticmethod
    def forward(ctx, x, wr, w1, w2, opts: dict, stats: dict | None):
        cfg = api.make_config(x.shape[0], x.shape[1], wr.shape[1], opts["top_k"], opts["ffn_hidden"],
                              opts.get("block_size", 128), opts.get("act", api.ACT_GELU),
                              renormalize=opts.get("renormalize", False),
                              aux_loss_coeff=opts.get("aux_loss_coeff", 0.0))
        x = x.contiguous()
        y, saved = api.moe_forward(cfg, wr, w1, w2, x)
        if stats is not None and cfg.aux_loss_coeff > 0:
            stats["aux_loss"] = api.aux_region(cfg, saved.ws)[0:1].clone()
        if stats is not None:
            stats["expert_idx"] = saved.expert_idx
        ctx.cfg, ctx.saved_moe = cfg, saved
        ctx.save_for_backward(x, wr, w1, w2)
        return y

    @staticmethod
    def backward(ctx, dy):
        x, wr, w1, w2 = ctx.saved_tensors
        dx, (dwr, dw1, dw2) = api.moe_backward(ctx.cfg, wr, w1, w2, ctx.saved_moe, x,
                                               dy.to(torch.bfloat16).contiguous())
        ctx.saved_moe = None
        return dx, dwr.to(wr.dtype), dw1, dw2, None, None


class DroplessMoE(torch.nn.Module):
    """The dropless MoE FFN layer (Fig. 1, Fig. 5) as a module.

    x [..., hidden] bf16 -> y [..., hidden] bf16. Weights are initialised
    like the synthetic workloads (DESIGN.md input recipe): Wr, W1 ~ N(0, 1/h),
    W2 ~ N(0, 1/f). `self.stats` holds the last forward's expert_idx and (with
    aux_loss_coeff > 0) aux_loss."""

    def __init__(self, hidden: int, num_experts: int, top_k: int, ffn_hidden: int, act: int = api.ACT_GELU,
                 block_size: int = 128, renormalize: bool = False, aux_loss_coeff: float = 0.0,
                 device="cuda", generator: torch.Generator | None = None):
        super().__init__()
        bf = torch.bfloat16

        def normal(shape, std):
            return (torch.randn(*shape, generator=generator) * std).to(bf).to(device)
        self.wr = torch.nn.Parameter(normal((hidden, num_experts), 1 / math.sqrt(hidden)))
        self.w1 = torch.nn.Parameter(normal((hidden, num_experts * ffn_hidden), 1 / math.sqrt(hidden)))
        self.w2 = torch.nn.Parameter(normal((num_experts * ffn_hidden, hidden), 1 / math.sqrt(ffn_hidden)))
        self.opts = dict(top_k=top_k, ffn_hidden=ffn_hidden, block_size=block_size, act=act,
                         renormalize=renormalize, aux_loss_coeff=aux_loss_coeff)
        self.stats: dict = {}

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        shape = x.shape
        self.stats = {}
        y = DroplessMoEFunction.apply(x.reshape(-1, shape[-1]), self.wr, self.w1, self.w2, self.opts, self.stats)
        return y.reshape(shape)
