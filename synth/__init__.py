"""Seeded synthetic input generators (no method arithmetic; see inputs.py)."""
from .inputs import (CONFIGS, MoEShape, make_inputs, random_expert_idx, random_logits,
                     to_f64, uniform_expert_idx)

__all__ = ["CONFIGS", "MoEShape", "make_inputs", "random_expert_idx", "random_logits",
           "to_f64", "uniform_expert_idx"]
