"""Seeded synthetic inputs shared by tests, bench and the oracle.

No checkpoints or datasets exist offline, so the layer runs on random-init
weights of the Qwen3-30B-A3B MoE shape. Router inputs are drawn on a dyadic
grid so every fp32 logit is exact in any summation order:

  x[t, h]  = a / 8,   a in {-4..4}      (exact in bf16)
  Wr[e, h] = b / 64,  b in {-4..4}      (exact in bf16)
  x[:, H-1] = 1,  Wr[e, H-1] = (E-1-e) * 2**-tb   (tie-breaker, < 1/512)

Every product is a multiple of 1/512, |logit| <= 16*(H-1)/512 and the
tie-breaker resolution is 2**-tb, so for H <= 2048 and E <= 256 a logit needs
at most 23 significant bits: exact in fp32 whatever the order of the sum, and
pairwise distinct, so the CPU oracle and the tensor-core router agree on the
top-k bit for bit. Expert weights are N(0, std^2) rounded to bf16; the oracle
consumes exactly those rounded values in fp32.
"""

from __future__ import annotations

import math

import torch


def tie_break_shift(num_experts: int) -> int:
    # (E-1) * 2**-shift < 2**-9 (one grid step of x*Wr)
    return 9 + max(1, math.ceil(math.log2(max(num_experts, 2))))


def router_weight(E: int, H: int, seed: int, tie_break: bool = True) -> torch.Tensor:
    """wr [E, H] bf16 on the dyadic grid (b/64) with the tie-breaker column."""
    g = torch.Generator().manual_seed(seed)
    wr = torch.randint(-4, 5, (E, H), generator=g, dtype=torch.int32).to(torch.float32) / 64.0
    wr[:, H - 1] = (E - 1 - torch.arange(E, dtype=torch.float32)) * 2.0 ** (-tie_break_shift(E)) if tie_break else 0.0
    return wr.to(torch.bfloat16)


def router_tokens(T: int, H: int, seed: int, tie_break: bool = True) -> torch.Tensor:
    """x [T, H] bf16 on the dyadic grid (a/8); column H-1 is 1 (tie-breaker on) or 0."""
    g = torch.Generator().manual_seed(seed)
    x = torch.randint(-4, 5, (T, H), generator=g, dtype=torch.int32).to(torch.float32) / 8.0
    x[:, H - 1] = 1.0 if tie_break else 0.0
    return x.to(torch.bfloat16)


def expert_weights(E: int, H: int, I: int, seed: int, std: float = 0.02,
                   device: str | torch.device = "cpu") -> tuple[torch.Tensor, torch.Tensor]:
    """(w13 [E,2I,H], w2 [E,H,I]) bf16, N(0, std^2)."""
    g = torch.Generator(device=device).manual_seed(seed)
    w13 = torch.empty((E, 2 * I, H), dtype=torch.bfloat16, device=device)
    w2 = torch.empty((E, H, I), dtype=torch.bfloat16, device=device)
    # fill expert by expert to bound the fp32 temporary
    for e in range(E):
        w13[e] = (torch.randn((2 * I, H), generator=g, device=device) * std).to(torch.bfloat16)
        w2[e] = (torch.randn((H, I), generator=g, device=device) * std).to(torch.bfloat16)
    return w13, w2


def hidden_states(T: int, H: int, seed: int, device: str | torch.device = "cpu") -> torch.Tensor:
    """Generic N(0,1) bf16 activations (routing not exact-by-construction)."""
    g = torch.Generator(device=device).manual_seed(seed)
    return torch.randn((T, H), generator=g, device=device).to(torch.bfloat16)
