"""Shape and byte constants of the MoE layer, mirroring the reference domain types.

`ModelSpec` carries the same fields and invariants as the simulator's
(moesim/types.py:19-57) so a reference config maps 1:1 onto the GPU layer;
`MoEShape` adds what a numerical layer needs and the reference leaves
implicit: the expert FFN width I, recovered from bytes_per_expert = 3*H*I*dtype
(configs/qwen30b.toml:6), and the router's renormalisation flag.
"""

from __future__ import annotations

from dataclasses import dataclass


class ValidationError(ValueError):
    """An argument violates a documented invariant; the message names the field."""


def require(cond: bool, message: str) -> None:
    if not cond:
        raise ValidationError(message)


@dataclass(frozen=True)
class ModelSpec:
    """MoE decoder architecture constants (reference moesim/types.py:19-57)."""

    name: str
    num_layers: int
    num_experts: int
    top_k: int
    bytes_per_expert: int
    dense_bytes_per_layer: int
    flops_per_token_per_expert: int
    attn_flops_per_token_per_ctx: int
    kv_bytes_per_token: int
    hidden_dim: int
    dtype_bytes: int = 2

    def __post_init__(self):
        require(self.num_layers >= 1, f"num_layers must be >= 1, got {self.num_layers}")
        require(self.num_experts >= 1, f"num_experts must be >= 1, got {self.num_experts}")
        require(
            1 <= self.top_k <= self.num_experts,
            f"top_k out of range: need 1 <= top_k <= num_experts, got top_k={self.top_k}, "
            f"num_experts={self.num_experts}",
        )
        for name in ("bytes_per_expert", "dense_bytes_per_layer", "flops_per_token_per_expert",
                     "attn_flops_per_token_per_ctx", "kv_bytes_per_token", "hidden_dim", "dtype_bytes"):
            v = getattr(self, name)
            require(v > 0, f"{name} must be > 0, got {v}")


def total_expert_bytes(spec: ModelSpec) -> int:
    """All expert weight bytes of the model (reference types.py:70-72)."""
    return spec.num_layers * spec.num_experts * spec.bytes_per_expert


@dataclass(frozen=True)
class MoEShape:
    """One MoE layer as the kernels see it."""

    hidden: int          # H
    ffn: int             # I (per-expert intermediate width)
    num_experts: int     # E
    top_k: int           # k
    norm_topk_prob: bool = True

    def __post_init__(self):
        require(self.hidden > 0 and self.hidden % 64 == 0, f"hidden must be a positive multiple of 64, got {self.hidden}")
        require(self.ffn > 0 and self.ffn % 64 == 0, f"ffn must be a positive multiple of 64, got {self.ffn}")
        require(1 <= self.num_experts <= 256, f"num_experts must be in [1, 256], got {self.num_experts}")
        require(
            1 <= self.top_k <= min(self.num_experts, 32),
            f"top_k out of range: need 1 <= top_k <= min(num_experts, 32), got {self.top_k}",
        )

    @property
    def bytes_per_expert(self) -> int:
        """gate + up + down bf16 weights of one expert: 3*H*I*2."""
        return 3 * self.hidden * self.ffn * 2

    @property
    def flops_per_token_per_expert(self) -> int:
        return 2 * 3 * self.hidden * self.ffn

    @classmethod
    def from_model(cls, spec: ModelSpec, norm_topk_prob: bool = True) -> "MoEShape":
        denom = 3 * spec.hidden_dim * spec.dtype_bytes
        require(spec.bytes_per_expert % denom == 0,
                f"bytes_per_expert={spec.bytes_per_expert} is not 3*hidden_dim*dtype_bytes*I for integer I")
        return cls(spec.hidden_dim, spec.bytes_per_expert // denom, spec.num_experts, spec.top_k, norm_topk_prob)


# Shapes named by BASELINE.json
QWEN3_30B_A3B = MoEShape(hidden=2048, ffn=768, num_experts=128, top_k=8, norm_topk_prob=True)
TINY = MoEShape(hidden=256, ffn=128, num_experts=16, top_k=2, norm_topk_prob=True)

# The reference's second model config (configs/gptoss20b.toml: hidden 2880, MoE
# intermediate 2880, 32 experts top-4; bytes_per_expert 49,766,400 = 3*2880*2880*2).
# Shape only: the layer math is the Qwen3-MoE one (router softmax/top-k, SiLU*mul).
GPT_OSS_20B = MoEShape(hidden=2880, ffn=2880, num_experts=32, top_k=4, norm_topk_prob=True)

GPT_OSS_20B_MODEL = ModelSpec(
    name="gptoss-20b", num_layers=24, num_experts=32, top_k=4, bytes_per_expert=49766400,
    dense_bytes_per_layer=53268480, flops_per_token_per_expert=49766400, attn_flops_per_token_per_ctx=393216,
    kv_bytes_per_token=32768, hidden_dim=2880, dtype_bytes=2,
)

QWEN3_30B_A3B_MODEL = ModelSpec(
    name="qwen30b-a3b", num_layers=48, num_experts=128, top_k=8, bytes_per_expert=9437184,
    dense_bytes_per_layer=38273024, flops_per_token_per_expert=9437184, attn_flops_per_token_per_ctx=786432,
    kv_bytes_per_token=49152, hidden_dim=2048, dtype_bytes=2,
)
