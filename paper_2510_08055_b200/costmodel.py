"""Roofline cost arithmetic and the coverage curves the coverage models need.

Host-side restatement of the reference's cost arithmetic (the a2/a5 rows of
SURVEY §8) for the package's own coverage models (coverage.py), which must run
on the GPU box without the reference installed:

  moe_cost        costmodel.py:57-85   expert bytes = cov*E*bytes_per_expert*layers
  attention_cost  costmodel.py:88-125
  dense_cost      costmodel.py:128-145
  kernel_runtime  costmodel.py:148-152 max(flops/(peak*mfu), bytes/(bw*mbu))
  coverage        coverage.py:38-89    closed form, tokens/expert, table interpolation

Floating-point operations are issued in the reference's order (pinned against
reference outputs by tests/test_coverage.py and tests/test_types.py). Serving
runs use the reference's own engine and cost model (refdrive.py), not this file.
"""

from __future__ import annotations

import math
from bisect import bisect_left
from dataclasses import dataclass

from .types import ModelSpec, require

MOE, ATTN_PREFILL, ATTN_DECODE, DENSE = "moe_ffn", "attention_prefill", "attention_decode", "dense_proj"


@dataclass(frozen=True)
class HardwareSpec:
    """Accelerator coefficients (reference types.py:75-112)."""

    name: str
    peak_flops: float
    peak_hbm_bw: float
    mfu: float = 0.6
    mbu: float = 0.8
    kv_capacity_bytes: float = 40e9
    iteration_overhead_s: float = 0.0

    def __post_init__(self):
        for f in ("peak_flops", "peak_hbm_bw", "mfu", "mbu", "kv_capacity_bytes"):
            require(getattr(self, f) > 0, f"{f} must be > 0, got {getattr(self, f)}")
        require(self.mfu <= 1.0 and self.mbu <= 1.0, "mfu and mbu must be <= 1")
        require(self.iteration_overhead_s >= 0, "iteration_overhead_s must be >= 0")


H100_LIKE = HardwareSpec("h100-like", 989e12, 3.35e12, 0.6, 0.8, 40e9, 2e-3)          # configs/h100like.toml
# B200 peaks from MEASURED_PEAKS.json with the reference's default mfu/mbu; used for the
# modelled (non-MoE) kernels of measured runs. KV budget: 180 GB minus 58 GB of expert weights.
B200_MODELLED = HardwareSpec("b200", 1660.8e12, 6556.5e9, 0.6, 0.8, 100e9, 0.0)


@dataclass(frozen=True)
class Kernel:
    kind: str
    flops: float
    hbm_bytes: float
    expert_weight_bytes: float = 0.0
    measured_s: float | None = None  # device time when the kernel was actually run


def moe_cost(model: ModelSpec, routed_tokens: int, coverage_fraction: float, layers_in_scope: int) -> Kernel:
    require(routed_tokens >= 0, f"routed_tokens must be >= 0, got {routed_tokens}")
    require(0.0 <= coverage_fraction <= 1.0, f"coverage_fraction must be in [0,1], got {coverage_fraction}")
    require(1 <= layers_in_scope <= model.num_layers,
            f"layers_in_scope must be in [1, num_layers], got {layers_in_scope}")
    expert = coverage_fraction * model.num_experts * model.bytes_per_expert * layers_in_scope
    act = 2.0 * routed_tokens * model.hidden_dim * model.dtype_bytes * layers_in_scope
    flops = float(routed_tokens * model.top_k * model.flops_per_token_per_expert * layers_in_scope)
    return Kernel(MOE, flops, expert + act, expert)


def attention_cost(model: ModelSpec, new_tokens: int, context_len: int, decode_kv_tokens: int,
                   decode_new_tokens: int = 0, layers_in_scope: int | None = None) -> Kernel:
    layers = model.num_layers if layers_in_scope is None else layers_in_scope
    require(1 <= layers <= model.num_layers, f"layers_in_scope out of range: {layers}")
    frac = layers / model.num_layers
    flops, nbytes, kind = 0.0, 0.0, ATTN_DECODE
    if new_tokens > 0:
        kind = ATTN_PREFILL
        pairs = new_tokens * (context_len + (new_tokens - 1) / 2.0 + 1.0)
        flops += model.attn_flops_per_token_per_ctx * pairs * frac
        nbytes += (context_len + new_tokens) * model.kv_bytes_per_token * frac
        nbytes += new_tokens * model.kv_bytes_per_token * frac
    if decode_kv_tokens > 0 or decode_new_tokens > 0:
        flops += model.attn_flops_per_token_per_ctx * decode_kv_tokens * frac
        nbytes += decode_kv_tokens * model.kv_bytes_per_token * frac
        nbytes += decode_new_tokens * model.kv_bytes_per_token * frac
    return Kernel(kind, flops, nbytes)


def dense_cost(model: ModelSpec, tokens: int, layers_in_scope: int) -> Kernel:
    params = model.dense_bytes_per_layer / model.dtype_bytes
    flops = 2.0 * params * tokens * layers_in_scope
    weights = float(model.dense_bytes_per_layer * layers_in_scope)
    act = 2.0 * tokens * model.hidden_dim * model.dtype_bytes * layers_in_scope
    return Kernel(DENSE, flops, weights + act)


def kernel_runtime(k: Kernel, hw: HardwareSpec) -> float:
    if k.measured_s is not None:
        return k.measured_s
    return max(k.flops / (hw.peak_flops * hw.mfu), k.hbm_bytes / (hw.peak_hbm_bw * hw.mbu))


def iteration_runtime(kernels: list[Kernel], hw: HardwareSpec) -> float:
    return sum(kernel_runtime(k, hw) for k in kernels)


# ------------------------------------------------------------------ coverage curves (coverage.py:24-89)
DEFAULT_COVERAGE_TABLE: tuple[tuple[int, float], ...] = (
    (1, 0.0625), (2, 0.117), (4, 0.213), (8, 0.290), (16, 0.445),
    (32, 0.547), (64, 0.694), (128, 0.863), (256, 0.934), (512, 0.98),
)


def expected_coverage_uniform(batch: int, top_k: int, num_experts: int) -> float:
    """1 - (1 - k/E)^B: each expert is missed by one uniform top-k draw with prob 1 - k/E."""
    require(batch >= 0, f"batch must be >= 0, got {batch}")
    require(1 <= top_k <= num_experts, f"top_k out of range: need 1 <= top_k <= num_experts, got top_k={top_k}, "
                                       f"num_experts={num_experts}")
    return 1.0 - (1.0 - top_k / num_experts) ** batch


def tokens_per_expert(batch: int, top_k: int, num_experts: int) -> float:
    require(batch >= 0, f"batch must be >= 0, got {batch}")
    return batch * top_k / num_experts


def check_table(table) -> None:
    require(len(table) > 0, "coverage table must be non-empty")
    pb, pc = 0, -1.0
    for b, c in table:
        require(b > pb, f"coverage table batch sizes must be strictly increasing at B={b}")
        require(c >= pc, f"coverage table must be nondecreasing in coverage at B={b}")
        require(0.0 <= c <= 1.0, f"coverage fraction must be in [0,1], got {c} at B={b}")
        pb, pc = b, c


def coverage_from_table(batch: int, table=DEFAULT_COVERAGE_TABLE) -> float:
    """Log-linear interpolation in B, clamped to the end points; B=0 -> 0."""
    require(batch >= 0, f"batch must be >= 0, got {batch}")
    if batch == 0:
        return 0.0
    bs = [b for b, _ in table]
    cs = [c for _, c in table]
    if batch <= bs[0]:
        return cs[0]
    if batch >= bs[-1]:
        return cs[-1]
    hi = bisect_left(bs, batch)
    if bs[hi] == batch:
        return cs[hi]
    lo = hi - 1
    t = (math.log(batch) - math.log(bs[lo])) / (math.log(bs[hi]) - math.log(bs[lo]))
    return cs[lo] + (cs[hi] - cs[lo]) * t
