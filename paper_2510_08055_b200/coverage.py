"""Coverage models with the reference's `CoverageModel` protocol, plus the measured one.

The reference engine asks `coverage_model.coverage(routed_tokens, rng)` for the
fraction of experts a routed batch touches and charges
`moe_cost(model, routed, coverage, layers)` (moesim/engine.py:144-154,
cli.py:222-223). Mirrored here with the same names, arguments, determinism and
error behaviour (moesim/coverage.py:99-257):

* `UniformAnalytic` / `EmpiricalTable` — closed forms (coverage.py:216-237);
* `Sampled` — Monte Carlo routing surrogate; the per-slab uniforms are drawn on
  the host with the caller's rng exactly as coverage.py:113-137 does, and the
  union counts run on the B200 (`lp_union_counts_*`, bit-identical to the
  reference's numba kernels), so a given rng state yields the reference's
  numbers;
* `MeasuredCoverage` — SURVEY §8(f)2, `coverage.kind = "measured"`: the
  coverage is read off a real routed layer call on the GPU (nnz of the
  per-expert counts / E), and `measured_cost` returns the reference's
  `KernelCost`-shaped record with the measured device time in place of
  `kernel_runtime` (costmodel.py:57-85, :148-152).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import costmodel as cm
from . import kernels
from .types import ModelSpec, ValidationError, require

_MAX_TOKENS_PER_SLAB = 65_536  # coverage.py:110


def rank_power_weights(num_experts: int, skew_exponent: float) -> np.ndarray:
    """Expert popularity ~ (rank+1)^(-skew) (coverage.py:101-106)."""
    require(skew_exponent >= 0, f"skew_exponent must be >= 0, got {skew_exponent}")
    require(skew_exponent <= 64, f"skew_exponent must be <= 64, got {skew_exponent}")
    ranks = np.arange(num_experts, dtype=np.float64) + 1.0
    return ranks ** (-skew_exponent)


def sample_union_counts(batch: int, top_k: int, num_experts: int, skew_exponent: float, rng: np.random.Generator,
                        trials: int) -> np.ndarray:
    """Per-trial distinct-expert counts; same rng consumption as coverage.py:113-137."""
    counts = np.empty(trials, dtype=np.int64)
    weights = rank_power_weights(num_experts, skew_exponent) if skew_exponent > 0 else None
    trials_per_slab = max(1, _MAX_TOKENS_PER_SLAB // max(batch, 1))
    done = 0
    while done < trials:
        n = min(trials_per_slab, trials - done)
        u = rng.random((n, batch, top_k))
        if weights is None:
            c = kernels.uniform_union_counts(u, batch, top_k, num_experts)
        else:
            c = kernels.weighted_union_counts(u, batch, top_k, num_experts, weights)
        counts[done:done + n] = c.cpu().numpy() if isinstance(c, torch.Tensor) else c
        done += n
    return counts


@dataclass(frozen=True)
class ActivationResult:
    coverage_fraction: float
    experts_activated: float
    tokens_per_active_expert: float


def sample_activation(batch: int, top_k: int, num_experts: int, skew_exponent: float, rng: np.random.Generator,
                      trials: int = 1) -> ActivationResult:
    """Mean activation stats over `trials` sampled batches (coverage.py:140-169)."""
    require(batch >= 0, f"batch must be >= 0, got {batch}")
    require(trials >= 1, f"trials must be >= 1, got {trials}")
    require(1 <= top_k <= num_experts,
            f"top_k out of range: need 1 <= top_k <= num_experts, got top_k={top_k}, num_experts={num_experts}")
    if batch == 0:
        return ActivationResult(0.0, 0.0, 0.0)
    counts = sample_union_counts(batch, top_k, num_experts, skew_exponent, rng, trials)
    routed = batch * top_k
    return ActivationResult(coverage_fraction=float(counts.mean()) / num_experts,
                            experts_activated=float(counts.mean()),
                            tokens_per_active_expert=float((routed / counts).mean()))


@dataclass(frozen=True)
class UniformAnalytic:
    """Closed-form independence model (coverage.py:216-224)."""

    top_k: int
    num_experts: int

    def coverage(self, routed_tokens: int, rng: np.random.Generator | None = None) -> float:
        return cm.expected_coverage_uniform(routed_tokens, self.top_k, self.num_experts)


@dataclass(frozen=True)
class EmpiricalTable:
    """Interpolated measured curve (coverage.py:227-237)."""

    table: tuple[tuple[int, float], ...] = cm.DEFAULT_COVERAGE_TABLE

    def __post_init__(self):
        cm.check_table(self.table)

    def coverage(self, routed_tokens: int, rng: np.random.Generator | None = None) -> float:
        return cm.coverage_from_table(routed_tokens, self.table)


@dataclass(frozen=True)
class Sampled:
    """One Monte Carlo draw per query on the GPU sampler (coverage.py:240-254)."""

    top_k: int
    num_experts: int
    skew_exponent: float = 0.0
    trials: int = 1

    def coverage(self, routed_tokens: int, rng: np.random.Generator | None = None) -> float:
        if rng is None:
            raise ValidationError("Sampled coverage model requires an rng")
        return sample_activation(routed_tokens, self.top_k, self.num_experts, self.skew_exponent, rng,
                                 self.trials).coverage_fraction


@dataclass
class MeasuredCoverage:
    """Coverage and MoE cost measured on a real GpuMoE layer.

    `coverage(routed_tokens, rng)` routes `routed_tokens` hidden rows through the
    layer (rows drawn from `hidden` — e.g. the engine's current hybrid batch —
    or synthetic N(0,1) rows when None) and returns nnz(counts)/E. The device
    time of that call is kept for `measured_cost`.
    """

    layer: object                       # GpuMoE
    hidden: torch.Tensor | None = None  # [N, H] bf16 rows to route (cycled if N < routed_tokens)
    seed: int = 0
    last_device_s: float = field(default=0.0, init=False)
    last_routed: int = field(default=-1, init=False)   # routed_tokens of the last coverage() call
    last_experts_hit: int = field(default=0, init=False)

    def _rows(self, n: int) -> torch.Tensor:
        dev = self.layer.device
        H = self.layer.shape.hidden
        if self.hidden is None:
            g = torch.Generator(device=dev).manual_seed(self.seed + n)
            return torch.randn((n, H), generator=g, device=dev).to(torch.bfloat16)
        reps = -(-n // self.hidden.shape[0])
        return self.hidden.repeat(reps, 1)[:n].contiguous() if reps > 1 else self.hidden[:n].contiguous()

    def coverage(self, routed_tokens: int, rng: np.random.Generator | None = None) -> float:
        require(routed_tokens >= 0, f"routed_tokens must be >= 0, got {routed_tokens}")
        x = self._rows(routed_tokens)
        stream = torch.cuda.current_stream(self.layer.device)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _, stats = self.layer(x)
        e1.record(stream)
        e1.synchronize()
        self.last_device_s = e0.elapsed_time(e1) * 1e-3
        self.last_routed = routed_tokens
        self.last_experts_hit = stats.experts_hit
        return self.last_experts_hit / self.layer.shape.num_experts

    def measured_cost(self, model: ModelSpec, routed_tokens: int, layers_in_scope: int) -> cm.Kernel:
        """`moe_cost` (costmodel.py:57-85) with measured coverage and device time.

        Coverage and time come from one real layer call on `routed_tokens` rows;
        bytes and flops follow the reference formulas (:77-79) and the runtime is
        the measured time times the layers in scope (same batch per layer).
        """
        cov = self.coverage(routed_tokens)
        k = cm.moe_cost(model, routed_tokens, cov, layers_in_scope)
        return cm.Kernel(k.kind, k.flops, k.hbm_bytes, k.expert_weight_bytes,
                         measured_s=self.last_device_s * layers_in_scope)


CoverageModel = UniformAnalytic | EmpiricalTable | Sampled | MeasuredCoverage
