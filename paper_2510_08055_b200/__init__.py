"""B200-native MoE-layer hot path for layered-prefill serving (arXiv 2510.08055).

The reference (`moesim`) cost-models the MoE layer of a hybrid decode+prefill
batch; this package runs it: router/top-k, permutation, tcgen05 grouped expert
FFN and combine on sm_100a through the C ABI in include/lpmoe.h, plus the
reference-facing adapters (coverage models, union-count sampler).
"""

from .types import GPT_OSS_20B, MoEShape, ModelSpec, QWEN3_30B_A3B, TINY, ValidationError  # noqa: F401

__version__ = "0.1.0"
