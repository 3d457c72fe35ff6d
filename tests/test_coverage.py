"""Coverage models with the reference CoverageModel protocol (paper_2510_08055_b200/coverage.py).

Golden values: tests/golden/coverage_sampled.json, produced by the reference
itself (moesim.coverage, numba backend) by tests/golden/make_coverage.py.
The closed forms run on CPU; `Sampled` runs its union counts on the GPU and
must reproduce the reference's numbers from the same rng seeds exactly.
"""

import json
import os

import numpy as np
import pytest

from paper_2510_08055_b200 import coverage as cv
from paper_2510_08055_b200.types import ValidationError

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "coverage_sampled.json")))


def test_closed_forms_match_reference():
    for b, c in GOLD["uniform"]:
        assert cv.UniformAnalytic(8, 128).coverage(b) == c
    for b, c in GOLD["table"]:
        assert cv.EmpiricalTable().coverage(b) == c


def test_protocol_errors_mirror_reference():
    with pytest.raises(ValidationError, match="requires an rng"):
        cv.Sampled(8, 128).coverage(8, None)
    with pytest.raises(ValidationError, match="skew_exponent"):
        cv.rank_power_weights(128, -1.0)
    with pytest.raises(ValidationError, match="top_k out of range"):
        cv.sample_activation(8, 200, 128, 0.0, np.random.default_rng(0))
    assert cv.sample_activation(0, 8, 128, 0.0, np.random.default_rng(0)) == cv.ActivationResult(0.0, 0.0, 0.0)


@pytest.mark.gpu
@pytest.mark.parametrize("case", GOLD["sampled"], ids=lambda c: f"B{c['batch']}k{c['top_k']}s{c['skew']}")
def test_sampled_on_gpu_reproduces_reference(cuda, case):
    r = cv.sample_activation(case["batch"], case["top_k"], case["num_experts"], case["skew"],
                             np.random.default_rng(case["seed"]), case["trials"])
    assert r.coverage_fraction == case["coverage_fraction"]
    assert r.experts_activated == case["experts_activated"]
    assert r.tokens_per_active_expert == case["tokens_per_active_expert"]
    model = cv.Sampled(case["top_k"], case["num_experts"], case["skew"], case["trials"])
    assert model.coverage(case["batch"], np.random.default_rng(case["seed"])) == case["coverage_fraction"]


@pytest.mark.gpu
def test_measured_coverage_is_the_layer_routing(cuda):
    import torch

    from oracle import moe_oracle as mo
    from paper_2510_08055_b200 import QWEN3_30B_A3B as s
    from paper_2510_08055_b200.moe import GpuMoE
    from paper_2510_08055_b200.types import QWEN3_30B_A3B_MODEL
    from paper_2510_08055_b200.synthetic import expert_weights, router_tokens, router_weight

    wr = router_weight(s.num_experts, s.hidden, 3)
    w13, w2 = expert_weights(s.num_experts, s.hidden, s.ffn, 4)
    layer = GpuMoE(s, wr.to(cuda), w13.to(cuda), w2.to(cuda))
    for T in (1, 8, 32, 200):
        x = router_tokens(T, s.hidden, 10 + T)
        m = cv.MeasuredCoverage(layer, hidden=x.to(cuda))
        c = m.coverage(T)
        ids = mo.route(x.float().numpy(), wr.float().numpy(), s.top_k, s.norm_topk_prob)[0]
        assert c == len(np.unique(ids)) / s.num_experts
        k = m.measured_cost(QWEN3_30B_A3B_MODEL, T, 3)
        assert k.measured_s > 0 and k.expert_weight_bytes == m.last_experts_hit * s.bytes_per_expert * 3
    torch.cuda.synchronize()
