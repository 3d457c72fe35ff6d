"""Layered executor on the B200: real MoE layers driven by the serving planner.

SURVEY §8(d) C1 criterion: layered and chunked prefill run the same per-token
math, so every prompt's final hidden states must agree — on this GPU path they
are bit-identical (per-token routing and per-column tcgen05 accumulation do not
depend on which other tokens share the batch).
"""

import pytest
import torch

from paper_2510_08055_b200 import costmodel as cm
from paper_2510_08055_b200 import serving as sv
from paper_2510_08055_b200.executor import MeasuredCost, MoEModel
from paper_2510_08055_b200.types import TINY, ModelSpec

pytestmark = pytest.mark.gpu

TINY_MODEL = ModelSpec(name="tiny-moe", num_layers=4, num_experts=16, top_k=2, bytes_per_expert=196608,
                       dense_bytes_per_layer=524288, flops_per_token_per_expert=196608,
                       attn_flops_per_token_per_ctx=4096, kv_bytes_per_token=4096, hidden_dim=256)


@pytest.fixture(scope="module")
def stack(cuda):
    return MoEModel(TINY, 4, device=cuda, seed=3)


def _run(stack, policy, reqs, chunk=512, target=512):
    cost = MeasuredCost(TINY_MODEL, stack, keep_final_prompt=True)
    recs, done, makespan = sv.run(TINY_MODEL, cm.B200_MODELLED, sv.Planner(policy, chunk, target), reqs, cost)
    return recs, done, makespan, cost


def test_layered_equals_chunked_final_hidden(stack):
    reqs = [sv.Request(i, 0.0, n, 4) for i, n in enumerate((1024, 700, 300))]
    lay = _run(stack, "layered", reqs)
    chk = _run(stack, "chunked", reqs)
    hyb = _run(stack, "hybrid", reqs, chunk=256)
    for rid in range(3):
        a = lay[3].final_prompt[rid]
        assert torch.equal(a, chk[3].final_prompt[rid]), rid
        assert torch.equal(a, hyb[3].final_prompt[rid]), rid
        assert a.abs().max().item() > 0


def test_measured_iterations_follow_the_modelled_plan(stack):
    reqs = [sv.Request(i, 0.0, n, 6) for i, n in enumerate((1024, 64, 64))]
    recs, done, _, cost = _run(stack, "layered", reqs)
    ref, rdone, _ = sv.run(TINY_MODEL, cm.B200_MODELLED, sv.Planner("layered", 512, 512), reqs)
    assert len(recs) == len(ref) and len(done) == 3
    assert [r.prefill_tokens for r in recs] == [r.prefill_tokens for r in ref]
    for rec, log in zip(recs, cost.iter_log):
        assert log["moe_s"] > 0
        assert rec.moe_runtime_s == log["moe_s"]
        # each layer's experts hit never exceed E and cover at least top_k when tokens are routed
        for n, h in zip(log["routed"], log["experts_hit"]):
            assert (h == 0) == (n == 0) and h <= 16 and (n == 0 or h >= 2)
        assert rec.expert_load_bytes == sum(log["experts_hit"]) * TINY_MODEL.bytes_per_expert


def test_decode_graphs_match_eager(cuda):
    """Per-layer CUDA graphs for decode-size segments (MoEModel(graph_tokens=...)) give the
    same hidden states, routing and expert bytes as eager calls."""
    # all arrivals at t=0: the plan stream cannot depend on the measured (graph vs eager) timings
    reqs = [sv.Request(i, 0.0, n, 7) for i, n in enumerate((700, 40, 300, 5))]
    eager = MoEModel(TINY, 4, device=cuda, seed=3)
    graphed = MoEModel(TINY, 4, device=cuda, seed=3, graph_tokens=16)
    res = []
    for stack in (eager, graphed):
        cost = MeasuredCost(TINY_MODEL, stack, keep_final_prompt=True)
        recs, done, _ = sv.run(TINY_MODEL, cm.B200_MODELLED, sv.Planner("layered", 512, 512), reqs, cost)
        res.append((recs, cost))
    (ra, ca), (rb, cb) = res
    assert len(graphed.graphs.graphs) > 0
    assert [r.expert_load_bytes for r in ra] == [r.expert_load_bytes for r in rb]
    assert [g["experts_hit"] for g in ca.iter_log] == [g["experts_hit"] for g in cb.iter_log]
    for rid in range(4):
        assert torch.equal(ca.final_prompt[rid], cb.final_prompt[rid]), rid
        last = [c.final_decode.get(rid, c.decode_row.get(rid)) for c in (ca, cb)]  # finished / still live
        assert last[0] is not None and torch.equal(last[0], last[1]), rid
