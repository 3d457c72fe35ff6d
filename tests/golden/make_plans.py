"""Plan-stream and engine fixtures from the REFERENCE simulator (moesim), for the
host-side planner/engine restatement (paper_2510_08055_b200/serving.py).

Run only in the build container (needs /root/reference); called by
make_golden.py or directly:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_plans.py

Writes tests/golden/plans.json:
  scenarios[name] = {model, hw, policy, chunk_size, group_token_target, requests,
                     iterations: [[decode_ids, assignments, runtime_s, expert_load_bytes]],
                     summary: {...}}
  arxiv: the 100-request arXiv-length trace of configs/qwen_arxiv_*.toml (seed 2)
         and the reference's summaries for chunked / layered / hybrid on it.
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

QWEN = dict(name="qwen30b-a3b", num_layers=48, num_experts=128, top_k=8, bytes_per_expert=9437184,
            dense_bytes_per_layer=38273024, flops_per_token_per_expert=9437184, attn_flops_per_token_per_ctx=786432,
            kv_bytes_per_token=49152, hidden_dim=2048, dtype_bytes=2)
# BASELINE config 1: 4 MoE layers, 16 experts top-2, d=256, ffn=128 (bytes_per_expert = 3*256*128*2)
TINY = dict(name="tiny-moe", num_layers=4, num_experts=16, top_k=2, bytes_per_expert=196608,
            dense_bytes_per_layer=524288, flops_per_token_per_expert=196608, attn_flops_per_token_per_ctx=4096,
            kv_bytes_per_token=4096, hidden_dim=256, dtype_bytes=2)
H100 = dict(name="h100-like", peak_flops=989e12, peak_hbm_bw=3.35e12, mfu=0.6, mbu=0.8, static_power_w=100.0,
            energy_per_flop_j=5e-13, energy_per_hbm_byte_j=5e-11, kv_capacity_bytes=40e9, iteration_overhead_s=2e-3)


def _run(model, hw, policy, chunk, target, requests, coverage=None):
    from moesim.coverage import EmpiricalTable
    from moesim.engine import run
    from moesim.metrics import summarize
    from moesim.types import HardwareSpec, ModelSpec, Policy, SchedulerConfig, SloSpec

    m = ModelSpec(**model)
    h = HardwareSpec(**hw)
    cfg = SchedulerConfig(policy=Policy(policy), chunk_size=chunk, group_token_target=target)
    res = run(m, h, cfg, requests, coverage or EmpiricalTable(), seed=7)
    summ = summarize(res, SloSpec(ttft_slo_s=10.0, tbt_slo_s=0.125)).to_dict()
    return res, summ


def _record_iterations(model, hw, policy, chunk, target, requests):
    """Re-run with a wrapped planner to capture every BatchPlan."""
    import moesim.engine as eng

    plans = []
    orig = eng.plan_for

    def spy(state, cfg):
        p = orig(state, cfg)
        plans.append(p)
        return p

    eng.plan_for = spy
    try:
        res, summ = _run(model, hw, policy, chunk, target, requests)
    finally:
        eng.plan_for = orig
    its = []
    for p, rec in zip(plans, res.records):
        its.append([list(p.decode_ids),
                    [[a.request_id, a.token_start, a.token_end, a.layer_start, a.layer_end]
                     for a in p.prefill_assignments],
                    rec.runtime_s, rec.expert_load_bytes])
    return its, summ


def make_plans(path):
    from moesim.types import Request
    from moesim.workload import LogNormalLengths, WorkloadConfig, generate_requests

    out = {"scenarios": {}}
    small = generate_requests(WorkloadConfig(request_rate_rps=1.3, seed=2, num_requests=12,
                                             length_dist=LogNormalLengths(9194, 5754, 231, 104)))
    small = [Request(id=r.id, arrival_s=r.arrival_s, input_len=r.input_len, output_len=min(r.output_len, 40))
             for r in small]
    reqs_small = [[r.id, r.arrival_s, r.input_len, r.output_len] for r in small]
    for policy, chunk, target in (("chunked", 512, 512), ("layered", 512, 512), ("hybrid", 2048, 512),
                                  ("chunked", 2048, 512), ("layered", 512, 2048)):
        its, summ = _record_iterations(QWEN, H100, policy, chunk, target, small)
        out["scenarios"][f"qwen_{policy}_c{chunk}_g{target}"] = dict(
            model=QWEN, hw=H100, policy=policy, chunk_size=chunk, group_token_target=target,
            requests=reqs_small, iterations=its, summary=summ)
    tiny_reqs = [Request(id=i, arrival_s=0.05 * i, input_len=1024, output_len=8) for i in range(3)]
    for policy in ("chunked", "layered", "hybrid"):
        its, summ = _record_iterations(TINY, H100, policy, 512, 512, tiny_reqs)
        out["scenarios"][f"tiny_{policy}"] = dict(
            model=TINY, hw=H100, policy=policy, chunk_size=512, group_token_target=512,
            requests=[[r.id, r.arrival_s, r.input_len, r.output_len] for r in tiny_reqs], iterations=its,
            summary=summ)

    arxiv = generate_requests(WorkloadConfig(request_rate_rps=1.3, seed=2, num_requests=100,
                                             length_dist=LogNormalLengths(9194, 5754, 231, 104)))
    arx = {"requests": [[r.id, r.arrival_s, r.input_len, r.output_len] for r in arxiv], "summaries": {}}
    for policy in ("chunked", "layered"):
        _, summ = _run(QWEN, H100, policy, 512, 512, arxiv)
        arx["summaries"][policy] = summ
    out["arxiv"] = arx
    with open(path, "w") as f:
        json.dump(out, f)
    print("plans.json:", {k: len(v["iterations"]) for k, v in out["scenarios"].items()},
          {k: (v["ttft_mean_s"], v["num_iterations"]) for k, v in arx["summaries"].items()})


if __name__ == "__main__":
    make_plans(os.path.join(HERE, "plans.json"))
