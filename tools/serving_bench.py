"""Measured layered-vs-chunked serving on one B200 (BASELINE configs 3, 4, 5).

All 48 Qwen3-30B-A3B MoE layers are resident (58 GB of bf16 expert weights,
random init); every planned iteration runs its MoE work on the GPU
(executor.MeasuredCost) and charges the measured device time; attention and
dense projections are modelled on B200 peaks.

  python tools/serving_bench.py --config c3        # 8192-token prompt + 32 concurrent decodes
  python tools/serving_bench.py --config c4        # chunk-size / layer-group sweep on an 8192-token prompt
  python tools/serving_bench.py --config c5 [--requests 100]   # arXiv-length trace (plans.json)

Prints one JSON object per run on stdout.
"""

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2510_08055_b200.types import QWEN3_30B_A3B, QWEN3_30B_A3B_MODEL  # noqa: E402
from paper_2510_08055_b200 import costmodel as cm  # noqa: E402
from paper_2510_08055_b200 import serving as sv  # noqa: E402


def run_one(stack, name, policy, chunk, target, reqs, focus=None, emit=True):
    from paper_2510_08055_b200.executor import MeasuredCost

    cost = MeasuredCost(QWEN3_30B_A3B_MODEL, stack)
    t0 = time.time()
    recs, done, makespan = sv.run(QWEN3_30B_A3B_MODEL, cm.B200_MODELLED, sv.Planner(policy, chunk, target), reqs, cost)
    wall = time.time() - t0
    s = sv.summarize(recs, done, makespan)
    out = {"run": name, "policy": policy, "chunk_size": chunk, "group_token_target": target, **s,
           "expert_load_GB": s["total_expert_load_bytes"] / 1e9, "moe_time_ms": s["moe_time_s"] * 1e3,
           "wall_s": wall}
    if focus is not None:
        r = next(r for r in done if r.id == focus)
        out["focus_ttft_s"] = r.first_token_s - r.arrival_s
        pf = [rec for rec in recs if rec.prefill_tokens]
        out["prefill_iterations"] = len(pf)
        out["prefill_expert_load_GB"] = sum(rec.expert_load_bytes for rec in pf) / 1e9
        out["prefill_moe_ms"] = sum(rec.moe_runtime_s for rec in pf) * 1e3
        # decode gaps while the long prompt was being prefilled
        gaps = [rec.runtime_s for rec in pf if rec.decode_batch_size]
        out["tbt_during_prefill_mean_ms"] = 1e3 * sum(gaps) / len(gaps) if gaps else 0.0
        out["tbt_during_prefill_max_ms"] = 1e3 * max(gaps) if gaps else 0.0
    # modelled reference numbers for the same plan stream (costmodel on h100-like, table coverage)
    mrecs, mdone, mspan = sv.run(QWEN3_30B_A3B_MODEL, cm.H100_LIKE, sv.Planner(policy, chunk, target), reqs)
    ms = sv.summarize(mrecs, mdone, mspan)
    out["reference_model_h100"] = {k: ms[k] for k in ("ttft_mean_s", "tbt_mean_s", "total_expert_load_bytes",
                                                      "num_iterations")}
    if emit:
        print(json.dumps(out), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", choices=["c3", "c4", "c5"], default="c3")
    ap.add_argument("--requests", type=int, default=100)
    ap.add_argument("--prompt", type=int, default=8192)
    ap.add_argument("--graph-tokens", type=int, default=0,
                    help="capture per-layer CUDA graphs for decode segments up to this many rows (0: eager)")
    ap.add_argument("--trace", default=None, help="c5: a reference trace CSV (workload.export_trace) instead of "
                                                 "the committed arXiv request fixture")
    a = ap.parse_args()

    from paper_2510_08055_b200.executor import MoEModel

    t0 = time.time()
    stack = MoEModel(QWEN3_30B_A3B, QWEN3_30B_A3B_MODEL.num_layers, device="cuda", seed=11,
                     graph_tokens=a.graph_tokens)
    if stack.graphs is not None:  # decode-only layer steps replay CUDA graphs (captured up front)
        stack.graphs.capture(range(1, a.graph_tokens + 1))
    print(json.dumps({"setup": "48 resident layers", "seconds": time.time() - t0,
                      "decode_graph_tokens": a.graph_tokens}), flush=True)
    L = a.prompt
    if a.config == "c3":
        reqs = [sv.Request(i, 0.0, 128, 256) for i in range(32)] + [sv.Request(32, 0.0005, L, 16)]
        # untimed warm-up of the first configuration: the first layer call at each new batch
        # size grows the shared workspace and builds tensor maps (one-off host + cudaMalloc cost)
        run_one(stack, "warmup", "layered", 512, 512, reqs, focus=32, emit=False)
        for policy, chunk, target in (("layered", 512, 512), ("chunked", 512, 512), ("chunked", 2048, 512),
                                      ("hybrid", 2048, 512)):
            run_one(stack, f"c3_{policy}_c{chunk}_g{target}", policy, chunk, target, reqs, focus=32)
    elif a.config == "c4":
        reqs = [sv.Request(0, 0.0, L, 1)]
        run_one(stack, "warmup", "chunked", 8192, 512, reqs, focus=0, emit=False)
        for chunk in (512, 1024, 2048, 4096, 8192):
            run_one(stack, f"c4_chunked_c{chunk}", "chunked", chunk, 512, reqs, focus=0)
        for groups in (1, 2, 3, 4, 6, 8, 12, 16, 24, 48):
            target = math.ceil(L / groups)
            run_one(stack, f"c4_layered_G{groups}", "layered", 512, target, reqs, focus=0)
    else:
        if a.trace:
            reqs = sv.load_trace(a.trace)[: a.requests]
        else:
            gold = json.load(open(os.path.join(ROOT, "tests", "golden", "plans.json")))
            reqs = [sv.Request(i, t, li, lo) for i, t, li, lo in gold["arxiv"]["requests"][: a.requests]]
        run_one(stack, "warmup", "layered", 512, 512, reqs[:10], emit=False)
        for policy in ("layered", "chunked"):
            run_one(stack, f"c5_{policy}", policy, 512, 512, reqs)


if __name__ == "__main__":
    main()
