"""Measured layered-vs-chunked serving on one B200 (BASELINE configs 3, 4, 5), planned and
clocked by the UNMODIFIED reference engine.

All 48 Qwen3-30B-A3B MoE layers are resident (58 GB of bf16 expert weights,
random init). `moesim.engine.run` (engine.py:272-351) plans every iteration with
the reference's own scheduler; inside `refdrive.measured_costs(executor=...)` the
iteration's BatchPlan runs through the layer stack on the GPU and the reference
engine charges the measured MoE device time (attention and dense projections
stay the reference's modelled costs on B200 peaks). Beside every
measured run the same request stream is run through the unmodified, fully
modelled reference on its own h100-like config (configs/h100like.toml, table
coverage).

  python tools/serving_bench.py --config c3        # 8192-token prompt + 32 concurrent decodes
  python tools/serving_bench.py --config c4        # chunk-size / layer-group sweep on an 8192-token prompt
  python tools/serving_bench.py --config c5 [--requests 100]   # configs/qwen_arxiv_layered.toml workload
  python tools/serving_bench.py --config c5 --gpus 8           # expert-parallel stack, one rank per GPU

With --gpus N > 1 the N ranks (started with torchrun unless WORLD_SIZE is set) each hold E/N
experts of every layer (executor.EPMoEModel: ep.PeerEP over peer memory) and run the same
reference-planned iterations on their share of each segment's rows; the MoE time charged is the
slowest rank's. Rank 0 prints. LPMOE_BENCH_SHARED_GPU=1 puts every rank on cuda:0 over gloo
(protocol check only: the ranks time-slice one GPU).

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

from paper_2510_08055_b200 import refdrive  # noqa: E402
from paper_2510_08055_b200.types import QWEN3_30B_A3B, QWEN3_30B_A3B_MODEL  # noqa: E402

ms = refdrive.import_moesim()
MODEL = refdrive.reference_model(QWEN3_30B_A3B_MODEL)
EMIT = True  # rank 0 prints
SLO = ms.types.SloSpec(ttft_slo_s=10.0, tbt_slo_s=0.125)  # configs/qwen_arxiv_layered.toml [slo]


def _h100():
    return ms.config.load_run_config(refdrive.reference_config("qwen_arxiv_layered.toml")).hardware


ATTENTION = False  # --attention: measured attention + dense projections (executor.AttentionDense)
IGRAPHS = True  # --attention + pooled KV: decode-only iterations replay one CUDA graph of all layers
KV_POOL = True  # --attention: one pooled KV tensor, one masked SDPA for all decode rows (--no-kv-pool: per request)


def run_one(stack, name, policy, chunk, target, reqs, focus=None, emit=True, graphs=0):
    from paper_2510_08055_b200.executor import AttentionDense, LayeredExecutor

    cfg = ms.types.SchedulerConfig(policy=ms.types.Policy(policy), chunk_size=chunk, group_token_target=target)
    att = None
    if ATTENTION:
        # pooled KV: one slot per request, each as long as the longest request, when that fits 48 GB
        # (C3: 33 x 8208 positions = 27 GB); otherwise per-request caches
        plen = max(r.input_len + r.output_len for r in reqs)
        slots = len(reqs) if KV_POOL and len(reqs) * plen * MODEL.num_layers * 4 * 128 * 2 * 2 <= 48e9 else 0
        att = AttentionDense(QWEN3_30B_A3B.hidden, MODEL.num_layers, stack.device, seed=11,
                             pool_slots=slots, pool_len=plen)
    ex = LayeredExecutor(stack, attention=att,
                         iteration_graphs=64 if att is not None and att.Kp is not None and IGRAPHS else 0)
    t0 = time.time()
    with refdrive.measured_costs(executor=ex):
        res = ms.engine.run(MODEL, refdrive.b200_hardware(), cfg, reqs, ms.coverage.EmpiricalTable())
    wall = time.time() - t0
    s = ms.metrics.summarize(res, SLO).to_dict()
    moe_s = sum(it["moe_s"] for it in ex.iter_log)
    out = {"run": name, "policy": policy, "chunk_size": chunk, "group_token_target": target, **s,
           "expert_load_GB": s["total_expert_load_bytes"] / 1e9, "moe_time_ms": moe_s * 1e3,
           "moe_us_per_layer_call": 1e6 * moe_s / max(1, sum(sum(1 for n in it["routed"] if n)
                                                             for it in ex.iter_log)),
           "decode_graph_tokens": graphs, "wall_s": wall,
           "kv_pool_slots": att.Kp.shape[1] if att is not None and att.Kp is not None else 0,
           "measured": "MoE + attention + dense projections (attention: PyTorch SDPA, dense: cuBLAS)" if ATTENTION
           else "MoE (attention / dense projections: the reference's roofline model on B200 peaks)"}
    if focus is not None:
        r = next(r for r in res.requests if r.id == focus)
        out["focus_ttft_s"] = r.first_token_s - r.arrival_s
        pf = [(rec, it) for rec, it in zip(res.records, ex.iter_log) if rec.prefill_tokens]
        out["prefill_iterations"] = len(pf)
        out["prefill_expert_load_GB"] = sum(rec.expert_load_bytes for rec, _ in pf) / 1e9
        out["prefill_moe_ms"] = sum(it["moe_s"] for _, it in pf) * 1e3
        # decode gaps while the long prompt was being prefilled
        gaps = [rec.runtime_s for rec, _ in pf if rec.decode_batch_size]
        out["tbt_during_prefill_mean_ms"] = 1e3 * sum(gaps) / len(gaps) if gaps else 0.0
        out["tbt_during_prefill_max_ms"] = 1e3 * max(gaps) if gaps else 0.0
    # the unmodified reference, fully modelled, on its own h100-like config, same request stream
    mres = ms.engine.run(MODEL, _h100(), cfg, reqs, ms.coverage.EmpiricalTable())
    m = ms.metrics.summarize(mres, SLO).to_dict()
    out["reference_model_h100"] = {k: m[k] for k in ("ttft_mean_s", "tbt_mean_s", "total_expert_load_bytes",
                                                     "num_iterations")}
    out["gpus"] = getattr(stack, "world", 1)
    if ATTENTION:
        # eager iterations only (a graphed decode iteration is timed as a whole, in moe_time_ms)
        out["attention_dense_ms"] = 1e3 * sum(it["attn_s"] for it in ex.iter_log)
        out["graphed_iterations"] = sum(it.get("graphed", False) for it in ex.iter_log)
    if emit and EMIT:
        print(json.dumps(out), flush=True)
    return out


def _shared_gpu() -> bool:
    return os.environ.get("LPMOE_BENCH_SHARED_GPU", "0") == "1"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", choices=["c3", "c4", "c5"], default="c3")
    ap.add_argument("--requests", type=int, default=100)
    ap.add_argument("--prompt", type=int, default=8192)
    ap.add_argument("--graph-tokens", type=int, default=16,
                    help="replay per-layer CUDA graphs for decode segments up to this many rows (0: eager)")
    ap.add_argument("--trace", default=None, help="c5: a reference trace CSV (moesim workload.export_trace) "
                                                 "instead of the config's generated workload")
    ap.add_argument("--gpus", type=int, default=1, help="expert-parallel ranks (one per GPU)")
    ap.add_argument("--attention", action="store_true",
                    help="measure attention + dense projections too (library kernels; single GPU)")
    ap.add_argument("--no-iteration-graphs", action="store_true", help="--attention: eager decode iterations")
    ap.add_argument("--no-kv-pool", action="store_true", help="--attention: per-request KV caches")
    ap.add_argument("--max-tokens", type=int, default=40960,
                    help="--gpus > 1: the largest segment (rows of one layer call, all ranks) to size EP buffers")
    a = ap.parse_args()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        import socket
        import subprocess

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        sys.exit(subprocess.call([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                  f"--nproc-per-node={a.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
                                  os.path.abspath(__file__), *sys.argv[1:]]))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    global ATTENTION, KV_POOL, IGRAPHS
    ATTENTION = a.attention
    KV_POOL = not a.no_kv_pool
    IGRAPHS = not a.no_iteration_graphs
    if ATTENTION and world > 1:
        raise SystemExit("serving_bench.py: --attention is a single-GPU mode")
    if world != a.gpus:
        raise SystemExit(f"serving_bench.py: --gpus {a.gpus} but WORLD_SIZE={world}")

    import torch

    from paper_2510_08055_b200.executor import EPMoEModel, MoEModel

    t0 = time.time()
    if world > 1:
        import torch.distributed as dist

        dev = torch.device("cuda", 0 if _shared_gpu() else int(os.environ.get("LOCAL_RANK", 0)))
        torch.cuda.set_device(dev)
        dist.init_process_group("gloo" if _shared_gpu() else "nccl")
        stack = EPMoEModel(QWEN3_30B_A3B, MODEL.num_layers, rank, world, a.max_tokens, device=dev, seed=11)
        a.graph_tokens = 0  # (per-layer graphs are a single-GPU path)
    else:
        stack = MoEModel(QWEN3_30B_A3B, MODEL.num_layers, device="cuda", seed=11, graph_tokens=a.graph_tokens)
    if stack.graphs is not None:  # decode-only layer steps replay CUDA graphs (captured up front)
        stack.graphs.capture(range(1, a.graph_tokens + 1))
    global EMIT
    EMIT = rank == 0
    if EMIT:
        print(json.dumps({"setup": "48 resident layers", "seconds": time.time() - t0, "gpus": world,
                          "experts_per_gpu": QWEN3_30B_A3B.num_experts // world,
                          "decode_graph_tokens": a.graph_tokens}), flush=True)
    g = a.graph_tokens
    R = ms.types.Request
    L = a.prompt
    if a.config == "c3":
        reqs = [R(id=i, arrival_s=0.0, input_len=128, output_len=256) for i in range(32)]
        reqs.append(R(id=32, arrival_s=0.0005, input_len=L, output_len=16))
        # untimed warm-up of the first configuration: the first layer call at each new batch
        # size grows the shared workspace and builds tensor maps (one-off host + cudaMalloc cost)
        run_one(stack, "warmup", "layered", 512, 512, reqs, focus=32, emit=False)
        for policy, chunk, target in (("layered", 512, 512), ("chunked", 512, 512), ("chunked", 2048, 512),
                                      ("hybrid", 2048, 512)):
            run_one(stack, f"c3_{policy}_c{chunk}_g{target}", policy, chunk, target, reqs, focus=32, graphs=g)
    elif a.config == "c4":
        reqs = [R(id=0, arrival_s=0.0, input_len=L, output_len=1)]
        run_one(stack, "warmup", "chunked", 8192, 512, reqs, focus=0, emit=False)
        for chunk in (512, 1024, 2048, 4096, 8192):
            if ATTENTION:  # untimed pass first: cuDNN builds an attention plan per new (chunk, context) shape
                run_one(stack, "warmup", "chunked", chunk, 512, reqs, focus=0, emit=False)
            run_one(stack, f"c4_chunked_c{chunk}", "chunked", chunk, 512, reqs, focus=0, graphs=g)
        for groups in (1, 2, 3, 4, 6, 8, 12, 16, 24, 48):
            target = math.ceil(L / groups)
            if ATTENTION:
                run_one(stack, "warmup", "layered", 512, target, reqs, focus=0, emit=False)
            run_one(stack, f"c4_layered_G{groups}", "layered", 512, target, reqs, focus=0, graphs=g)
    else:
        if a.trace:
            reqs = ms.workload.load_trace(a.trace)[: a.requests]
        else:  # the reference's own arXiv-shaped workload (lognormal 9194/5754 in, 231/104 out, 1.3 req/s)
            cfg = ms.config.load_run_config(refdrive.reference_config("qwen_arxiv_layered.toml"))
            reqs = ms.workload.generate_requests(cfg.workload)[: a.requests]
        run_one(stack, "warmup", "layered", 512, 512, reqs[:10], emit=False)
        for policy in ("layered", "chunked"):
            run_one(stack, f"c5_{policy}" + (f"_ep{world}" if world > 1 else ""), policy, 512, 512, reqs, graphs=g)
    if world > 1:
        stack.close()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
