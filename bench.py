#!/usr/bin/env python
"""Benchmark of the MoE-layer hot path (BASELINE.json metric, config 2).

Workload (BASELINE.json configs[1]): one Qwen3-30B-A3B MoE layer
(E=128, top-8, H=2048, I=768) over a hybrid batch of 64 decode + 512 prefill
tokens = T=576 routed tokens, random-init bf16 weights, synthetic dyadic
inputs. One "step" = one full layer forward (router, top-k, permute, grouped
expert FFN, combine). Eight distinct layer weight sets (9.7 GB) are rotated
step to step, so every step streams its expert weights from HBM (inputs far
larger than the 126 MB L2).

  value  : device-timed µs per layer step, inputs resident in HBM (lower is better)
  e2e    : the same through GpuMoE.forward_host with pinned host x / y, H2D+D2H inside
  roofline: dominant kernel (the expert kernel) vs measured HBM copy bandwidth, or vs the measured
            dense bf16 peak when the batch is above the ridge (tensor-bound)
  cpu_baseline: the fp32 oracle port timed on this host's cores

Multi-GPU (torchrun, N>1): each rank runs its own T=576 batch (tokens
data-parallel) with the experts it owns (expert-parallel, E/N per rank) and
NCCL all-to-all dispatch/return (paper_2510_08055_b200.ep); value = max over
ranks of the per-step time, "scaling": "weak".

`--impl reference` times the reference's CPU path for the same workload
(the oracle port of the layer; the reference has no numerical layer) on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MoE layer us/iter (Qwen3-30B-A3B, 64 decode + 512 prefill tokens)"
UNIT = "us/iter"
T_DECODE, T_PREFILL = 64, 512
N_LAYER_SETS = 8
N_INPUTS = 4
GRAPHED_E2E_T = 2  # e2e at or below this many tokens: one CUDA graph per call (moe.GraphedHostStep); B200:
# T=1 / 2 48.4 / 60.5 vs 61.0 / 62.9 us pipelined, but T=4 / 8 / 16 73.5 / 110.2 / 147.0 vs 70.8 / 90.2 / 132.0 —
# in-graph copies serialise with the layer, where the pipeline overlaps them with neighbouring steps


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--tokens", type=int, default=T_DECODE + T_PREFILL)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shape", choices=["qwen", "gptoss"], default="qwen",
                    help="layer shape: Qwen3-30B-A3B (the BASELINE metric) or the reference's GPT-OSS-20B config")
    ap.add_argument("--ep", choices=["p2p", "nccl"], default="p2p",
                    help="N>1 exchange: fused dispatch/combine over peer memory (ep.PeerEP) or NCCL all_to_all")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling around the timed region (B200_PROFILING.md clocks line).

    Started before the warm-up so the 100 ms sampler is already running when
    the (often only tens of ms long) timed region starts; each sample is
    stamped with host time and summary() keeps those inside the timed window
    (padded by one sampling period), falling back to the whole busy phase.
    """

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None
        self.err = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except FileNotFoundError as exc:
            self.err = str(exc)
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.monotonic(), [c.strip() for c in line.split(",")]))

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.th.join(timeout=2)
            if not self.rows:
                self.err = (self.proc.stderr.read() or "no samples")[:200]

    def summary(self, t0: float, t1: float):
        def num(v):
            try:
                return float(v)
            except ValueError:
                return None

        win = [r for t, r in self.rows if t0 - 0.06 <= t <= t1 + 0.06]
        window = "timed"
        if not win:
            win = [r for _, r in self.rows]
            window = "run"
        if not win:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "error": self.err}
        sm = [num(r[1]) for r in win if len(r) > 2 and num(r[1]) is not None]
        mx = [num(r[2]) for r in win if len(r) > 2 and num(r[2]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in win if len(r) >= 9 for n, v in zip(names, r[5:9]) if v == "Active"})
        pw = [num(r[3]) for r in win if len(r) > 3 and num(r[3]) is not None]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "power_w": statistics.median(pw) if pw else None, "power_max_w": max(pw) if pw else None,
                "reasons": reasons, "samples": len(win), "window": window}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def measured_tensor_peak():
    """Dense bf16 TFLOP/s: the burst figure (the expert kernel is timed alone per launch)."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        if "bf16_tflops" in d:
            return float(d["bf16_tflops"]), "measured (MEASURED_PEAKS.json bf16_tflops, burst)"
    return 2250.0, "fallback (nominal dense bf16 2.25 PF/s)"


def ncu_traffic(T: int, kernel: str = "k_experts"):
    """DRAM bytes per launch of the dominant kernel at this T from the latest committed `ncu --set
    full` capture (profiles/rNN/k_experts_traffic.json, written by tools/summarize_evidence.py)."""
    import glob

    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "k_experts_traffic.json")), reverse=True):
        d = json.load(open(path)).get(f"{kernel}_{T}")
        if d:
            return d["dram_bytes_per_launch"], os.path.relpath(path, ROOT)
    return None, None


# ----------------------------------------------------------------------------- CPU legs
def cpu_layer_inputs(T: int, seed: int = 0):
    from paper_2510_08055_b200 import QWEN3_30B_A3B as s
    from paper_2510_08055_b200.synthetic import expert_weights, router_tokens, router_weight

    wr = router_weight(s.num_experts, s.hidden, seed).float().numpy()
    w13, w2 = expert_weights(s.num_experts, s.hidden, s.ffn, seed + 1)
    x = router_tokens(T, s.hidden, seed + 2).float().numpy()
    return x, wr, w13.float().numpy(), w2.float().numpy(), s


def time_cpu_oracle(T: int, seconds: float, max_iters: int | None = None):
    """The oracle port of the layer on all host cores: µs per layer forward."""
    import torch

    from oracle import moe_oracle

    cores = os.cpu_count() or 1
    torch.set_num_threads(cores)
    x, wr, w13, w2, s = cpu_layer_inputs(T)
    moe_oracle.moe_forward(x, wr, w13, w2, s.top_k, s.norm_topk_prob)  # warm
    times = []
    t_end = time.perf_counter() + seconds
    while (max_iters is None and time.perf_counter() < t_end) or (max_iters is not None and len(times) < max_iters):
        t0 = time.perf_counter()
        moe_oracle.moe_forward(x, wr, w13, w2, s.top_k, s.norm_topk_prob)
        times.append(time.perf_counter() - t0)
    return statistics.median(times) * 1e6, cores, len(times)


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    T = args.tokens
    from oracle import moe_oracle

    x, wr, w13, w2, s = cpu_layer_inputs(T)
    for _ in range(args.warmup):
        moe_oracle.moe_forward(x, wr, w13, w2, s.top_k, s.norm_topk_prob)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        moe_oracle.moe_forward(x, wr, w13, w2, s.top_k, s.norm_topk_prob)
    dt = (time.perf_counter() - t0) / args.steps
    v = dt * 1e6
    cores = os.cpu_count() or 1
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
        "config": {"workload": f"qwen3-30b-a3b MoE layer, T={T} ({T_DECODE} decode + {T - T_DECODE} prefill)",
                   "tokens": T, "hidden": 2048, "ffn": 768, "experts": 128, "top_k": 8},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{args.steps} full layer forwards (fp32 numpy oracle, all {cores} host threads; "
                                   "the reference moesim has no numerical layer, only moe_cost)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU leg
def run_ours(args, rank: int, world: int):
    import torch
    import torch.distributed as dist

    from paper_2510_08055_b200 import GPT_OSS_20B, QWEN3_30B_A3B
    from paper_2510_08055_b200 import _native
    from paper_2510_08055_b200.moe import GpuMoE
    from paper_2510_08055_b200.synthetic import router_tokens, router_weight

    local = _local_device()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    clocks = ClockSampler(local).start()
    T = args.tokens
    s = GPT_OSS_20B if args.shape == "gptoss" else QWEN3_30B_A3B
    lib = _native.load()

    if world > 1:
        from paper_2510_08055_b200.ep import EPMoE, PeerEP
    layers = []
    for i in range(N_LAYER_SETS):
        g = torch.Generator(device=dev).manual_seed(1000 + i)
        wr = router_weight(s.num_experts, s.hidden, 1000 + i).to(dev)
        w13 = (torch.randn((s.num_experts, 2 * s.ffn, s.hidden), generator=g, device=dev) * 0.02).to(torch.bfloat16)
        w2 = (torch.randn((s.num_experts, s.hidden, s.ffn), generator=g, device=dev) * 0.02).to(torch.bfloat16)
        if world > 1:
            if args.ep == "p2p":  # one symmetric IPC region shared by the layer sets (layers run in sequence)
                layers.append(PeerEP.from_full(s, wr, w13, w2, rank, world, max_tokens=T,
                                               region=layers[0].region if layers else None))
            else:
                layers.append(EPMoE.from_full(s, wr, w13, w2, rank, world))
        else:
            layers.append(GpuMoE(s, wr, w13, w2))
        del g
    xs = [router_tokens(T, s.hidden, 50 + rank * N_INPUTS + i).to(dev) for i in range(N_INPUTS)]
    xs_host = [x.cpu().pin_memory() for x in xs]
    ys = [torch.empty_like(xs[0]) for _ in range(N_INPUTS)]
    torch.cuda.synchronize()

    def step(i):
        return layers[i % N_LAYER_SETS](xs[i % N_INPUTS], out=ys[i % N_INPUTS])

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- warmup: W steps, then keep stepping (untimed) until ~0.5 s of load so
    # clocks reach steady state before the timed region
    for i in range(max(args.warmup, 3)):
        step(i)
    torch.cuda.synchronize()
    t_w = time.perf_counter()
    i = 0
    while time.perf_counter() - t_w < 0.5:
        step(i)
        i += 1
        if i % 50 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()

    # ---- timed region (device events on the launching stream) with live stage events
    stream = torch.cuda.current_stream(dev)
    K = args.steps
    stage_ev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(K)]
    for evs in stage_ev:  # materialise the cudaEvent_t handles
        for e in evs:
            e.record(stream)
    torch.cuda.synchronize()
    ptr_arrays = []
    for evs in stage_ev:
        import ctypes

        arr = (ctypes.c_void_p * 5)(*[e.cuda_event for e in evs])
        ptr_arrays.append(arr)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    # timed region: plain back-to-back steps (stage events would split the PDL chain)
    t_region0 = time.monotonic()
    n_launch0 = lib.lp_launch_count()
    start.record(stream)
    for i in range(K):
        step(i)
    end.record(stream)
    n_launches = lib.lp_launch_count() - n_launch0
    torch.cuda.synchronize()
    t_region1 = time.monotonic()
    clocks.stop()
    # profiling pass over the same K steps: events at the stage boundaries (this
    # serialises the stages, so per-stage times include each kernel's launch)
    peer = world > 1 and args.ep == "p2p"
    if world == 1:
        for i in range(K):
            lib.lp_profile_events(ptr_arrays[i], 5)
            step(i)
        lib.lp_profile_events(None, 0)
        torch.cuda.synchronize()
    elif peer:  # PeerEP records its own stage boundaries
        barrier()
        for i in range(K):
            layers[i % N_LAYER_SETS](xs[i % N_INPUTS], out=ys[i % N_INPUTS], prof=stage_ev[i])
        torch.cuda.synchronize()
    barrier()
    ms = start.elapsed_time(end) / K
    if world > 1:
        t = torch.tensor([ms], device="cpu" if _shared_gpu() else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # per-stage device time (single GPU: route | permute | experts | combine; PeerEP: route+permute |
    # counts+dispatch (with their barriers) | experts (+ barrier) | combine (+ barrier)); max over ranks
    stage_us = None
    if world == 1 or peer:
        names = ["route", "permute", "experts", "combine"] if world == 1 else \
            ["route_permute", "dispatch", "experts", "combine"]
        sums = [0.0] * 4
        for evs in stage_ev:
            for j in range(4):
                sums[j] += evs[j].elapsed_time(evs[j + 1])
        if world > 1:
            t = torch.tensor(sums, dtype=torch.float64, device="cpu" if _shared_gpu() else dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            sums = t.cpu().tolist()
        stage_us = {n: 1e3 * v / K for n, v in zip(names, sums)}

    # ---- end-to-end through the public API with host buffers: every step uploads
    # its input from pinned host memory and downloads its result; the copies of
    # neighbouring steps overlap the layer compute (HostPipeline, two copy streams)
    # decode sizes (T <= GRAPHED_E2E_T): one CUDA graph per call (GraphedHostStep: H2D, layer, D2H),
    # since a few KiB of copies cost less than the host side of an event-ordered submit
    y_host = torch.empty((T, s.hidden), dtype=torch.bfloat16, pin_memory=True)
    e2e_layers = layers if world == 1 else None
    graphed_e2e = world == 1 and T <= GRAPHED_E2E_T
    if graphed_e2e:
        from paper_2510_08055_b200.moe import GraphedHostStep

        pipe = GraphedHostStep(dev, T, s.hidden)
        for i in range(K):  # capture every (layer, input) pair the timed loop uses, outside it
            pipe.prepare(layers[i % N_LAYER_SETS], xs_host[i % N_INPUTS], y_host)
        for i in range(3):
            pipe.submit(layers[i % N_LAYER_SETS], xs_host[i % N_INPUTS], y_host)
    elif world == 1:
        from paper_2510_08055_b200.moe import HostPipeline

        pipe = HostPipeline(dev, T, s.hidden)
        for i in range(3):
            pipe.submit(layers[i % N_LAYER_SETS], xs_host[i % N_INPUTS], y_host)
        pipe.drain()
    else:
        x_dev = torch.empty((T, s.hidden), dtype=torch.bfloat16, device=dev)
        for i in range(3):
            layers[i % N_LAYER_SETS].forward_host(xs_host[i % N_INPUTS], y_host, x_dev=x_dev)
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    if graphed_e2e:
        for i in range(K):
            pipe.submit(layers[i % N_LAYER_SETS], xs_host[i % N_INPUTS], y_host)
    elif e2e_layers is not None:
        pipe.start(e0)
        for i in range(K):
            pipe.submit(layers[i % N_LAYER_SETS], xs_host[i % N_INPUTS], y_host)
        pipe.drain()
    else:
        for i in range(K):
            layers[i % N_LAYER_SETS].forward_host(xs_host[i % N_INPUTS], y_host, x_dev=x_dev)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / K
    if world > 1:
        t = torch.tensor([e2e_ms], device="cpu" if _shared_gpu() else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    # ---- per-call latency through the public API: one synchronous forward_host per step
    # (H2D of x, the layer, D2H of y, nothing overlapped) — what a single caller waits for
    x_dev1 = torch.empty((T, s.hidden), dtype=torch.bfloat16, device=dev)
    lat = []
    barrier()
    for i in range(max(3, min(K, 20))):
        l0, l1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0.record(stream)
        layers[i % N_LAYER_SETS].forward_host(xs_host[i % N_INPUTS], y_host, x_dev=x_dev1)
        l1.record(stream)
        torch.cuda.synchronize()
        if i >= 2:
            lat.append(l0.elapsed_time(l1))
    lat_ms = statistics.median(lat)
    if world > 1:
        t = torch.tensor([lat_ms], device="cpu" if _shared_gpu() else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        lat_ms = float(t.item())

    # routing stats for the roofline (same inputs as the timed steps): experts this rank's kernel
    # streams (single GPU: all hit experts; EP: the hit experts it owns) and rows it processes
    hits, rows = [], []
    for i in range(N_LAYER_SETS):
        _, st = layers[i](xs[i % N_INPUTS])
        if world == 1:
            hits.append(st.experts_hit)
            rows.append(T * s.top_k)
        else:
            c = st.counts.to(torch.int64)
            c = c.cpu() if _shared_gpu() else c
            dist.all_reduce(c)
            el = s.num_experts // world
            mine = c[rank * el:(rank + 1) * el]
            hits.append(int((mine > 0).sum()))
            rows.append(int(mine.sum()))
    torch.cuda.synchronize()

    if rank != 0:
        return
    peak, peak_src = measured_peaks()
    out = {
        "metric": METRIC if args.shape == "qwen" else METRIC.replace("Qwen3-30B-A3B", "GPT-OSS-20B shape"),
        "value": ms * 1e3, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": f"synthetic (random-init {'Qwen3-30B-A3B' if args.shape == 'qwen' else 'GPT-OSS-20B'}-shaped "
                "weights, dyadic-grid tokens)",
        "config": {"workload": f"{'qwen3-30b-a3b' if args.shape == 'qwen' else 'gpt-oss-20b-shaped'} MoE layer, "
                               f"T={T} ({min(T, T_DECODE)} decode + {max(T - T_DECODE, 0)} prefill)",
                   "tokens": T, "hidden": s.hidden, "ffn": s.ffn, "experts": s.num_experts, "top_k": s.top_k,
                   "parallelism": f"ep{world}" if world > 1 else "single",
                   "ep_exchange": (("peer-memory fused dispatch/combine (CUDA IPC, NVLink P2P)" if args.ep == "p2p"
                                    else "NCCL all_to_all_single") if world > 1 else None),
                   "l2": f"inputs larger than L2: {N_LAYER_SETS} layer weight sets "
                         f"({N_LAYER_SETS * s.num_experts * s.bytes_per_expert / 1e9:.1f} GB) rotated per step"},
        "e2e": {"value": e2e_ms * 1e3, "unit": UNIT, "h2d_bytes_per_step": T * s.hidden * 2,
                "d2h_bytes_per_step": T * s.hidden * 2,
                "note": ("one CUDA graph per step: H2D of the step's pinned input, the layer, D2H of y "
                         "(moe.GraphedHostStep), steps back to back" if graphed_e2e else
                         "pipelined: step i's H2D/D2H overlap neighbouring steps' layers (moe.HostPipeline)")
                        if world == 1 else "one forward_host per step (H2D, EP layer, D2H), back to back"},
        "e2e_latency": {"value": lat_ms * 1e3, "unit": UNIT, "h2d_bytes_per_step": T * s.hidden * 2,
                        "d2h_bytes_per_step": T * s.hidden * 2,
                        "note": "one synchronous forward_host call (H2D of x, layer, D2H of y, no overlap), "
                                "median, max over ranks"},
        # our kernels launched inside the timed region, counted by liblpmoe (lp_launch_count):
        # single GPU 4 per step (router, scan+slots, experts, combine) in the gather regime,
        # 5 with x_perm (router, scan, scatter, experts, combine); EP adds its plan/dispatch/
        # combine kernels and barriers (NCCL's own kernels are not counted)
        "gpu_launches": n_launches,
        "clocks": clocks.summary(t_region0, t_region1),
    }
    if stage_us is not None:
        nnz = statistics.mean(hits)
        R = statistics.mean(rows)  # token rows through this rank's expert kernel
        # single GPU (gather regime): the kernel reads each token row from x once and writes y_perm rows
        # at slot granularity; with EP the rows it reads are the received ones
        algo_bytes = nnz * s.bytes_per_expert + (2 * T * s.hidden * 2 if world == 1 else 2 * R * s.hidden * 2)
        t_kernel = stage_us["experts"]
        achieved = algo_bytes / (t_kernel * 1e-6) / 1e9
        decode = world == 1 and n_launches == K  # one launch per step: the fused decode-size kernel ran
        traffic, traffic_src = ncu_traffic(T, "k_decode" if decode else "k_experts")
        if traffic_src:
            traffic_src += " (ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum per launch)"
        layer_bytes = nnz * s.bytes_per_expert + s.num_experts * s.hidden * 2 + 2 * T * s.hidden * 2 + T * s.top_k * 8
        flops = 2.0 * R * 3 * s.hidden * s.ffn  # expert GEMMs (gate/up + down) of this rank's rows
        tpeak, tpeak_src = measured_tensor_peak()
        kernel = ("k_experts / k_experts_pair (grouped gate/up+SiLU*mul and down, tcgen05); duration from CUDA "
                  "events around its launch in a second pass over the same K steps")
        if decode:
            kernel = ("k_decode (the whole decode-size layer in one launch: routing, permutation, expert stream, "
                      "combine); duration from CUDA events around it in a second pass over the same K steps")
            stage_us = {"decode_kernel": stage_us["experts"]}
        if flops / algo_bytes > tpeak * 1e12 / (peak * 1e9):
            # arithmetic intensity above the measured ridge: the expert kernel is tensor-bound
            tf = flops / (t_kernel * 1e-6) / 1e12
            out["roofline"] = {"bound": "tensor", "kernel": kernel, "achieved": tf, "peak": tpeak, "unit": "TFLOP/s",
                               "frac": tf / tpeak, "traffic": traffic, "traffic_source": traffic_src,
                               "peak_source": tpeak_src, "algo_flops_per_launch": flops,
                               "algo_bytes_per_launch": algo_bytes,
                               "hbm_frac": achieved / peak}
        else:
            out["roofline"] = {"bound": "hbm", "kernel": kernel,
                               "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                               "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
                               "algo_bytes_per_launch": algo_bytes,
                               "layer_frac": (layer_bytes / (ms * 1e-3)) / 1e9 / peak}
        if world > 1:
            out["roofline"]["per_rank"] = (f"rank {rank}: its {s.num_experts // world} experts ({nnz:g} hit) and "
                                           f"{R:g} received rows; stage times max over ranks")
            out["roofline"].pop("layer_frac", None)
        out["stages_us"] = stage_us
        out["experts_hit_mean"] = nnz
    if not args.no_cpu_baseline and world == 1:  # the CPU baseline is a rank-0, N=1 measurement
        v, cores, n = time_cpu_oracle(T, args.cpu_seconds)
        out["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                               "sample": f"median of {n} full T={T} layer forwards of the fp32 numpy oracle "
                                         f"(torch/BLAS threads={cores}); reference moesim has no numerical layer"}
    print(json.dumps(out), flush=True)


def _shared_gpu() -> bool:
    return os.environ.get("LPMOE_BENCH_SHARED_GPU", "0") == "1"


def _local_device() -> int:
    return 0 if _shared_gpu() else int(os.environ.get("LOCAL_RANK", 0))


def _free_port() -> int:
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        # `python bench.py --gpus N` without a launcher: start the N ranks ourselves (torchrun, one
        # process per GPU, rendezvous on 127.0.0.1) and exit with their status
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__),
               *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "ours" and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(_local_device())
        # LPMOE_BENCH_SHARED_GPU=1 (protocol testing only): every rank on cuda:0 over gloo, so the
        # N>1 path (peer-memory EP over CUDA IPC) runs end to end on a one-GPU box; its timings
        # are meaningless (the ranks' contexts time-slice one GPU)
        dist.init_process_group("gloo" if _shared_gpu() else "nccl")
    try:
        run_ours(args, rank, world)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
