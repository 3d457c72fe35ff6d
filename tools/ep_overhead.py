"""Peer-memory EP machinery cost on ONE GPU: ep.PeerEP with world size 1 (exchange, dispatch into the
own receive buffer, two device barriers, expert kernel on the received rows, fused combine) against
the single-GPU layer (GpuMoE, 4 launches) on the same tokens and weights, CUDA-event timed, 8 layer
weight sets rotated (inputs larger than L2). Outputs must be bit-identical.

    python tools/ep_overhead.py [T ...]
"""
import json
import os
import socket
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2510_08055_b200 import QWEN3_30B_A3B as s  # noqa: E402
from paper_2510_08055_b200.ep import PeerEP  # noqa: E402
from paper_2510_08055_b200.moe import GpuMoE  # noqa: E402
from paper_2510_08055_b200.synthetic import router_tokens, router_weight  # noqa: E402


def timed(fn, steps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    e0.record()
    for i in range(steps):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / steps


def main():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    Ts = [int(a) for a in sys.argv[1:]] or [1, 8, 64, 576, 2048]
    sets = []
    for i in range(8):
        g = torch.Generator(device=dev).manual_seed(i)
        w13 = (torch.randn((s.num_experts, 2 * s.ffn, s.hidden), generator=g, device=dev) * 0.02).to(torch.bfloat16)
        w2 = (torch.randn((s.num_experts, s.hidden, s.ffn), generator=g, device=dev) * 0.02).to(torch.bfloat16)
        sets.append((router_weight(s.num_experts, s.hidden, i).to(dev), w13, w2))
    region = None
    for T in Ts:
        x = router_tokens(T, s.hidden, 7).to(dev)
        single = [GpuMoE(s, *w) for w in sets]
        eps = []
        for w in sets:
            ep = PeerEP(s, w[0], w[1], w[2], 0, 1, max_tokens=max(Ts), region=region)
            region = ep.region
            eps.append(ep)
        y1 = torch.empty_like(x)
        y2 = torch.empty_like(x)
        t_single = timed(lambda i: single[i % 8](x, out=y1), 40)
        t_ep = timed(lambda i: eps[i % 8](x, out=y2), 40)
        single[0](x, out=y1)
        eps[0](x, out=y2)
        torch.cuda.synchronize()
        same = bool(torch.equal(y1, y2))
        import time
        t0 = time.perf_counter()
        for i in range(20):
            eps[i % 8](x, out=y2)
        host_us = (time.perf_counter() - t0) * 1e6 / 20  # host time per call (no sync inside)
        torch.cuda.synchronize()
        # stage split of the EP layer (events at PeerEP's stage boundaries, one layer at a time)
        names = ["route+permute", "exchange+dispatch+barrier", "experts+barrier", "combine"]
        acc = [0.0] * 4
        for i in range(20):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
            eps[i % 8](x, out=y2, prof=ev)
            torch.cuda.synchronize()
            for j in range(4):
                acc[j] += ev[j].elapsed_time(ev[j + 1]) * 1e3 / 20
        print(json.dumps({"T": T, "single_gpu_layer_us": round(t_single, 1), "peer_ep_world1_us": round(t_ep, 1),
                          "ep_overhead_us": round(t_ep - t_single, 1), "bit_identical": same, "host_us_per_call": round(host_us, 1),
                          "ep_stages_us": {n: round(v, 1) for n, v in zip(names, acc)}}), flush=True)
    region.close()
    dist.destroy_process_group()


def micro():
    """Per-launch device time of the EP control kernels alone (world size 1)."""
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    wr = router_weight(s.num_experts, s.hidden, 1).to(dev)
    w13 = torch.zeros((s.num_experts, 2 * s.ffn, s.hidden), dtype=torch.bfloat16, device=dev)
    w2 = torch.zeros((s.num_experts, s.hidden, s.ffn), dtype=torch.bfloat16, device=dev)
    ep = PeerEP(s, wr, w13, w2, 0, 1, max_tokens=576)
    rg = ep.region
    st = torch.cuda.current_stream(dev).cuda_stream
    counts = torch.randint(0, 40, (s.num_experts,), dtype=torch.int32, device=dev)
    out = {}
    for name, fn in (("exchange", lambda: rg.exchange(counts, st)), ("barrier", lambda: rg.barrier(st))):
        out[name + "_us"] = round(timed(lambda i: fn(), 200), 2)
    print(json.dumps(out), flush=True)
    rg.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    if "--micro" in sys.argv:
        micro()
    else:
        main()
