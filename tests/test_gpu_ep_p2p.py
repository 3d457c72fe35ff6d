"""Peer-memory expert parallelism (ep.PeerEP): 2 processes on one B200, and one
process per physical GPU when the box has several.

Shared-device tests: two ranks share cuda:0: CUDA IPC maps each rank's symmetric region into the
other process exactly as it would map a peer GPU's memory over NVLink, and the
device-side barriers, fused dispatch stores and fused combine loads run for
real (contexts time-slice, so each barrier costs a scheduling quantum — this
is a protocol test, not a timing). Every rank's output must equal the
single-GPU layer (GpuMoE) on the same tokens bit for bit.

Physical-device tests (skipped on a 1-GPU box): rank r runs on cuda:r, so the
system-scope barriers, the dispatch's remote stores and the combine's remote
loads cross NVLink/NVSwitch between distinct GPUs.
"""

import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shape_name, tokens, skew, layers, q, physical=False, graph=False):
    import sys

    sys.path.insert(0, ROOT)
    try:
        import torch.distributed as dist

        from paper_2510_08055_b200 import QWEN3_30B_A3B, TINY, MoEShape
        from paper_2510_08055_b200.ep import PeerEP
        from paper_2510_08055_b200.moe import GpuMoE
        from paper_2510_08055_b200.synthetic import expert_weights, router_tokens, router_weight

        dev = torch.device("cuda", rank if physical else 0)
        torch.cuda.set_device(dev)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        from paper_2510_08055_b200 import GPT_OSS_20B

        s = {"tiny": TINY, "qwen": QWEN3_30B_A3B, "e256": MoEShape(512, 256, 256, 8, False),
             "gptoss": GPT_OSS_20B}[shape_name]
        wr = router_weight(s.num_experts, s.hidden, 21).float()
        if skew:  # every token of every rank prefers the experts of rank 0
            wr[: s.top_k, s.hidden - 1] = 16.0
        wr = wr.to(torch.bfloat16).to(dev)
        w13, w2 = expert_weights(s.num_experts, s.hidden, s.ffn, 22)
        w13, w2 = w13.to(dev), w2.to(dev)
        T = tokens[rank]
        ep = PeerEP.from_full(s, wr, w13, w2, rank, world, max_tokens=max(tokens))
        ep2 = PeerEP.from_full(s, wr, w13, w2, rank, world, max_tokens=max(tokens), region=ep.region)
        ref = GpuMoE(s, wr, w13, w2)
        ok = True
        if graph:  # two EP layers captured in ONE CUDA graph per rank (device-side sequence numbers)
            xs = router_tokens(T, s.hidden, 100 + rank).to(dev)
            y1 = torch.empty_like(xs)
            y2 = torch.empty_like(xs)
            ep(xs, out=y1)  # warm-up (tensor maps, kernel attributes) outside the capture
            ep2(y1, out=y2)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream(dev)
            side.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(side):
                g.capture_begin()
                ep(xs, out=y1)
                ep2(y1, out=y2)
                g.capture_end()
            torch.cuda.current_stream(dev).wait_stream(side)
            for it in range(layers):
                xs.copy_(router_tokens(T, s.hidden, 200 + 10 * it + rank).to(dev))
                g.replay()
                r1, _ = ref(xs)
                r2, _ = ref(r1)
                torch.cuda.synchronize()
                ok &= bool(torch.equal(y1, r1)) and bool(torch.equal(y2, r2))
            st = ep2(y1)[1]
        for it in range(0 if graph else layers):
            x = router_tokens(T, s.hidden, 100 + 10 * it + rank).to(dev)
            y, st = (ep if it % 2 == 0 else ep2)(x)
            y_ref, st_ref = ref(x)
            torch.cuda.synchronize()
            ok &= bool(torch.equal(y, y_ref))
            ok &= bool(torch.equal(st.counts, st_ref.counts))
        rows = torch.tensor([int(st.recv_rows)], dtype=torch.int64)
        dist.all_reduce(rows)
        ok &= int(rows.item()) == sum(tokens) * s.top_k  # every routing entry landed exactly once
        ep.region.close()  # collective
        dist.destroy_process_group()
        q.put((rank, ok, ""))
    except Exception as e:  # report instead of hanging the parent
        import traceback

        q.put((rank, False, traceback.format_exc()[-2000:]))


def _run(shape_name, tokens, skew=False, layers=3, world=2, physical=False, graph=False):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape_name, tokens, skew, layers, q, physical, graph))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    try:
        import queue

        for _ in range(world):
            try:
                r, ok, err = q.get(timeout=300)
            except queue.Empty:
                break  # a rank hung (typically in a device barrier after a peer failed): report what we have
            res[r] = (ok, err)
            if not ok:
                break  # its peers may now spin in a device barrier forever
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for r, (ok, err) in res.items():
        assert ok, f"rank {r}: {err}"
    for r in range(world):
        assert r in res, f"rank {r} reported nothing"


def test_peer_ep2_tiny_matches_single_gpu(cuda):
    _run("tiny", [96, 64])


def test_peer_ep2_qwen_matches_single_gpu(cuda):
    _run("qwen", [72, 40])


def test_peer_ep2_graph_captured_layers(cuda):
    """Two EP layers captured in one CUDA graph per rank and replayed on new inputs: the barrier
    and exchange sequence numbers advance on the device, so replays stay in step."""
    _run("qwen", [40, 24], graph=True)


def test_peer_ep2_skewed_to_rank0_and_empty_rank(cuda):
    _run("tiny", [80, 0], skew=True)


def test_peer_ep2_gpt_oss_shape(cuda):
    """The reference's second model config (H = I = 2880: not multiples of 128; 32 experts top-4)."""
    _run("gptoss", [300, 45])


def test_peer_ep2_large_uneven_batches_max_experts(cuda):
    """E = 256 (128 per rank), 3001 vs 7 tokens: the owners' expert kernels run large
    expert-major receive buffers (CTA-pair kernel through the staged API)."""
    _run("e256", [3001, 7], layers=1)


def test_peer_ep1_max_local_experts(cuda):
    """world 1 with E = 256 local experts: the plan kernel must write all El + 1 = 257
    receive offsets with its 256 threads (the last one is the received-row total)."""
    _run("e256", [500], layers=1, world=1)


def _gpus():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.skipif(_gpus() < 2, reason="needs 2 physical GPUs")
def test_peer_ep2_physical_gpus_qwen(cuda):
    """Two distinct GPUs: barriers, remote stores and remote loads over NVLink."""
    _run("qwen", [576, 300], physical=True)


@pytest.mark.skipif(_gpus() < 2, reason="needs 2 physical GPUs")
def test_peer_ep2_physical_gpus_skewed(cuda):
    _run("tiny", [80, 0], skew=True, physical=True)


@pytest.mark.skipif(_gpus() < 4, reason="needs 4+ physical GPUs")
def test_peer_ep_all_physical_gpus_qwen(cuda):
    """One rank per GPU on the whole box (4 or 8): every rank sends to every peer."""
    n = 8 if _gpus() >= 8 else 4
    _run("qwen", [576 - 37 * r for r in range(n)], physical=True, world=n)
