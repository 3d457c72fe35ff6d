"""Expert-parallel layer stack under the unmodified reference engine (BASELINE config 5's EP path).

Two processes share one B200 (CUDA IPC maps each rank's PeerRegion exactly as it would map a peer
GPU's memory over NVLink; contexts time-slice, so this is a protocol test, not a timing). Each rank
holds half the experts of every layer (executor.EPMoEModel over ep.PeerEP), the reference engine
plans the same iterations on both ranks, and every iteration's rows are split over the ranks and
gathered back. The final hidden states must equal the single-GPU stack's (executor.MoEModel, same
seed) bit for bit, and the experts hit per layer must match.
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


def _model(ms, shape_name):
    if shape_name == "tiny":
        return ms.types.ModelSpec(name="tiny-moe", num_layers=4, num_experts=16, top_k=2, bytes_per_expert=196608,
                                  dense_bytes_per_layer=524288, flops_per_token_per_expert=196608,
                                  attn_flops_per_token_per_ctx=4096, kv_bytes_per_token=4096, hidden_dim=256)
    import dataclasses

    from paper_2510_08055_b200 import refdrive
    from paper_2510_08055_b200.types import QWEN3_30B_A3B_MODEL

    return dataclasses.replace(refdrive.reference_model(QWEN3_30B_A3B_MODEL), num_layers=4)  # 4-layer Qwen stack


def _engine_run(stack, policy, lens, out, shape_name="tiny"):
    from paper_2510_08055_b200 import refdrive
    from paper_2510_08055_b200.executor import LayeredExecutor

    ms = refdrive.import_moesim()
    model = _model(ms, shape_name)
    cfg = ms.types.SchedulerConfig(policy=ms.types.Policy(policy), chunk_size=512, group_token_target=512)
    reqs = [ms.types.Request(id=i, arrival_s=0.0, input_len=n, output_len=out) for i, n in enumerate(lens)]
    ex = LayeredExecutor(stack, keep_final_prompt=True)
    with refdrive.measured_costs(executor=ex):
        res = ms.engine.run(model, refdrive.b200_hardware(), cfg, reqs, ms.coverage.EmpiricalTable())
    return res, ex


def _worker(rank, world, port, policy, lens, out, q, shape_name="tiny"):
    import sys

    sys.path.insert(0, ROOT)
    try:
        import torch.distributed as dist

        from paper_2510_08055_b200.executor import EPMoEModel, MoEModel
        from paper_2510_08055_b200.types import QWEN3_30B_A3B, TINY

        shape = TINY if shape_name == "tiny" else QWEN3_30B_A3B
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        ep = EPMoEModel(shape, 4, rank, world, max_tokens=4096, device=dev, seed=3)
        res, ex = _engine_run(ep, policy, lens, out, shape_name)
        ref_res, ref_ex = _engine_run(MoEModel(shape, 4, device=dev, seed=3), policy, lens, out, shape_name)
        torch.cuda.synchronize()
        ok, msg = True, ""
        for rid in range(len(lens)):
            same = torch.equal(ex.final_prompt[rid], ref_ex.final_prompt[rid])
            ok &= same
            if not same:
                msg += f"prompt {rid} differs; "
        hits = [it["experts_hit"] for it in ex.iter_log]
        ref_hits = [it["experts_hit"] for it in ref_ex.iter_log]
        if hits != ref_hits:
            ok, msg = False, msg + "experts hit differ; "
        ok &= all(it["moe_s"] > 0 for it in ex.iter_log)
        ok &= [r.prefill_tokens for r in res.records] == [r.prefill_tokens for r in ref_res.records]
        ep.close()  # collective
        dist.destroy_process_group()
        q.put((rank, bool(ok), msg))
    except Exception:  # report instead of hanging the parent
        import traceback

        q.put((rank, False, traceback.format_exc()[-3000:]))


def _run(policy, lens, out=3, world=2, shape_name="tiny"):
    import queue

    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, policy, lens, out, q, shape_name))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in range(world):
            try:
                r, ok, err = q.get(timeout=600)
            except queue.Empty:
                break
            res[r] = (ok, err)
            if not ok:
                break
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for r, (ok, err) in res.items():
        assert ok, f"rank {r}: {err}"
    for r in range(world):
        assert r in res, f"rank {r} reported nothing"


def test_ep_stack_layered_matches_single_gpu(cuda):
    from paper_2510_08055_b200 import refdrive

    if not refdrive.reference_available():
        pytest.skip("the reference (moesim) is not importable: tools/vendor_reference.sh")
    _run("layered", (1024, 700, 301))


def test_ep_stack_chunked_matches_single_gpu(cuda):
    from paper_2510_08055_b200 import refdrive

    if not refdrive.reference_available():
        pytest.skip("the reference (moesim) is not importable: tools/vendor_reference.sh")
    _run("chunked", (900, 77))


def test_ep_stack_qwen_layered_matches_single_gpu(cuda):
    """Qwen3-30B-A3B-shaped 4-layer stack (64 experts per rank): layered prefill of two prompts with
    decodes riding along, EP ≡ single GPU bit for bit."""
    from paper_2510_08055_b200 import refdrive

    if not refdrive.reference_available():
        pytest.skip("the reference (moesim) is not importable: tools/vendor_reference.sh")
    _run("layered", (700, 300), out=2, shape_name="qwen")
