"""Token-level sharding of the expert-parallel layer stack (executor.EPMoEModel) on the CPU: gloo,
world sizes 2 and 3, uneven shares (T not a multiple of the world size, T < world size).

Every rank owns rows [T*r/P, T*(r+1)/P) of a segment; after its layers it all-gathers the shares
back so every rank holds the full hidden state again (executor.gather_rows, the same code the GPU
stack runs over NCCL / host-staged gloo)."""

import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_08055_b200.executor import gather_rows, shard_rows


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        ok = True
        for T in (0, 1, 2, 3, 5, 16, 97, 576):
            H = 8
            x = torch.full((T, H), -1.0)  # the other ranks' rows are stale before the gather
            lo, hi = shard_rows(T, rank, world)
            x[lo:hi] = torch.arange(lo, hi, dtype=torch.float32)[:, None] + 1000 * rank
            gather_rows(x, x[lo:hi], rank, world, via_host=True)
            want = torch.empty((T, H))
            for r in range(world):
                a, b = shard_rows(T, r, world)
                want[a:b] = torch.arange(a, b, dtype=torch.float32)[:, None] + 1000 * r
            ok &= bool(torch.equal(x, want))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def _run(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    assert all(res[r] for r in range(world)), res


def test_shards_cover_every_row_once():
    for world in (1, 2, 3, 8):
        for T in (0, 1, 7, 8, 576, 8224):
            spans = [shard_rows(T, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == T
            assert all(spans[r][1] == spans[r + 1][0] for r in range(world - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


def test_gather_rows_world2():
    _run(2)


def test_gather_rows_world3_uneven():
    _run(3)
