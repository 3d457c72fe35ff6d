"""Expert-parallel exchange logic on CPU: world size 2, gloo, oracle compute injected.

The product EP path (paper_2510_08055_b200.ep.EPMoE) runs the C-ABI kernels
through GpuOps; here the same EPMoE host logic (count exchange, uneven
all_to_all dispatch, local re-permutation, return, combine) runs with the
fp32 oracle as the compute so it can be checked without a GPU: every rank's
output must equal the single-device oracle layer on its own tokens.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import moe_oracle as mo
from paper_2510_08055_b200.types import MoEShape


class OracleOps:
    """CPU stand-in for GpuOps (test-only)."""

    def route(self, x, wr, top_k, renorm):
        ids, w, _ = mo.route(x.float().numpy(), wr.float().numpy(), top_k, renorm)
        return torch.from_numpy(ids), torch.from_numpy(w)

    def permute(self, ids, x, num_experts):
        counts, offsets, slot_of, tok_of = mo.permute(ids.numpy(), num_experts)
        x_perm = x[torch.from_numpy(tok_of).long()] if ids.numel() else x.new_zeros((0, x.shape[1]))
        return (torch.from_numpy(counts), torch.from_numpy(offsets), torch.from_numpy(slot_of),
                torch.from_numpy(tok_of), x_perm)

    def experts(self, x_perm, offsets, w13, w2):
        _, y = mo.experts(x_perm.float().numpy(), offsets.numpy(), w13.float().numpy(), w2.float().numpy())
        return torch.from_numpy(y)

    def combine(self, y_perm, slot_of, w):
        if w.shape[0] == 0:
            return y_perm.new_zeros((0, y_perm.shape[1]))
        return torch.from_numpy(mo.combine(y_perm.float().numpy(), slot_of.numpy(), w.float().numpy()))


SHAPE = MoEShape(hidden=256, ffn=128, num_experts=16, top_k=4, norm_topk_prob=True)


def _weights(seed, skew=False):
    from paper_2510_08055_b200.synthetic import expert_weights, router_weight

    wr = router_weight(SHAPE.num_experts, SHAPE.hidden, seed).float()
    if skew:  # every token prefers experts 0..3 (all owned by rank 0)
        wr[:4, SHAPE.hidden - 1] = 16.0
    w13, w2 = expert_weights(SHAPE.num_experts, SHAPE.hidden, SHAPE.ffn, seed + 1)
    return wr, w13.float(), w2.float()


def _worker(rank, world, port, tokens, skew, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2510_08055_b200.ep import EPMoE
        from paper_2510_08055_b200.synthetic import router_tokens

        wr, w13, w2 = _weights(5, skew)
        layer = EPMoE.from_full(SHAPE, wr, w13, w2, rank, world, ops=OracleOps())
        x = router_tokens(tokens[rank], SHAPE.hidden, 100 + rank).float()
        y, st = layer(x)
        ref = mo.moe_forward(x.numpy(), wr.numpy(), w13.numpy(), w2.numpy(), SHAPE.top_k, True)
        err = mo.rel_l2(y.numpy(), ref["y"]) if tokens[rank] else 0.0
        q.put((rank, err, st.send_splits, st.recv_splits, int(st.counts.sum()), st.recv_rows))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(tokens, skew=False, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, tokens, skew, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=240)
        res[r[0]] = r[1:]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_ep2_matches_single_device_oracle():
    res = _run([37, 50])
    for rank, (err, send, recv, nroute, nrecv) in res.items():
        assert err < 1e-5, (rank, err)
        assert sum(send) == nroute == [37, 50][rank] * SHAPE.top_k
    # what rank 0 sent to rank 1 is what rank 1 received from rank 0, and vice versa
    assert res[0][1][1] == res[1][2][0] and res[1][1][0] == res[0][2][1]
    assert res[0][4] + res[1][4] == (37 + 50) * SHAPE.top_k


def test_ep2_skewed_all_to_rank0_and_empty_rank():
    res = _run([24, 0], skew=True)
    err, send, recv, nroute, nrecv = res[0]
    assert err < 1e-5
    assert send == [24 * SHAPE.top_k, 0]      # experts 0..3 live on rank 0
    assert res[1][4] == 0 and res[1][1] == [0, 0]
