"""EP path on one B200 (NCCL, world size 1): GpuOps stages + all_to_all plumbing must
reproduce the fused single-GPU layer bit for bit (same kernels, same slot order)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist

from paper_2510_08055_b200 import QWEN3_30B_A3B
from paper_2510_08055_b200.synthetic import expert_weights, router_tokens, router_weight

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pg(cuda):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    yield
    dist.destroy_process_group()


def test_ep_world1_equals_fused(cuda, pg):
    from paper_2510_08055_b200.ep import EPMoE
    from paper_2510_08055_b200.moe import GpuMoE

    s = QWEN3_30B_A3B
    wr = router_weight(s.num_experts, s.hidden, 3).to(cuda)
    w13, w2 = expert_weights(s.num_experts, s.hidden, s.ffn, 4)
    w13, w2 = w13.to(cuda), w2.to(cuda)
    x = router_tokens(300, s.hidden, 6).to(cuda)
    y_ref, st_ref = GpuMoE(s, wr, w13, w2)(x)
    ep = EPMoE.from_full(s, wr, w13, w2, 0, 1)
    y, st = ep(x)
    torch.cuda.synchronize()
    assert torch.equal(y, y_ref)
    assert torch.equal(st.counts, st_ref.counts)
    assert st.recv_rows == 300 * s.top_k and st.send_splits == [300 * s.top_k]
