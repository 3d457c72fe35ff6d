"""Short driver for ncu: a few Qwen3-MoE layer forwards at T tokens (default 576).

    ncu --set full -k regex:k_experts -s 2 -c 1 -o gpurun_out/prof python tools/prof_layer.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2510_08055_b200 import QWEN3_30B_A3B as s  # noqa: E402
from paper_2510_08055_b200.moe import GpuMoE  # noqa: E402
from paper_2510_08055_b200.synthetic import router_tokens, router_weight  # noqa: E402


def main():
    T = int(os.environ.get("LP_T", "576"))
    iters = int(os.environ.get("LP_ITERS", "6"))
    nl = 2
    dev = torch.device("cuda", 0)
    layers = []
    for i in range(nl):
        g = torch.Generator(device=dev).manual_seed(i)
        w13 = (torch.randn((s.num_experts, 2 * s.ffn, s.hidden), generator=g, device=dev) * 0.02).to(torch.bfloat16)
        w2 = (torch.randn((s.num_experts, s.hidden, s.ffn), generator=g, device=dev) * 0.02).to(torch.bfloat16)
        layers.append(GpuMoE(s, router_weight(s.num_experts, s.hidden, i).to(dev), w13, w2))
    x = router_tokens(T, s.hidden, 7).to(dev)
    for i in range(iters):
        layers[i % nl](x)
    torch.cuda.synchronize()
    print("done", T, iters)


if __name__ == "__main__":
    main()
