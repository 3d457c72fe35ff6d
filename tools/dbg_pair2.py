import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2510_08055_b200 import QWEN3_30B_A3B as s
from paper_2510_08055_b200.moe import GpuMoE
from paper_2510_08055_b200.synthetic import router_tokens, router_weight
dev = torch.device("cuda", 0)
T = int(sys.argv[1]); NL = 8; NI = int(sys.argv[2])
layers = []
for i in range(NL):
    g = torch.Generator(device=dev).manual_seed(1000 + i)
    wr = router_weight(s.num_experts, s.hidden, 1000 + i).to(dev)
    w13 = (torch.randn((s.num_experts, 2 * s.ffn, s.hidden), generator=g, device=dev) * 0.02).to(torch.bfloat16)
    w2 = (torch.randn((s.num_experts, s.hidden, s.ffn), generator=g, device=dev) * 0.02).to(torch.bfloat16)
    layers.append(GpuMoE(s, wr, w13, w2))
xs = [router_tokens(T, s.hidden, 50 + i).to(dev) for i in range(NI)]
nsteps = int(sys.argv[3]); every = int(sys.argv[4])
for i in range(nsteps):
    y, st = layers[i % NL](xs[i % NI])
    if (i + 1) % every == 0:
        torch.cuda.synchronize()
        print(i, flush=True)
torch.cuda.synchronize()
print("done")
