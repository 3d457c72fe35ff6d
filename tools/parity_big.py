import os, sys
sys.path[:0] = [os.getcwd(), os.path.join(os.getcwd(), "tests")]
import torch
from paper_2510_08055_b200 import QWEN3_30B_A3B, MoEShape
from test_gpu_moe import check_layer
d = torch.device("cuda", 0)
for s, T in ((QWEN3_30B_A3B, 12000), (QWEN3_30B_A3B, 20000), (QWEN3_30B_A3B, 33534), (MoEShape(512, 256, 256, 8, False), 20000)):
    err, st, _ = check_layer(s, T, 5, d)
    print(f"H={s.hidden} E={s.num_experts} T={T} ok rel_l2={err:.2e} hit={st.experts_hit}", flush=True)
