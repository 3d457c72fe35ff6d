"""Quick parity check of the Qwen layer at given T values (env knobs select the path).

    LPMOE_PAIR=1 python tools/parity_quick.py 4100 8224
"""
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests")]
import torch  # noqa: E402

from paper_2510_08055_b200 import QWEN3_30B_A3B  # noqa: E402
from test_gpu_moe import check_layer  # noqa: E402

d = torch.device("cuda", 0)
for T in (int(a) for a in sys.argv[1:]):
    err, stats, _ = check_layer(QWEN3_30B_A3B, T, 5, d)
    print(f"T={T} ok rel_l2={err:.3e} hit={stats.experts_hit}", flush=True)
