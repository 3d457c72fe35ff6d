"""Small driver for compute-sanitizer (tools/sanitize.sh): one Qwen3-30B-A3B-shaped layer forward per
T given on the command line (decode-size T <= 16 runs the one-launch k_decode), checked against the
fp32 oracle (ids / counts bit-exact, rel-L2 <= 1e-2)."""
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests")]
import torch  # noqa: E402

from paper_2510_08055_b200 import QWEN3_30B_A3B  # noqa: E402
from test_gpu_moe import check_layer  # noqa: E402

dev = torch.device("cuda", 0)
for T in [int(a) for a in sys.argv[1:]] or [1, 64]:
    err, stats, _ = check_layer(QWEN3_30B_A3B, T, 5, dev)
    print(f"T={T} ok rel_l2={err:.3e} experts_hit={stats.experts_hit}", flush=True)
