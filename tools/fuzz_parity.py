"""Randomised parity sweep of the fused layer against the fp32 oracle (GPU).

Random shapes (the BASELINE / reference configs plus odd ones), batch sizes
1..9000 (both expert kernels, every token-tile regime), optional routing skew.
Each case: ids and counts bit-exact, output rel-L2 <= 1e-2.

    python tools/fuzz_parity.py [cases] [seed]
"""
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_08055_b200 import GPT_OSS_20B, QWEN3_30B_A3B, TINY, MoEShape  # noqa: E402
from paper_2510_08055_b200.synthetic import router_tokens, router_weight  # noqa: E402
from test_gpu_moe import check_layer  # noqa: E402

SHAPES = [QWEN3_30B_A3B, TINY, GPT_OSS_20B, MoEShape(1024, 512, 64, 6, True), MoEShape(512, 256, 256, 8, False),
          MoEShape(768, 384, 8, 2, True)]


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    dev = torch.device("cuda", 0)
    fails = 0
    for i in range(n):
        s = SHAPES[int(rng.integers(len(SHAPES)))]
        T = int(rng.choice([1, 2, 3, 4, 5, 8, 16, 7, 33, 64, 100, 255, 576, 1000, 1553, 2048, 3001, 4100, 5784, 6000, 8224]))
        if s.hidden * s.ffn > 4_000_000 and T > 4100:
            T = 4100  # keep the fp32 oracle quick on the large shapes
        skew = bool(rng.integers(2))
        seed = int(rng.integers(1000))
        wr = None
        if skew:  # a few hot experts (tie-breaker column), the rest cold
            w = router_weight(s.num_experts, s.hidden, seed).float()
            hot = rng.choice(s.num_experts, size=min(s.num_experts, s.top_k + 1), replace=False)
            w[torch.as_tensor(hot), s.hidden - 1] = 8.0
            wr = w.to(torch.bfloat16)
        try:
            err, stats, _ = check_layer(s, T, seed, dev, wr_override=wr)
            print(f"[{i}] ok H={s.hidden} I={s.ffn} E={s.num_experts} k={s.top_k} T={T} skew={skew} "
                  f"hit={stats.experts_hit} rel_l2={err:.2e}", flush=True)
        except AssertionError as e:
            fails += 1
            print(f"[{i}] FAIL H={s.hidden} I={s.ffn} E={s.num_experts} k={s.top_k} T={T} skew={skew}: {e}",
                  flush=True)
    print(f"{n - fails}/{n} passed")
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
