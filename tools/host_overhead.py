"""Host-side cost of one fused layer call (Python + ctypes + descriptor encoding + launches),
measured without synchronising: if it exceeds the device time, a decode step is host-bound
(capture the layer stack in a CUDA graph then; the layer is graph-capturable).

    python tools/host_overhead.py [T ...]
"""
import os
import sys
import time

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests")]
import torch  # noqa: E402

from paper_2510_08055_b200 import QWEN3_30B_A3B as s  # noqa: E402
from paper_2510_08055_b200.synthetic import router_tokens  # noqa: E402
from test_gpu_moe import make  # noqa: E402

d = torch.device("cuda", 0)
layer = make(s, 3, d)[3]
for T in [int(a) for a in sys.argv[1:]] or [1, 576]:
    x = router_tokens(T, s.hidden, 4).to(d)
    y = torch.empty_like(x)
    for _ in range(20):
        layer(x, out=y)
    torch.cuda.synchronize()
    n = 200
    t0 = time.perf_counter()
    for _ in range(n):
        layer(x, out=y)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"T={T}: host {1e6 * (t1 - t0) / n:.1f} us/call, wall (host+drain) {1e6 * (t2 - t0) / n:.1f} us/call",
          flush=True)
