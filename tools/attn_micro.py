"""Per-layer device time of AttentionDense's pooled decode step (B rows, context ctx) and the kernels
it launches (B200 experiment: which SDPA backend the masked GQA decode takes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2510_08055_b200.executor import AttentionDense  # noqa: E402

dev = torch.device("cuda")
att = AttentionDense(2048, 2, dev, seed=1, pool_slots=33, pool_len=8208)
B = 33
for ctx_pos in (127, 383, 8200):
    spans = [(r, min(ctx_pos, 8207) - (r % 7), 1, 8208) for r in range(B)]
    x = torch.randn((B, 2048), device=dev).to(torch.bfloat16)
    for _ in range(3):
        att.layer(0, x, spans)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        att.layer(0, x, spans)
    e1.record()
    torch.cuda.synchronize()
    print(f"B={B} ctx~{ctx_pos + 1}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per layer (eager, incl. host gaps)")
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        att.layer(0, x, spans)
        torch.cuda.synchronize()
    for ev in prof.key_averages():
        if ev.device_time_total > 0:
            print(f"   {ev.device_time_total:8.1f} us  {ev.key[:110]}")
    sys.stdout.flush()
