"""Debug driver: the c3 serving run with a device sync + sanity check after every layer call.

On the first failure it prints the layer, T, and input statistics, and saves the
failing input to gpurun_out/fail_x.pt.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2510_08055_b200 import moe as moe_mod  # noqa: E402

_orig = moe_mod.GpuMoE.forward
_n = [0]


def checked(self, x, out=None):
    torch.cuda.synchronize()
    xf = x.float()
    info = dict(call=_n[0], T=x.shape[0], nan=int(torch.isnan(xf).sum()), inf=int(torch.isinf(xf).sum()),
                absmax=float(xf.abs().max()) if x.numel() else 0.0)
    _n[0] += 1
    try:
        y, st = _orig(self, x, out)
        torch.cuda.synchronize()
        ids = self.last_ids
        if ids.numel() and (int(ids.min()) < 0 or int(ids.max()) >= self.shape.num_experts):
            raise RuntimeError(f"ids out of range {int(ids.min())}..{int(ids.max())}")
        if int(st.counts.sum()) != x.shape[0] * self.shape.top_k:
            raise RuntimeError(f"counts sum {int(st.counts.sum())} != {x.shape[0] * self.shape.top_k}")
    except Exception as exc:  # noqa: BLE001
        print("FAIL", info, repr(exc), flush=True)
        os.makedirs("gpurun_out", exist_ok=True)
        try:
            torch.save(x.cpu(), "gpurun_out/fail_x.pt")
        except Exception:  # noqa: BLE001
            pass
        raise
    if _n[0] % 500 == 0:
        print("ok", info, flush=True)
    return y, st


moe_mod.GpuMoE.forward = checked
moe_mod.GpuMoE.__call__ = checked

sys.argv = [sys.argv[0]] + sys.argv[1:]
import runpy  # noqa: E402

runpy.run_path(os.path.join(ROOT, "tools", "serving_bench.py"), run_name="__main__")
