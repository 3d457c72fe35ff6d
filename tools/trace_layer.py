"""Phase timeline of one MoE-layer forward from the -DLP_TRACE build.

    python -m paper_2510_08055_b200.build --trace
    LP_T=576 python tools/trace_layer.py
Prints %globaltimer deltas (ns) relative to the router's first CTA start.
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["LPMOE_LIB"] = os.path.join(ROOT, "paper_2510_08055_b200", "_lib", "liblpmoe_trace.so")
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2510_08055_b200 import QWEN3_30B_A3B as s  # noqa: E402
from paper_2510_08055_b200 import _native  # noqa: E402
from paper_2510_08055_b200.moe import GpuMoE  # noqa: E402
from paper_2510_08055_b200.synthetic import router_tokens, router_weight  # noqa: E402

NAMES = {0: "router blk0 start", 1: "router blk0 setup done", 2: "router blk0 first TMA issued",
         3: "router blk0 all TMA issued", 4: "router blk0 MMA done", 5: "router blk0 top-k done",
         6: "router blk0 end", 8: "router first CTA start", 9: "router last CTA end",
         16: "scan start", 17: "scan staged", 18: "scan end (staged)",
         24: "scatter first", 25: "scatter last", 10: "router blk0 post-mma sync", 11: "router blk0 cluster sync1",
         12: "router blk0 cluster sync2", 13: "router blk0 top-k done(2)", 14: "router blk0 hist done",
         15: "router blk0 grid barrier passed", 32: "experts first CTA start", 33: "experts blk0 start",
         34: "experts last CTA end", 35: "experts blk0 end", 40: "combine first", 41: "combine last",
         48: "decode first CTA start", 54: "decode blk0 pdl_wait done", 49: "decode blk0 routing MMA drained",
         50: "decode blk0 logits folded", 51: "decode blk0 top-k + permutation done", 52: "decode first item claimed",
         53: "decode last CTA end", 55: "decode blk0 top-k done", 56: "decode blk0 perm zeroed",
         57: "decode blk0 cluster arrive done"}


def tiny_items(lib, t0, layer):
    """Per-CTA work-item timeline of k_experts_tiny (us from the router start):
    id claimed | dependency met | last TMA issued | epilogue done | first MMA | last MMA | acc to epilogue |
    k-block n-2 ready | k-block n-1 ready."""
    C, N, F = 160, 8, 10
    buf = (ctypes.c_ulonglong * (C * N * F))()
    lib.lp_trace_items.argtypes = [ctypes.c_void_p, ctypes.c_int]
    lib.lp_trace_items(buf, C * N * F)
    hit = int(torch.unique(layer.last_ids).numel())
    n_up = 12 * hit if hit else None
    rows, ups, dns = [], [], []
    for c in range(C):
        items = []
        for n in range(N):
            f = [buf[(c * N + n) * F + i] for i in range(F)]
            if f[1] == 0:
                continue
            us = [(v - t0) / 1000 if v else float("nan") for v in f[1:]]
            kind = "?" if n_up is None else ("U" if f[0] < n_up else ("D" if f[0] < n_up + 16 * hit else "end"))
            items.append(f"{kind}{f[0]}:" + "/".join(f"{u:.1f}" for u in us))
            if kind == "U":
                ups.append(us)
            elif kind == "D":
                dns.append(us)
        if items:
            rows.append(f"cta{c}: " + " ".join(items))
    print("\n".join(rows))
    if ups:
        print(f"UP items {len(ups)}: claimed {min(u[0] for u in ups):.1f}-{max(u[0] for u in ups):.1f}, "
              f"done {min(u[3] for u in ups):.1f}-{max(u[3] for u in ups):.1f} us")
    if dns:
        print(f"DN items {len(dns)}: claimed {min(u[0] for u in dns):.1f}-{max(u[0] for u in dns):.1f}, "
              f"dep met {min(u[1] for u in dns):.1f}-{max(u[1] for u in dns):.1f}, "
              f"done {min(u[3] for u in dns):.1f}-{max(u[3] for u in dns):.1f} us")


def main():
    T = int(os.environ.get("LP_T", "576"))
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    w13 = (torch.randn((s.num_experts, 2 * s.ffn, s.hidden), generator=g, device=dev) * 0.02).to(torch.bfloat16)
    w2 = (torch.randn((s.num_experts, s.hidden, s.ffn), generator=g, device=dev) * 0.02).to(torch.bfloat16)
    layer = GpuMoE(s, router_weight(s.num_experts, s.hidden, 0).to(dev), w13, w2)
    x = router_tokens(T, s.hidden, 7).to(dev)
    lib = _native.load()
    lib.lp_trace_fetch.argtypes = [ctypes.c_void_p, ctypes.c_int]
    for _ in range(5):
        layer(x)
    torch.cuda.synchronize()
    for rep in range(3):
        lib.lp_trace_reset()
        torch.cuda.synchronize()
        layer(x)
        torch.cuda.synchronize()
        buf = (ctypes.c_ulonglong * 512)()
        lib.lp_trace_fetch(buf, 512)
        t0 = buf[8] if buf[8] not in (0, 2**64 - 1) else buf[48]
        print(f"--- T={T} rep {rep}")
        for k in sorted(NAMES):
            v = buf[k]
            if v in (0, 2**64 - 1):
                continue
            print(f"{NAMES[k]:32s} {(v - t0) / 1000:9.2f} us")
        if os.environ.get("LP_TINY_ITEMS"):
            tiny_items(lib, t0, layer)
        if os.environ.get("LP_ITEMS"):
            for cta in range(4):
                ts = [buf[64 + cta * 32 + i] for i in range(30)]
                its = [buf[192 + cta * 32 + i] for i in range(30)]
                row = [f"{its[i]}@{(ts[i] - t0) / 1000:.1f}" for i in range(30) if ts[i] not in (0, 2**64 - 1)]
                print(f"cta{cta}:", " ".join(row))


if __name__ == "__main__":
    main()

