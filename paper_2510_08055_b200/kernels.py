"""GPU routing-surrogate sampler with the reference's kernel API.

Drop-in for moesim.kernels.uniform_union_counts / weighted_union_counts
(kernels.py:209-222): same arguments (pre-drawn float64 uniforms
u[trials, batch, k]), same int64 [trials] result, bit-identical values —
computed by liblpmoe.so (union_counts.cuh). Inputs may be numpy arrays (copied
to the GPU and back) or CUDA float64 tensors (result stays on the device).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native
from .types import require


def _as_device(a, dtype=torch.float64) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        require(a.is_cuda, "tensor inputs must live on a CUDA device")
        return a.to(dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to("cuda", non_blocking=False)


def _check(u, batch: int, k: int, num_experts: int):
    require(batch >= 0, f"batch must be >= 0, got {batch}")
    require(1 <= k <= num_experts,
            f"top_k out of range: need 1 <= top_k <= num_experts, got top_k={k}, num_experts={num_experts}")
    shp = tuple(u.shape)
    require(len(shp) == 3 and shp[1] == batch and shp[2] == k, f"u must have shape (trials, {batch}, {k}), got {shp}")


def uniform_union_counts(u, batch: int, k: int, num_experts: int):
    """Per-trial union sizes for `batch` uniform top-k draws; u: (trials, batch, k)."""
    _check(u, batch, k, num_experts)
    host = not isinstance(u, torch.Tensor)
    trials = u.shape[0]
    ud = _as_device(u)
    out = torch.zeros(trials, dtype=torch.int64, device=ud.device)
    if trials and batch:
        rc = _native.load().lp_union_counts_uniform(ud.data_ptr(), trials, batch, k, num_experts, out.data_ptr(),
                                                    torch.cuda.current_stream(ud.device).cuda_stream)
        _native.check(rc, "lp_union_counts_uniform")
    return out.cpu().numpy() if host else out


def weighted_union_counts(u, batch: int, k: int, num_experts: int, weights):
    """Per-trial union sizes for rank-weighted top-k draws without replacement."""
    _check(u, batch, k, num_experts)
    host = not isinstance(u, torch.Tensor)
    trials = u.shape[0]
    ud = _as_device(u)
    wd = _as_device(weights)
    require(tuple(wd.shape) == (num_experts,), f"weights must have shape ({num_experts},), got {tuple(wd.shape)}")
    out = torch.zeros(trials, dtype=torch.int64, device=ud.device)
    if trials and batch:
        rc = _native.load().lp_union_counts_weighted(ud.data_ptr(), trials, batch, k, num_experts, wd.data_ptr(),
                                                     out.data_ptr(), torch.cuda.current_stream(ud.device).cuda_stream)
        _native.check(rc, "lp_union_counts_weighted")
    return out.cpu().numpy() if host else out
