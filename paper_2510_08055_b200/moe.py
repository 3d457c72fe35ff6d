"""`GpuMoE`: the MoE layer forward over a hybrid decode+prefill batch on B200.

This is the numerical layer the reference only cost-models: at the engine's
call sites (moesim/engine.py:144-154) the simulator charges
`moe_cost(model, routed, coverage_model.coverage(routed), layers)`
(costmodel.py:57-85). Here `routed` tokens are actually routed and run:

    y, stats = layer(x)          # x: [T, H] bf16 on cuda
    stats.coverage               # nnz(counts)/E — what CoverageModel estimates
    stats.expert_weight_bytes    # nnz * bytes_per_expert — moe_cost's expert_bytes

Every stage is a call into liblpmoe.so through the C ABI (include/lpmoe.h);
torch only supplies device memory and the current stream. There is no CPU or
eager fallback: non-CUDA inputs raise.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _native
from .types import MoEShape, ValidationError, require


@dataclass
class MoEStats:
    """Routing statistics of one layer call (device tensors until read)."""

    counts: torch.Tensor        # int32 [E] tokens routed to each expert
    shape: MoEShape

    @property
    def experts_hit(self) -> int:
        return int((self.counts > 0).sum().item())

    @property
    def coverage(self) -> float:
        """Fraction of experts activated (the reference's coverage_fraction)."""
        return self.experts_hit / self.shape.num_experts

    @property
    def expert_weight_bytes(self) -> int:
        """Expert-weight HBM bytes one call streams (costmodel.py:77 with measured coverage)."""
        return self.experts_hit * self.shape.bytes_per_expert


def _stream_ptr(device: torch.device) -> int:
    # the raw current-stream handle (torch.cuda.current_stream() builds a Stream object per call:
    # a few us of host time on every decode-size layer call)
    return torch._C._cuda_getCurrentRawStream(device.index if device.index is not None else
                                              torch.cuda.current_device())


def _check_tensor(name: str, t: torch.Tensor, shape: tuple, dtype: torch.dtype) -> None:
    # one cheap combined test on the hot path; the messages are only formatted on failure
    if (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == dtype and t.shape == shape
            and t.is_contiguous()):
        return
    require(isinstance(t, torch.Tensor), f"{name} must be a torch.Tensor")
    require(t.is_cuda, f"{name} must be a CUDA tensor (no CPU path exists), got device {t.device}")
    require(t.dtype == dtype, f"{name} must be {dtype}, got {t.dtype}")
    require(tuple(t.shape) == tuple(shape), f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    require(t.is_contiguous(), f"{name} must be contiguous")


class Workspace:
    """Grow-only device scratch for `lp_moe_*` calls, shareable by every layer that
    runs on one stream (the library's workspace is per-call scratch whose fixed
    header every call leaves zeroed, lpmoe.h). A stack of 48 layers then holds one
    workspace sized for its largest batch instead of 48."""

    def __init__(self, device: torch.device):
        self.device = torch.device(device)
        self.buf: torch.Tensor | None = None

    def get(self, nbytes: int) -> torch.Tensor:
        nbytes = max(int(nbytes), 256)
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = None  # release first: the caching allocator reuses it stream-ordered
            self.buf = torch.zeros(nbytes, dtype=torch.uint8, device=self.device)
        return self.buf


class GpuMoE:
    """One Qwen3-MoE-style sparse MoE block (router + E SwiGLU experts) on sm_100a.

    Weights use the HF layout (transformers 5.5 modeling_qwen3_moe.py:220-224, :255):
    wr [E,H], w13 [E,2I,H] (gate rows then up rows), w2 [E,H,I], all bf16.
    """

    def __init__(self, shape: MoEShape, wr: torch.Tensor, w13: torch.Tensor, w2: torch.Tensor,
                 workspace: Workspace | None = None):
        self.shape = shape
        H, I, E = shape.hidden, shape.ffn, shape.num_experts
        _check_tensor("wr", wr, (E, H), torch.bfloat16)
        _check_tensor("w13", w13, (E, 2 * I, H), torch.bfloat16)
        _check_tensor("w2", w2, (E, H, I), torch.bfloat16)
        self.wr, self.w13, self.w2 = wr, w13, w2
        self.device = wr.device
        self._lib = _native.load()
        self._ws = workspace if workspace is not None else Workspace(self.device)
        self._route_cap = 0
        self._route_bufs: tuple[torch.Tensor, torch.Tensor, torch.Tensor] | None = None
        self._ws_bytes: dict[int, int] = {}   # workspace bytes per T (one ctypes call per new T)
        self._wptrs = (wr.data_ptr(), w13.data_ptr(), w2.data_ptr())

    # ------------------------------------------------------------ workspace
    def workspace_bytes(self, T: int) -> int:
        n = self._ws_bytes.get(T)
        if n is None:
            s = self.shape
            n = int(self._lib.lp_moe_workspace_bytes(T, s.hidden, s.ffn, s.num_experts, s.top_k))
            self._ws_bytes[T] = n
        return n

    def workspace(self, T: int) -> torch.Tensor:
        # zero-filled on (re)allocation: the header holds self-resetting scheduler words (lpmoe.h)
        return self._ws.get(self.workspace_bytes(T))

    def _bufs(self, T: int):
        """ids [T,k], w [T,k], counts [E]: views of grow-only buffers (valid until the next call)."""
        k, E = self.shape.top_k, self.shape.num_experts
        if self._route_bufs is None or T > self._route_cap:
            cap = max(T, 2 * self._route_cap)
            self._route_bufs = (torch.empty((cap, k), dtype=torch.int32, device=self.device),
                                torch.empty((cap, k), dtype=torch.float32, device=self.device),
                                torch.empty((E,), dtype=torch.int32, device=self.device))
            self._route_cap = cap
        ids, w, counts = self._route_bufs
        return ids[:T], w[:T], counts

    # ------------------------------------------------------------ full layer
    def forward(self, x: torch.Tensor, out: torch.Tensor | None = None,
                counts_out: torch.Tensor | None = None) -> tuple[torch.Tensor, MoEStats]:
        """y = MoE(x). x: [T, H] bf16 CUDA. Returns (y, stats); ids/weights in stats buffers.

        counts_out (int32 [E], optional) receives the per-expert counts instead of
        the layer's internal per-T buffer (the executor keeps one row per layer).
        """
        s = self.shape
        require(x.dim() == 2, "x must be 2-D [T, H]")
        T = x.shape[0]
        _check_tensor("x", x, (T, s.hidden), torch.bfloat16)
        y = torch.empty_like(x) if out is None else out
        _check_tensor("out", y, (T, s.hidden), torch.bfloat16)
        ids, w, counts = self._bufs(T)
        if counts_out is not None:
            _check_tensor("counts_out", counts_out, (s.num_experts,), torch.int32)
            counts = counts_out
        ws = self.workspace(T)
        wr, w13, w2 = self._wptrs
        rc = self._lib.lp_moe_forward(
            x.data_ptr(), wr, w13, w2,
            T, s.hidden, s.ffn, s.num_experts, s.top_k, int(s.norm_topk_prob),
            y.data_ptr(), ids.data_ptr(), w.data_ptr(), counts.data_ptr(),
            ws.data_ptr(), ws.numel(), _stream_ptr(self.device))
        if rc:
            _native.check(rc, "lp_moe_forward")
        self.last_ids, self.last_weights = ids, w
        return y, MoEStats(counts, s)

    __call__ = forward

    def forward_host(self, x_host: torch.Tensor, y_host: torch.Tensor | None = None,
                     x_dev: torch.Tensor | None = None) -> tuple[torch.Tensor, MoEStats]:
        """End-to-end call with host buffers: H2D copy, layer, D2H copy (stream ordered)."""
        require(not x_host.is_cuda, "forward_host expects a host tensor")
        xd = x_dev if x_dev is not None else torch.empty(x_host.shape, dtype=x_host.dtype, device=self.device)
        xd.copy_(x_host, non_blocking=True)
        yd, stats = self.forward(xd)
        if y_host is None:
            y_host = torch.empty(yd.shape, dtype=yd.dtype, pin_memory=True)
        y_host.copy_(yd, non_blocking=True)
        return y_host, stats

    # ------------------------------------------------------------ staged API
    def route(self, x: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
        s = self.shape
        T = x.shape[0]
        _check_tensor("x", x, (T, s.hidden), torch.bfloat16)
        ids = torch.empty((T, s.top_k), dtype=torch.int32, device=self.device)
        w = torch.empty((T, s.top_k), dtype=torch.float32, device=self.device)
        ws = self.workspace(T)
        rc = self._lib.lp_moe_route(x.data_ptr(), self.wr.data_ptr(), T, s.hidden, s.num_experts, s.top_k,
                                    int(s.norm_topk_prob), ids.data_ptr(), w.data_ptr(), ws.data_ptr(), ws.numel(),
                                    _stream_ptr(self.device))
        _native.check(rc, "lp_moe_route")
        return ids, w

    def permute(self, ids: torch.Tensor, x: torch.Tensor | None):
        """-> counts [E], offsets [E+1], slot_of [T*k], tok_of [T*k], x_perm [T*k, H] (or None)."""
        s = self.shape
        T = ids.shape[0]
        _check_tensor("ids", ids, (T, s.top_k), torch.int32)
        S = T * s.top_k
        counts = torch.empty((s.num_experts,), dtype=torch.int32, device=self.device)
        offsets = torch.empty((s.num_experts + 1,), dtype=torch.int32, device=self.device)
        slot_of = torch.empty((S,), dtype=torch.int32, device=self.device)
        tok_of = torch.empty((S,), dtype=torch.int32, device=self.device)
        x_perm = None
        if x is not None:
            _check_tensor("x", x, (T, s.hidden), torch.bfloat16)
            x_perm = torch.empty((S, s.hidden), dtype=torch.bfloat16, device=self.device)
        ws = self.workspace(T)
        rc = self._lib.lp_moe_permute(ids.data_ptr(), x.data_ptr() if x is not None else None, T, s.hidden,
                                      s.num_experts, s.top_k, counts.data_ptr(), offsets.data_ptr(),
                                      slot_of.data_ptr(), tok_of.data_ptr(),
                                      x_perm.data_ptr() if x_perm is not None else None,
                                      ws.data_ptr(), ws.numel(), _stream_ptr(self.device))
        _native.check(rc, "lp_moe_permute")
        return counts, offsets, slot_of, tok_of, x_perm

    def experts(self, x_perm: torch.Tensor, offsets: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
        """-> act [S, I], y_perm [S, H] for expert-contiguous rows x_perm [S, H]."""
        s = self.shape
        S = x_perm.shape[0]
        _check_tensor("x_perm", x_perm, (S, s.hidden), torch.bfloat16)
        _check_tensor("offsets", offsets, (s.num_experts + 1,), torch.int32)
        act = torch.empty((S, s.ffn), dtype=torch.bfloat16, device=self.device)
        y_perm = torch.empty((S, s.hidden), dtype=torch.bfloat16, device=self.device)
        ws = self.workspace(max(1, S // s.top_k))
        rc = self._lib.lp_moe_experts(x_perm.data_ptr(), offsets.data_ptr(), S, self.w13.data_ptr(),
                                      self.w2.data_ptr(), s.hidden, s.ffn, s.num_experts, act.data_ptr(),
                                      y_perm.data_ptr(), ws.data_ptr(), ws.numel(), _stream_ptr(self.device))
        _native.check(rc, "lp_moe_experts")
        return act, y_perm

    def combine(self, y_perm: torch.Tensor, slot_of: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
        s = self.shape
        T = w.shape[0]
        _check_tensor("w", w, (T, s.top_k), torch.float32)
        _check_tensor("slot_of", slot_of, (T * s.top_k,), torch.int32)
        require(y_perm.is_cuda and y_perm.dtype == torch.bfloat16 and y_perm.shape[1] == s.hidden,
                "y_perm must be a CUDA bf16 [S, H] tensor")
        y = torch.empty((T, s.hidden), dtype=torch.bfloat16, device=self.device)
        rc = self._lib.lp_moe_combine(y_perm.data_ptr(), slot_of.data_ptr(), w.data_ptr(), T, s.hidden, s.top_k,
                                      y.data_ptr(), _stream_ptr(self.device))
        _native.check(rc, "lp_moe_combine")
        return y


class HostPipeline:
    """End-to-end forwards from pinned host buffers with the copies overlapped.

    Step i's H2D copy runs on an upload stream and step i's D2H copy on a
    download stream, so while layer i computes, the input of step i+1 is
    uploading and the output of step i-1 is downloading (PCIe is full duplex).
    `depth` device staging buffers per direction; every hazard is an event:
    an upload waits until the compute that last read its staging buffer is
    done, a compute waits for its upload and for the download that last read
    its output buffer. Results land in the caller's host tensors in order.
    """

    def __init__(self, device: torch.device, T: int, H: int, depth: int = 2):
        self.device, self.depth = device, depth
        self.up = torch.cuda.Stream(device)
        self.down = torch.cuda.Stream(device)
        self.xd = [torch.empty((T, H), dtype=torch.bfloat16, device=device) for _ in range(depth)]
        self.yd = [torch.empty((T, H), dtype=torch.bfloat16, device=device) for _ in range(depth)]
        self.ev_up = [torch.cuda.Event() for _ in range(depth)]
        self.ev_comp = [torch.cuda.Event() for _ in range(depth)]
        self.ev_down = [torch.cuda.Event() for _ in range(depth)]
        self.i = 0

    def start(self, event: torch.cuda.Event) -> None:
        """Order the first copies after `event` (the start of a timed region)."""
        self.up.wait_event(event)
        self.down.wait_event(event)

    def submit(self, layer: "GpuMoE", x_host: torch.Tensor, y_host: torch.Tensor) -> MoEStats:
        require(not x_host.is_cuda and not y_host.is_cuda, "HostPipeline.submit expects host tensors")
        b = self.i % self.depth
        self.i += 1
        comp = torch.cuda.current_stream(self.device)
        self.up.wait_event(self.ev_comp[b])          # staging buffer b no longer read by compute
        with torch.cuda.stream(self.up):
            self.xd[b].copy_(x_host, non_blocking=True)
            self.ev_up[b].record(self.up)
        comp.wait_event(self.ev_up[b])
        comp.wait_event(self.ev_down[b])              # output buffer b downloaded
        _, stats = layer.forward(self.xd[b], out=self.yd[b])
        self.ev_comp[b].record(comp)
        self.down.wait_event(self.ev_comp[b])
        with torch.cuda.stream(self.down):
            y_host.copy_(self.yd[b], non_blocking=True)
            self.ev_down[b].record(self.down)
        return stats

    def drain(self) -> None:
        """Make the current stream wait for every submitted download."""
        comp = torch.cuda.current_stream(self.device)
        for e in self.ev_down:
            comp.wait_event(e)


class GraphedHostStep:
    """End-to-end calls from pinned host buffers as ONE CUDA graph per call: the H2D copy of the
    caller's input, the layer, the D2H copy into the caller's output — for decode-size batches, where
    the copies are a few KiB and the host cost of an event-ordered submit (HostPipeline: ~25 us of
    stream / event / ctypes calls) is comparable to the layer itself. A graph is captured on first use
    per (layer, x_host, y_host) buffer triple and replayed on the current stream afterwards; the
    captured addresses stay valid while those buffers live and the layer's workspace is not regrown
    (a call with a larger T than any before it)."""

    def __init__(self, device: torch.device, T: int, H: int):
        self.device = device
        self.xd = torch.empty((T, H), dtype=torch.bfloat16, device=device)
        self.yd = torch.empty((T, H), dtype=torch.bfloat16, device=device)
        self.pool = torch.cuda.graph_pool_handle()
        # key -> (graph, layer, x_host, y_host): the references keep every captured address alive
        self.graphs: dict[tuple, tuple] = {}

    def _body(self, layer: "GpuMoE", x_host: torch.Tensor, y_host: torch.Tensor) -> None:
        self.xd.copy_(x_host, non_blocking=True)
        layer.forward(self.xd, out=self.yd)
        y_host.copy_(self.yd, non_blocking=True)

    def prepare(self, layer: "GpuMoE", x_host: torch.Tensor, y_host: torch.Tensor) -> None:
        """Capture the graph of this buffer triple now (outside any timed region)."""
        require(not x_host.is_cuda and not y_host.is_cuda and x_host.is_pinned() and y_host.is_pinned(),
                "GraphedHostStep expects pinned host tensors")
        require(tuple(x_host.shape) == tuple(self.xd.shape) and tuple(y_host.shape) == tuple(self.yd.shape),
                "GraphedHostStep: shape differs from the captured one")
        key = (id(layer), x_host.data_ptr(), y_host.data_ptr())
        if key in self.graphs:
            return
        cur = torch.cuda.current_stream(self.device)
        side = torch.cuda.Stream(self.device)
        side.wait_stream(cur)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(side):
            self._body(layer, x_host, y_host)  # warm-up off the capture: workspace, kernel attributes
            g.capture_begin(pool=self.pool)
            self._body(layer, x_host, y_host)
            g.capture_end()
        cur.wait_stream(side)
        self.graphs[key] = (g, layer, x_host, y_host)

    def submit(self, layer: "GpuMoE", x_host: torch.Tensor, y_host: torch.Tensor) -> None:
        key = (id(layer), x_host.data_ptr(), y_host.data_ptr())
        if key not in self.graphs:
            self.prepare(layer, x_host, y_host)
        self.graphs[key][0].replay()


def layer_from_seed(shape: MoEShape, seed: int, device: str = "cuda", tie_break: bool = True) -> GpuMoE:
    """Random-init layer on the dyadic router grid (see synthetic.py)."""
    from .synthetic import expert_weights, router_weight

    wr = router_weight(shape.num_experts, shape.hidden, seed, tie_break=tie_break)
    w13, w2 = expert_weights(shape.num_experts, shape.hidden, shape.ffn, seed + 1)
    return GpuMoE(shape, wr.to(device), w13.to(device), w2.to(device))


def add_rmsnorm(h: torch.Tensor, delta: torch.Tensor | None, xn: torch.Tensor, eps: float = 1e-6) -> None:
    """h += delta (if given); xn = RMSNorm(h) with unit gain (lp_add_rmsnorm, executor glue)."""
    require(h.is_cuda and h.dtype == torch.bfloat16 and h.dim() == 2 and h.is_contiguous(),
            "h must be a contiguous CUDA bf16 [T, H] tensor")
    _check_tensor("xn", xn, tuple(h.shape), torch.bfloat16)
    if delta is not None:
        _check_tensor("delta", delta, tuple(h.shape), torch.bfloat16)
    rc = _native.load().lp_add_rmsnorm(h.data_ptr(), delta.data_ptr() if delta is not None else None,
                                       xn.data_ptr(), h.shape[0], h.shape[1], eps, _stream_ptr(h.device))
    _native.check(rc, "lp_add_rmsnorm")
