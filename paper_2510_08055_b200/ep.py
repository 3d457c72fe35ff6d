"""Expert-parallel MoE layer: experts sharded over ranks,
tokens data-parallel, one exchange step each way over NCCL.

Rank r owns experts [r*E/P, (r+1)*E/P); the router weight is replicated.
Per layer call on each rank (T_local tokens):

  1. route + permute locally over the GLOBAL expert set       (K1, K2)
     -> x_perm is expert-contiguous, hence destination-rank-contiguous
  2. all_to_all_single of the per-(dest rank, local expert) counts
  3. all_to_all_single of x_perm rows (uneven splits)          dispatch
  4. permute the received rows by local expert (K2, topk=1) and run the
     local expert FFN (K3) on the owned weights
  5. un-permute to receive order (K4 with weight 1: exact copy) and
     all_to_all_single the rows back                           return
  6. weighted combine with the local routing weights           (K4)

The reference has no multi-GPU code; this is the B200-native EP
the north star asks for. All compute is liblpmoe.so through `GpuOps`; the
exchange logic is written against a small ops protocol so it is tested with
world-size-2 gloo on CPU (tests/test_ep.py injects CPU ops there).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _native
from .moe import MoEStats, _check_tensor, _stream_ptr
from .types import MoEShape, require


class GpuOps:
    """The four C-ABI stages with explicit (E, k) so they serve both the global
    routing (E experts, top-k) and the local re-permutation (E/P experts, k=1)."""

    def __init__(self, device: torch.device):
        self.device = device
        self.lib = _native.load()
        self._ws: torch.Tensor | None = None

    def _workspace(self, T: int, H: int, I: int, E: int, k: int) -> torch.Tensor:
        need = max(int(self.lib.lp_moe_workspace_bytes(max(T, 1), H, I, E, k)), 256)
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.zeros(need, dtype=torch.uint8, device=self.device)
        return self._ws

    def route(self, x, wr, top_k: int, renorm: bool):
        T, H = x.shape
        E = wr.shape[0]
        ids = torch.empty((T, top_k), dtype=torch.int32, device=self.device)
        w = torch.empty((T, top_k), dtype=torch.float32, device=self.device)
        if T:
            ws = self._workspace(T, H, 128, E, top_k)
            _native.check(self.lib.lp_moe_route(x.data_ptr(), wr.data_ptr(), T, H, E, top_k, int(renorm),
                                                ids.data_ptr(), w.data_ptr(), ws.data_ptr(), ws.numel(),
                                                _stream_ptr(self.device)), "lp_moe_route")
        return ids, w

    def permute(self, ids, x, num_experts: int):
        T, k = ids.shape
        H = x.shape[1]
        S = T * k
        counts = torch.zeros((num_experts,), dtype=torch.int32, device=self.device)
        offsets = torch.zeros((num_experts + 1,), dtype=torch.int32, device=self.device)
        slot_of = torch.empty((S,), dtype=torch.int32, device=self.device)
        tok_of = torch.empty((S,), dtype=torch.int32, device=self.device)
        x_perm = torch.empty((S, H), dtype=x.dtype, device=self.device)
        if T:
            ws = self._workspace(T, H, 128, num_experts, k)
            _native.check(self.lib.lp_moe_permute(ids.data_ptr(), x.data_ptr(), T, H, num_experts, k,
                                                  counts.data_ptr(), offsets.data_ptr(), slot_of.data_ptr(),
                                                  tok_of.data_ptr(), x_perm.data_ptr(), ws.data_ptr(), ws.numel(),
                                                  _stream_ptr(self.device)), "lp_moe_permute")
        return counts, offsets, slot_of, tok_of, x_perm

    def experts(self, x_perm, offsets, w13, w2):
        S, H = x_perm.shape
        E, I2, _ = w13.shape
        y_perm = torch.empty((S, H), dtype=x_perm.dtype, device=self.device)
        if S:
            act = torch.empty((S, I2 // 2), dtype=x_perm.dtype, device=self.device)
            ws = self._workspace(S, H, I2 // 2, E, 1)
            _native.check(self.lib.lp_moe_experts(x_perm.data_ptr(), offsets.data_ptr(), S, w13.data_ptr(),
                                                  w2.data_ptr(), H, I2 // 2, E, act.data_ptr(), y_perm.data_ptr(),
                                                  ws.data_ptr(), ws.numel(), _stream_ptr(self.device)),
                          "lp_moe_experts")
        return y_perm

    def combine(self, y_perm, slot_of, w):
        T, k = w.shape
        H = y_perm.shape[1]
        y = torch.empty((T, H), dtype=y_perm.dtype, device=self.device)
        if T:
            _native.check(self.lib.lp_moe_combine(y_perm.data_ptr(), slot_of.data_ptr(), w.data_ptr(), T, H, k,
                                                  y.data_ptr(), _stream_ptr(self.device)), "lp_moe_combine")
        return y


@dataclass
class EPStats:
    counts: torch.Tensor       # int32 [E] global-expert counts of this rank's tokens
    recv_rows: "int | torch.Tensor"    # rows this rank's experts processed (PeerEP: a device scalar, no sync)
    send_splits: "list[int] | None"      # EPMoE: rows sent per rank; PeerEP: None (counts.view(P, El).sum(1))
    recv_splits: list[int]
    shape: MoEShape

    @property
    def local(self) -> MoEStats:
        return MoEStats(self.counts, self.shape)


class EPMoE:
    """One MoE layer, experts sharded over the ranks of `group`."""

    def __init__(self, shape: MoEShape, wr: torch.Tensor, w13_local: torch.Tensor, w2_local: torch.Tensor,
                 rank: int, world: int, group=None, ops=None):
        E = shape.num_experts
        require(E % world == 0, f"num_experts={E} must be divisible by the EP world size {world}")
        self.shape, self.rank, self.world, self.group = shape, rank, world, group
        self.e_local = E // world
        self.e0 = rank * self.e_local
        H, I = shape.hidden, shape.ffn
        require(tuple(wr.shape) == (E, H), f"wr must have shape {(E, H)}, got {tuple(wr.shape)}")
        require(tuple(w13_local.shape) == (self.e_local, 2 * I, H),
                f"w13_local must have shape {(self.e_local, 2 * I, H)}, got {tuple(w13_local.shape)}")
        require(tuple(w2_local.shape) == (self.e_local, H, I),
                f"w2_local must have shape {(self.e_local, H, I)}, got {tuple(w2_local.shape)}")
        self.wr, self.w13, self.w2 = wr, w13_local, w2_local
        self.device = wr.device
        if ops is None:
            for name, t in (("wr", wr), ("w13_local", w13_local), ("w2_local", w2_local)):
                _check_tensor(name, t, tuple(t.shape), torch.bfloat16)
            ops = GpuOps(self.device)
        self.ops = ops
        self._ones: dict[int, torch.Tensor] = {}

    @classmethod
    def from_full(cls, shape: MoEShape, wr, w13, w2, rank: int, world: int, group=None, ops=None) -> "EPMoE":
        el = shape.num_experts // world
        sl = slice(rank * el, (rank + 1) * el)
        return cls(shape, wr, w13[sl].contiguous(), w2[sl].contiguous(), rank, world, group, ops)

    def _ones_w(self, n: int) -> torch.Tensor:
        t = self._ones.get(n)
        if t is None:
            t = torch.ones((n, 1), dtype=torch.float32, device=self.device)
            self._ones[n] = t
        return t

    def forward(self, x: torch.Tensor, out: torch.Tensor | None = None) -> tuple[torch.Tensor, EPStats]:
        s, P, el = self.shape, self.world, self.e_local
        require(x.dim() == 2 and x.shape[1] == s.hidden, f"x must be [T, {s.hidden}], got {tuple(x.shape)}")
        ids, w = self.ops.route(x, self.wr, s.top_k, s.norm_topk_prob)
        counts, offsets, slot_of, tok_of, x_perm = self.ops.permute(ids, x, s.num_experts)
        # (2) counts per (destination rank, its local expert)
        send_counts = counts.view(P, el).contiguous()
        recv_counts = torch.empty_like(send_counts)
        dist.all_to_all_single(recv_counts, send_counts, group=self.group)
        both = torch.stack([send_counts.sum(1), recv_counts.sum(1)]).cpu()  # one host sync per layer
        send_splits, recv_splits = both[0].tolist(), both[1].tolist()
        R = int(sum(recv_splits))
        # (3) dispatch: x_perm is destination-contiguous because slots are expert-contiguous
        x_recv = torch.empty((R, s.hidden), dtype=x.dtype, device=self.device)
        dist.all_to_all_single(x_recv, x_perm, recv_splits, send_splits, group=self.group)
        # (4) group received rows by local expert (stable: source rank, then source order) and run them
        local_ids = torch.repeat_interleave(
            torch.arange(el, device=self.device, dtype=torch.int32).repeat(P),
            recv_counts.reshape(-1).to(torch.int64), output_size=R).view(R, 1)
        _, off_l, slot_l, _, x_loc = self.ops.permute(local_ids, x_recv, el)
        y_loc = self.ops.experts(x_loc, off_l, self.w13, self.w2)
        # (5) back to receive order (weight 1.0: exact) and return to the source ranks
        y_recv = self.ops.combine(y_loc, slot_l, self._ones_w(R))
        y_back = torch.empty((x_perm.shape[0], s.hidden), dtype=x.dtype, device=self.device)
        dist.all_to_all_single(y_back, y_recv, send_splits, recv_splits, group=self.group)
        # (6) weighted combine of this rank's tokens
        y = self.ops.combine(y_back, slot_of, w)
        if out is not None:
            out.copy_(y)
            y = out
        self.last_ids, self.last_weights = ids, w
        return y, EPStats(counts, R, send_splits, recv_splits, s)

    __call__ = forward

    def forward_host(self, x_host: torch.Tensor, y_host: torch.Tensor | None = None,
                     x_dev: torch.Tensor | None = None):
        """End-to-end call with host buffers: H2D copy, EP layer, D2H copy."""
        xd = x_dev if x_dev is not None else torch.empty(x_host.shape, dtype=x_host.dtype, device=self.device)
        xd.copy_(x_host, non_blocking=True)
        yd, stats = self.forward(xd)
        if y_host is None:
            y_host = torch.empty(yd.shape, dtype=yd.dtype, pin_memory=True)
        y_host.copy_(yd, non_blocking=True)
        return y_host, stats


class PeerRegion:
    """One rank's symmetric EP buffers, exported over CUDA IPC and mapped by every rank.

    Layout (256-byte aligned): [control block: barrier counter, barrier / layer
    sequence numbers, ready tags, double-buffered count inbox [2][P][E] int32
    (lp_ep_ctl_bytes) | recv_x [cap, H] bf16 | y_out [cap, H] bf16], allocated
    with plain cudaMalloc (lp_ipc_alloc, zero-filled). `peer_*` are device arrays
    of the P ranks' addresses of each part. The layers of one stack run in
    sequence and share one region; its sequence numbers live on the device, so
    layers are CUDA-graph capturable. `group` is used to swap handles and to
    fence `close()`.
    """

    def __init__(self, device: torch.device, rank: int, world: int, cap: int, hidden: int, el: int, group=None):
        self.device, self.rank, self.world, self.cap, self.hidden, self.el = device, rank, world, cap, hidden, el
        self.group = group
        self.lib = _native.load()
        align = lambda n: (n + 255) // 256 * 256  # noqa: E731
        ctl = int(self.lib.lp_ep_ctl_bytes(world, world * el))
        require(ctl > 0, f"PeerRegion: unsupported EP world size {world} (max 32) for {world * el} experts")
        off_recv = align(ctl)
        off_y = align(off_recv + 2 * cap * hidden)
        total = align(off_y + 2 * cap * hidden)
        base = ctypes.c_void_p(0)
        _native.check(self.lib.lp_ipc_alloc(total, ctypes.byref(base)), "lp_ipc_alloc")
        self.base = int(base.value)
        handle = ctypes.create_string_buffer(64)
        off = ctypes.c_size_t(0)
        _native.check(self.lib.lp_ipc_handle(self.base, handle, ctypes.byref(off)), "lp_ipc_handle")
        allh: list = [None] * world
        dist.all_gather_object(allh, (bytes(handle.raw), int(off.value)), group=group)
        self._opened: list[int] = []
        bases = []
        for q, (h, o) in enumerate(allh):
            if q == rank:
                bases.append(self.base)
                continue
            p = ctypes.c_void_p(0)
            _native.check(self.lib.lp_ipc_open(ctypes.create_string_buffer(h, 64), ctypes.byref(p)), "lp_ipc_open")
            self._opened.append(int(p.value))
            bases.append(int(p.value) + o)
        arr = lambda o: torch.tensor([b + o for b in bases], dtype=torch.int64, device=device)  # noqa: E731
        self.peer_ctl = arr(0)
        self.peer_recv, self.peer_y = arr(off_recv), arr(off_y)
        self.recv_x_ptr = self.base + off_recv  # [cap, H] bf16
        self.y_out_ptr = self.base + off_y      # [cap, H] bf16
        self._act: torch.Tensor | None = None
        self._ws: torch.Tensor | None = None
        self.dest_base = torch.empty((world * el,), dtype=torch.int32, device=device)
        self.off_local = torch.empty((el + 1,), dtype=torch.int32, device=device)
        dist.barrier(group=group)  # every rank mapped every region before the first device barrier

    def workspace(self, need: int) -> torch.Tensor:
        """The stack's shared liblpmoe workspace (zeroed once: every call leaves its header zeroed).
        Grows only while layers are being built; a captured graph keeps the final address."""
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.zeros(need, dtype=torch.uint8, device=self.device)
        return self._ws

    def act(self, ffn: int) -> torch.Tensor:
        """Local [cap, ffn] bf16 scratch for the experts' SiLU(g)*u rows (shared by the stack)."""
        if self._act is None or self._act.shape[1] != ffn:
            self._act = torch.empty((self.cap, ffn), dtype=torch.bfloat16, device=self.device)
        return self._act

    def barrier(self, stream) -> None:
        """Device-side barrier over the P ranks, ordered on `stream`."""
        _native.check(self.lib.lp_ep_barrier(self.peer_ctl.data_ptr(), self.world, self.rank, stream),
                      "lp_ep_barrier")

    def exchange(self, counts: torch.Tensor, stream, rows_out: torch.Tensor | None = None) -> None:
        """Post this rank's per-global-expert counts to every rank, wait for every source's, plan
        dest_base / off_local (one launch); rows_out (int32 [1]) receives the rows this rank gets."""
        _native.check(self.lib.lp_ep_exchange(counts.data_ptr(), self.peer_ctl.data_ptr(), self.world, self.el,
                                              self.rank, self.dest_base.data_ptr(), self.off_local.data_ptr(),
                                              rows_out.data_ptr() if rows_out is not None else None, stream),
                      "lp_ep_exchange")

    def close(self) -> None:
        """Collective: every rank must call it (peers may still read this region until all have synced)."""
        if self.base:
            torch.cuda.synchronize(self.device)
            dist.barrier(group=self.group)
        for p in self._opened:
            self.lib.lp_ipc_close(p)
        self._opened = []
        if self.base:
            self.lib.lp_ipc_free(self.base)
            self.base = 0


class PeerEP:
    """Expert-parallel MoE layer over peer memory: no collective library on the data path.

    The NCCL path above moves rows with two `all_to_all_single` calls around a
    local re-permutation. Here every rank's `PeerRegion` is mapped by every rank
    (CUDA IPC: NVLink/NVSwitch P2P between GPUs) and each layer is (C-ABI calls,
    ep_p2p.cuh):
        route + index-only permute -> post counts -> barrier -> plan (per-destination
        row bases, own expert offsets) -> fused permute+dispatch into the owners'
        recv_x -> barrier -> grouped experts on recv_x -> y_out -> barrier ->
        fused receive+combine from the owners' y_out -> barrier.
    Received rows are expert-major, source-rank-major within an expert, so the
    owner's expert kernel runs on them directly (no re-permutation) and every
    (token, expert) row sees exactly the math of the single-GPU layer: outputs
    are bit-identical to GpuMoE on the same tokens (tests/test_gpu_ep_p2p.py).
    Pass the first layer's `.region` to the others of a stack (`region=`).
    """

    def __init__(self, shape: MoEShape, wr: torch.Tensor, w13_local: torch.Tensor, w2_local: torch.Tensor,
                 rank: int, world: int, max_tokens: int, group=None, region: PeerRegion | None = None):
        E, H, k = shape.num_experts, shape.hidden, shape.top_k
        require(E % world == 0, f"num_experts={E} must be divisible by the EP world size {world}")
        require(max_tokens >= 1, f"max_tokens must be >= 1, got {max_tokens}")
        self.shape, self.rank, self.world = shape, rank, world
        self.el = E // world
        self.max_tokens = max_tokens
        self.device = wr.device
        for name, t, shp in (("wr", wr, (E, H)), ("w13_local", w13_local, (self.el, 2 * shape.ffn, H)),
                             ("w2_local", w2_local, (self.el, H, shape.ffn))):
            _check_tensor(name, t, shp, torch.bfloat16)
        self.wr, self.w13, self.w2 = wr, w13_local, w2_local
        self.lib = _native.load()
        cap = max_tokens * k * world  # worst case: every rank's entries land on this rank
        if region is None:
            region = PeerRegion(self.device, rank, world, cap, H, self.el, group)
        require(region.world == world and region.rank == rank and region.cap >= cap and region.hidden == H
                and region.el == self.el, "region: incompatible PeerRegion for this layer")
        self.region = region
        # per-layer buffers sized once for max_tokens (no allocation on the layer path); the stats a
        # call returns alias them and stay valid until this layer's next call
        dev, S = self.device, max_tokens * k
        self._ids = torch.empty((max_tokens, k), dtype=torch.int32, device=dev)
        self._w = torch.empty((max_tokens, k), dtype=torch.float32, device=dev)
        self._counts = torch.zeros((E,), dtype=torch.int32, device=dev)
        self._offsets = torch.zeros((E + 1,), dtype=torch.int32, device=dev)
        self._slot_of = torch.empty((S,), dtype=torch.int32, device=dev)
        self._tok_of = torch.empty((S,), dtype=torch.int32, device=dev)
        self._dest_rank = torch.empty((S,), dtype=torch.int32, device=dev)
        self._dest_row = torch.empty((S,), dtype=torch.int32, device=dev)
        self._recv_rows = torch.zeros((1,), dtype=torch.int32, device=dev)
        need = max(int(self.lib.lp_moe_workspace_bytes(max_tokens, H, 128, E, k)),   # route + permute
                   int(self.lib.lp_moe_workspace_bytes(1, H, shape.ffn, self.el, 1)))  # expert tile plan
        self._ws_need = need
        region.workspace(need)  # one scratch per stack: its layers run in sequence on one stream

    @classmethod
    def from_full(cls, shape: MoEShape, wr, w13, w2, rank: int, world: int, max_tokens: int, group=None,
                  region: PeerRegion | None = None) -> "PeerEP":
        el = shape.num_experts // world
        sl = slice(rank * el, (rank + 1) * el)
        return cls(shape, wr, w13[sl].contiguous(), w2[sl].contiguous(), rank, world, max_tokens, group, region)

    def forward(self, x: torch.Tensor, out: torch.Tensor | None = None, prof=None) -> tuple[torch.Tensor, EPStats]:
        """prof: optional list of 5 CUDA events recorded at the stage boundaries (start | route +
        permute | exchange + dispatch | experts | combine) for bench.py's per-rank stage split.
        Every rank must call every layer (a rank with T = 0 still takes part in the exchange)."""
        s, P, el, lib, rg = self.shape, self.world, self.el, self.lib, self.region
        mark = (lambda i: prof[i].record()) if prof is not None else (lambda i: None)
        require(x.dim() == 2 and x.shape[1] == s.hidden, f"x must be [T, {s.hidden}], got {tuple(x.shape)}")
        T, H, k, E = x.shape[0], s.hidden, s.top_k, s.num_experts
        require(T <= self.max_tokens, f"T={T} exceeds max_tokens={self.max_tokens}")
        _check_tensor("x", x, (T, H), torch.bfloat16)
        st = _stream_ptr(self.device)
        ws = rg.workspace(self._ws_need)
        # (pointers from the full buffers: an empty view's data_ptr() is 0, which the ABI rejects)
        ids, w, counts = self._ids[:T], self._w[:T], self._counts
        mark(0)
        if T:  # route, then the index-only permutation: slots within each (global) expert, no x_perm
            _native.check(lib.lp_moe_route(x.data_ptr(), self.wr.data_ptr(), T, H, E, k, int(s.norm_topk_prob),
                                           self._ids.data_ptr(), self._w.data_ptr(), ws.data_ptr(), ws.numel(), st),
                          "lp_moe_route")
        _native.check(lib.lp_moe_permute(self._ids.data_ptr(), x.data_ptr(), T, H, E, k, counts.data_ptr(),
                                         self._offsets.data_ptr(), self._slot_of.data_ptr(), self._tok_of.data_ptr(),
                                         None, ws.data_ptr(), ws.numel(), st), f"lp_moe_permute (T={T})")
        mark(1)
        rg.exchange(counts, st, self._recv_rows)  # counts to every rank + wait for every source + plan
        _native.check(lib.lp_ep_dispatch(x.data_ptr(), self._ids.data_ptr(), self._slot_of.data_ptr(),
                                         self._offsets.data_ptr(), rg.dest_base.data_ptr(), rg.peer_recv.data_ptr(),
                                         T, H, k, el, self._dest_rank.data_ptr(), self._dest_row.data_ptr(), st),
                      "lp_ep_dispatch")
        rg.barrier(st)
        mark(2)
        # rows received stay on the device (off_local[El]): capacity-sized launch, tile width from the
        # expected T*k rows; no host sync, so the whole layer is stream-ordered and graph-capturable
        act = rg.act(s.ffn)
        _native.check(lib.lp_moe_experts_rows(rg.recv_x_ptr, rg.off_local.data_ptr(), rg.cap, max(T, 1) * k,
                                              self.w13.data_ptr(), self.w2.data_ptr(), H, s.ffn, el,
                                              act.data_ptr(), rg.y_out_ptr, ws.data_ptr(), ws.numel(), st),
                      "lp_moe_experts_rows")
        rg.barrier(st)
        mark(3)
        y = out if out is not None else torch.empty((T, H), dtype=torch.bfloat16, device=self.device)
        _native.check(lib.lp_ep_combine(rg.peer_y.data_ptr(), self._dest_rank.data_ptr(), self._dest_row.data_ptr(),
                                        self._w.data_ptr(), T, H, k, y.data_ptr(), st), "lp_ep_combine")
        # no end-of-layer barrier: see ep_p2p.cuh (the next exchange / dispatch barrier orders reuse)
        mark(4)
        self.last_ids, self.last_weights = ids, w
        # (send_splits: rows per destination = counts.view(P, El).sum(1), left to the caller: no extra launch)
        return y, EPStats(counts, self._recv_rows[0], None, [], s)

    __call__ = forward

    def forward_host(self, x_host: torch.Tensor, y_host: torch.Tensor | None = None,
                     x_dev: torch.Tensor | None = None):
        """End-to-end call with host buffers: H2D copy, EP layer, D2H copy."""
        xd = x_dev if x_dev is not None else torch.empty(x_host.shape, dtype=x_host.dtype, device=self.device)
        xd.copy_(x_host, non_blocking=True)
        yd, stats = self.forward(xd)
        if y_host is None:
            y_host = torch.empty(yd.shape, dtype=yd.dtype, pin_memory=True)
        y_host.copy_(yd, non_blocking=True)
        return y_host, stats
