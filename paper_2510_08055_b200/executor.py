"""Layered executor: runs the reference planner's iterations on real MoE layers on the B200.

SURVEY.md §8(f) row 1. The reference's own engine plans every iteration
(`moesim.engine.run` -> `scheduler.plan_for`, scheduler.py:286-291) and, inside
`refdrive.measured_costs(executor=...)`, hands each `BatchPlan`
(scheduler.py:82-92) to `LayeredExecutor.run_plan`, which runs the iteration's
MoE work through a stack of resident `GpuMoE` layers and returns the measured
device time and the experts each layer's routing really hit; attention / dense
projections stay the reference's modelled costs (out of scope).

Per iteration and per MoE layer l the routed batch is exactly what the
reference engine charges at engine.py:137-154: every decoding request's token
plus the prefill slices whose layer range contains l. Hidden states:
  * each prefilling request owns a stash [input_len, H] (bf16) that carries its
    prompt activations between iterations (layered: after group g; chunked:
    the processed chunk rows);
  * each decoding request owns one row, carried from iteration to iteration;
  * layers are applied as a residual stream h <- h + MoE_l(h), so routing sees
    O(1) activations at every depth (the MoE-only model has no attention/norm).
Layers whose active row set is identical are run back to back on one
contiguous buffer (decode rows first, then the slices), so a layered
iteration is two buffers (designated group: decode+prompt rows, other layers:
decode rows) and a chunked iteration is one.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from .moe import GpuMoE, Workspace, add_rmsnorm
from .synthetic import router_weight
from .types import MoEShape, require


class _DecodeGraphs:
    """CUDA graphs of single decode-size layer steps (T <= max_tokens rows): a step is
    `add_rmsnorm(x, y_prev, xn); layer(xn) -> y, counts`, captured once per (T, layer,
    first?) on static buffers and replayed. Decode layers move a few hundred MB in
    ~40 us, which the per-call host cost (Python + ctypes + 5 launches, ~40 us)
    would otherwise match: replay keeps a decode step device-bound. The captured
    layers run on their own small workspace (the shared one grows for prefill
    batches, which would move its address under a captured graph)."""

    def __init__(self, model: "MoEModel", max_tokens: int):
        self.model, self.max_tokens = model, max_tokens
        dev, s = model.device, model.shape
        self.workspace = Workspace(dev)
        self.layers = [GpuMoE(s, m.wr, m.w13, m.w2, workspace=self.workspace) for m in model.layers]
        # fixed size (the largest any T <= max_tokens asks for): never regrows under a graph
        self.workspace.get(max(self.layers[0].workspace_bytes(t) for t in range(1, max_tokens + 1)))
        for layer in self.layers:
            layer._bufs(max_tokens)
        self.pool = torch.cuda.graph_pool_handle()
        self.bufs: dict[int, tuple] = {}
        self.graphs: dict[tuple, torch.cuda.CUDAGraph] = {}

    def _buffers(self, T: int):
        b = self.bufs.get(T)
        if b is None:
            dev, s = self.model.device, self.model.shape
            b = (torch.zeros((T, s.hidden), dtype=torch.bfloat16, device=dev),   # x (residual, in place)
                 torch.zeros((T, s.hidden), dtype=torch.bfloat16, device=dev),   # xn
                 torch.zeros((T, s.hidden), dtype=torch.bfloat16, device=dev),   # y
                 torch.zeros((self.model.num_layers, s.num_experts), dtype=torch.int32, device=dev))  # counts
            self.bufs[T] = b
        return b

    def _graph(self, T: int, layer: int, first: bool) -> torch.cuda.CUDAGraph:
        key = (T, layer, first)
        g = self.graphs.get(key)
        if g is None:
            x, xn, y, c = self._buffers(T)
            step = lambda: (add_rmsnorm(x, None if first else y, xn),  # noqa: E731
                            self.layers[layer](xn, out=y, counts_out=c[layer]))
            dev = self.model.device
            side = torch.cuda.Stream(dev)
            side.wait_stream(torch.cuda.current_stream(dev))
            saved = x.clone(), y.clone()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(side):
                step()  # warm-up outside the capture (kernel attributes, descriptors)
                # capture_begin/end directly: the torch.cuda.graph context's gc.collect() and
                # empty_cache() per capture would dominate capturing hundreds of small graphs
                g.capture_begin(pool=self.pool)
                step()
                g.capture_end()
            torch.cuda.current_stream(dev).wait_stream(side)
            x.copy_(saved[0])
            y.copy_(saved[1])
            self.graphs[key] = g
        return g

    def capture(self, token_counts) -> None:
        """Capture every layer step for these batch sizes up front (outside timed iterations)."""
        for T in token_counts:
            if 0 < T <= self.max_tokens:
                for layer in range(self.model.num_layers):
                    for first in (True, False):
                        self._graph(T, layer, first)
        torch.cuda.synchronize(self.model.device)

    def run_segment(self, x: torch.Tensor, l0: int, l1: int, counts: torch.Tensor) -> torch.Tensor:
        T = x.shape[0]
        sx, sxn, sy, sc = self._buffers(T)
        sx.copy_(x)
        for i, layer in enumerate(range(l0, l1)):
            self._graph(T, layer, i == 0).replay()
        counts[l0:l1] += sc[l0:l1]
        add_rmsnorm(sx, sy, sxn)
        x.copy_(sx)
        return x


class MoEModel:
    """`num_layers` resident MoE layers of `shape` with random-init weights."""

    # tokens per lp_moe_forward call: a layered-prefill cohort can hold hundreds of thousands of prompt
    # tokens (C5 with measured attention reached 400 K), above the C-ABI's T limit and the x_perm /
    # y_perm workspace worth keeping; larger segments run each layer in row slices (per-token math,
    # so the rows are bit-identical to one call)
    max_call_tokens = 65536

    def __init__(self, shape: MoEShape, num_layers: int, device="cuda", seed: int = 0, std: float = 0.02,
                 graph_tokens: int = 0):
        self.shape, self.num_layers = shape, num_layers
        self.device = torch.device(device)
        self.layers: list[GpuMoE] = []
        self.workspace = Workspace(self.device)  # one scratch for the whole stack (layers run in order)
        for i in range(num_layers):
            wr, w13, w2 = layer_weights(shape, self.device, seed, i, std)
            self.layers.append(GpuMoE(shape, wr, w13, w2, workspace=self.workspace))
        # decode-size segments (T <= graph_tokens) replay per-layer CUDA graphs
        self.graphs = _DecodeGraphs(self, graph_tokens) if graph_tokens > 0 else None

    def run_segment(self, x: torch.Tensor, l0: int, l1: int, counts: torch.Tensor, events=None) -> torch.Tensor:
        """h <- h + MoE_l(RMSNorm(h)) for l in [l0, l1) (Qwen3's pre-MoE norm keeps the
        residual stream bounded); per-expert counts of layer l are added into counts[l].
        events: a list that receives the (start, end) CUDA events around the MoE work."""
        T = x.shape[0]
        e0, e1 = _timed(events)
        e0.record()
        if self.graphs is not None and 0 < T <= self.graphs.max_tokens:
            x = self.graphs.run_segment(x, l0, l1, counts)
            e1.record()
            return x
        xn = torch.empty_like(x)
        y = torch.empty_like(x)
        c = torch.empty((l1 - l0, self.shape.num_experts), dtype=torch.int32, device=self.device)
        delta = None
        M = self.max_call_tokens
        part = torch.empty((self.shape.num_experts,), dtype=torch.int32, device=self.device) if T > M else None
        for i, layer in enumerate(range(l0, l1)):
            add_rmsnorm(x, delta, xn)
            if part is None:
                self.layers[layer](xn, out=y, counts_out=c[i])
            else:
                c[i].zero_()
                for r0 in range(0, T, M):
                    self.layers[layer](xn[r0:r0 + M], out=y[r0:r0 + M], counts_out=part)
                    c[i] += part
            delta = y
        if delta is not None and T:
            add_rmsnorm(x, delta, xn)
        e1.record()
        counts[l0:l1] += c
        return x

    # single device: nothing to reduce across ranks
    def reduce_max(self, v: float) -> float:
        return v

    def reduce_counts(self, counts: torch.Tensor) -> torch.Tensor:
        return counts


def layer_weights(shape: MoEShape, device: torch.device, seed: int, i: int, std: float = 0.02):
    """Random-init weights of layer i (router on the dyadic grid, experts N(0, std^2) in bf16): the
    single-GPU and expert-parallel stacks build identical layers from the same seed."""
    g = torch.Generator(device=device).manual_seed(seed * 1000 + i)
    E, H, I = shape.num_experts, shape.hidden, shape.ffn
    w13 = (torch.randn((E, 2 * I, H), generator=g, device=device) * std).to(torch.bfloat16)
    w2 = (torch.randn((E, H, I), generator=g, device=device) * std).to(torch.bfloat16)
    wr = router_weight(E, H, seed * 1000 + i).to(device)
    return wr, w13, w2


def _timed(events):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if events is not None:
        events.append((e0, e1))
    return e0, e1


def shard_rows(T: int, rank: int, world: int) -> tuple[int, int]:
    """Rank `rank`'s contiguous share [lo, hi) of a segment's T rows (token-level data parallelism)."""
    return T * rank // world, T * (rank + 1) // world


def gather_rows(x: torch.Tensor, xl: torch.Tensor, rank: int, world: int, group=None,
                via_host: bool = False) -> torch.Tensor:
    """All-gather every rank's processed share back into the replicated x (in place; uneven shares
    padded to ceil(T / world) rows). via_host: stage through host memory (gloo; ranks sharing a GPU)."""
    T, H = x.shape
    n = (T + world - 1) // world
    pad = torch.zeros((n, H), dtype=x.dtype, device=x.device)
    pad[: xl.shape[0]].copy_(xl)
    if via_host:
        parts = [torch.empty((n, H), dtype=x.dtype) for _ in range(world)]
        dist.all_gather(parts, pad.cpu(), group=group)
        full = torch.cat(parts).to(x.device)
    else:
        full = torch.empty((world * n, H), dtype=x.dtype, device=x.device)
        dist.all_gather_into_tensor(full, pad, group=group)
    for r in range(world):
        a, b = shard_rows(T, r, world)
        if r != rank and b > a:
            x[a:b].copy_(full[r * n: r * n + (b - a)])
    return x


class EPMoEModel:
    """`num_layers` expert-parallel MoE layers (BASELINE config 5): rank r of P holds
    experts [r*E/P, (r+1)*E/P) of every layer (ep.PeerEP: fused dispatch / combine over peer
    memory, one PeerRegion shared by the stack). The MoE is token-data-parallel: every rank keeps
    the full hidden state (replicated, as attention/dense would produce it), runs the layers on
    its contiguous share of each segment's rows, and the processed rows are all-gathered back
    after the segment (outside the timed MoE region: it stands for the attention's own exchange).
    Per token the math is the single-GPU layer's, so hidden states are bit-identical to MoEModel
    built from the same seed (tests/test_gpu_ep_executor.py). Every rank must run every segment.
    max_tokens: the largest segment (all ranks' rows) the stack will see."""

    def __init__(self, shape: MoEShape, num_layers: int, rank: int, world: int, max_tokens: int,
                 device="cuda", seed: int = 0, std: float = 0.02, group=None):
        from .ep import PeerEP

        self.shape, self.num_layers, self.rank, self.world, self.group = shape, num_layers, rank, world, group
        self.device = torch.device(device)
        self.max_local = (max_tokens + world - 1) // world
        el = shape.num_experts // world
        sl = slice(rank * el, (rank + 1) * el)
        self.layers: list = []
        region = None
        for i in range(num_layers):
            wr, w13, w2 = layer_weights(shape, self.device, seed, i, std)
            ep = PeerEP(shape, wr, w13[sl].contiguous(), w2[sl].contiguous(), rank, world, self.max_local,
                        group=group, region=region)
            del w13, w2
            region = ep.region
            self.layers.append(ep)
        self.region = region
        self.graphs = None
        self._gloo = dist.get_backend(group) != "nccl"

    def _rows(self, T: int) -> tuple[int, int]:
        return shard_rows(T, self.rank, self.world)

    def run_segment(self, x: torch.Tensor, l0: int, l1: int, counts: torch.Tensor, events=None) -> torch.Tensor:
        T, H = x.shape
        lo, hi = self._rows(T)
        xl = x[lo:hi]
        xn = torch.empty_like(xl)
        y = torch.empty_like(xl)
        e0, e1 = _timed(events)
        e0.record()
        delta = None
        for layer in range(l0, l1):
            add_rmsnorm(xl, delta, xn)
            _, st = self.layers[layer](xn, out=y)
            counts[layer] += st.counts
            delta = y
        if delta is not None and hi > lo:
            add_rmsnorm(xl, delta, xn)
        e1.record()
        return self._gather(x, xl)

    def _gather(self, x: torch.Tensor, xl: torch.Tensor) -> torch.Tensor:
        return gather_rows(x, xl, self.rank, self.world, self.group, via_host=self._gloo)

    def _reduce(self, t: torch.Tensor, op) -> torch.Tensor:
        if self._gloo:
            c = t.cpu()
            dist.all_reduce(c, op=op, group=self.group)
            return c.to(t.device)
        dist.all_reduce(t, op=op, group=self.group)
        return t

    def reduce_max(self, v: float) -> float:
        """MoE device time of an iteration: the slowest rank's (the layers barrier every rank)."""
        return float(self._reduce(torch.tensor([v], dtype=torch.float64, device=self.device), dist.ReduceOp.MAX)[0])

    def reduce_counts(self, counts: torch.Tensor) -> torch.Tensor:
        """Per-layer expert counts of all ranks' tokens (experts hit = nnz of the sum)."""
        return self._reduce(counts.clone(), dist.ReduceOp.SUM)

    def close(self) -> None:
        if self.region is not None:
            self.region.close()
            self.region = None


@dataclass
class MoEIteration:
    """What one planned iteration's MoE work measured (refdrive turns it into a KernelCost)."""

    device_s: float            # device time of the MoE layer calls (CUDA events around the segments)
    routed: list               # routed tokens through each layer (engine.py:137-154 semantics)
    experts_hit: list          # experts the routing touched in each layer (nnz of the real counts)
    includes_attention: bool = False  # device_s also covers attention + dense projections (measured)


def _finished(r) -> bool:
    return getattr(r.phase, "value", r.phase) == "finished"


class AttentionDense:
    """Measured attention + dense projections for the serving executor: per layer,
    RMSNorm → QKV projection (cuBLAS) → causal GQA attention over each request's KV cache (PyTorch
    scaled_dot_product_attention, library kernels) → output projection (cuBLAS) → residual add.

    Qwen3-30B-A3B attention shapes (configs/qwen30b.toml): 32 query heads, 4 KV heads, head_dim 128
    (Wqkv [4096 + 2 x 512, 2048], Wo [2048, 4096], random init; no RoPE — positions only enter
    through the causal masks). Each request owns a KV cache [layers, input_len + output_len, 4, 128]
    (K and V, bf16), filled by its prefill slices (layered: the whole prompt per layer group;
    chunked: the chunk attends to the cached KV of the earlier chunks) and one row per decode step;
    decode rows at the same context length are batched into one SDPA call. These are library
    kernels on the serving path, not the MoE hot path: they replace the reference's modelled
    attention_cost / dense_cost (costmodel.py:88-145) with measured time."""

    HEADS, KV_HEADS, HEAD_DIM = 32, 4, 128

    def __init__(self, hidden: int, num_layers: int, device, seed: int = 0, std: float = 0.02,
                 pool_slots: int = 0, pool_len: int = 0):
        self.H, self.L = hidden, num_layers
        self.device = torch.device(device)
        qd, kd = self.HEADS * self.HEAD_DIM, self.KV_HEADS * self.HEAD_DIM
        self.qd, self.kd = qd, kd
        g = torch.Generator(device=self.device).manual_seed(seed * 7919 + 17)
        self.wqkv = [(torch.randn((qd + 2 * kd, hidden), generator=g, device=self.device) * std).to(torch.bfloat16)
                     for _ in range(num_layers)]
        self.wo = [(torch.randn((hidden, qd), generator=g, device=self.device) * std).to(torch.bfloat16)
                   for _ in range(num_layers)]
        self.kv: dict[int, tuple[torch.Tensor, torch.Tensor]] = {}
        # pooled KV (pool_slots > 0): every request's cache is a slot of one [L, slots, pool_len, 4, 128]
        # tensor, so a decode step's rows (any mix of context lengths) write and read their KV with a
        # few indexed ops and ONE padded, masked SDPA call per layer instead of per-request work
        self.Kp = self.Vp = None
        if pool_slots > 0:
            shape = (num_layers, pool_slots, pool_len, self.KV_HEADS, self.HEAD_DIM)
            # zero-filled: masked-out positions get softmax weight 0, and 0 x (uninitialised NaN) is NaN
            self.Kp = torch.zeros(shape, dtype=torch.bfloat16, device=self.device)
            self.Vp = torch.zeros(shape, dtype=torch.bfloat16, device=self.device)
            self.arange = torch.arange(pool_len, device=self.device)
            self.free = list(range(pool_slots - 1, -1, -1))
            self.slot: dict[int, int] = {}
            self.pool_len = pool_len
        self._plan_key = None
        self._plan = None

    def cache(self, rid: int, length: int):
        c = self.kv.get(rid)
        if c is None:
            if self.Kp is not None:
                require(length <= self.pool_len and self.free, "AttentionDense: KV pool exhausted")
                sl = self.free.pop()
                self.slot[rid] = sl
                c = (self.Kp[:, sl], self.Vp[:, sl])
            else:
                shape = (self.L, length, self.KV_HEADS, self.HEAD_DIM)
                c = (torch.empty(shape, dtype=torch.bfloat16, device=self.device),
                     torch.empty(shape, dtype=torch.bfloat16, device=self.device))
            self.kv[rid] = c
        return c

    def drop(self, rid: int) -> None:
        if self.kv.pop(rid, None) is not None and self.Kp is not None:
            self.free.append(self.slot.pop(rid))

    def pool_plan(self, spans: list):
        """Host side of the pooled decode step: (B, slots, positions, ctx) of the leading run of one-row
        spans (a one-token prefill chunk at position p computes exactly what a decode row does), with
        a slot assigned to every new request; ctx is the longest context rounded up to 128 (fewer
        distinct attention shapes), positions past a row's own are masked."""
        dec = []
        for sp in spans:
            if sp[2] != 1:
                break
            dec.append(sp)
        for sp in dec:
            self.cache(sp[0], sp[3])
        if not dec:
            return 0, [], [], 0
        ctx = min(self.pool_len, -(-(max(sp[1] for sp in dec) + 1) // 128) * 128)
        return len(dec), [self.slot[sp[0]] for sp in dec], [sp[1] for sp in dec], ctx

    def _decode_plan(self, spans: list):
        """Device index tensor [2, B] (slots; positions) of pool_plan, built once per segment."""
        if self._plan_key is spans:
            return self._plan
        B, slots, pos, ctx = self.pool_plan(spans)
        plan = (B, torch.tensor([slots, pos], device=self.device), ctx) if B else None
        self._plan_key, self._plan = spans, plan
        return plan

    def _heads(self, t: torch.Tensor) -> torch.Tensor:
        """[B, 4, ctx, 128] KV heads -> [B, 32, ctx, 128] (GQA by repetition: SDPA's fused backends then
        take the lower-right causal bias; with enable_gqa some shapes fell back to the math path)."""
        return t.repeat_interleave(self.HEADS // self.KV_HEADS, dim=1)

    def layer(self, l: int, h: torch.Tensor, spans: list, plan=None) -> None:
        """h [T, H] (in place) += Wo · attention(QKV(RMSNorm(h))); spans: (rid, pos0, n, cache_len) per
        consecutive row run, decode rows first (n = 1), in row order."""
        import torch.nn.functional as F
        from torch.nn.attention import SDPBackend, sdpa_kernel

        T = h.shape[0]
        # cuDNN's sm100 attention first (PyTorch's own flash kernel, built for sm80/90, ran the
        # lower-right-causal chunk case ~5x slower on B200)
        order = [SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION, SDPBackend.EFFICIENT_ATTENTION,
                 SDPBackend.MATH]
        with sdpa_kernel(order, set_priority=True):
            self._layer(F, l, h, T, spans, plan)

    def _layer(self, F, l: int, h: torch.Tensor, T: int, spans: list, plan=None) -> None:
        xn = torch.empty_like(h)
        add_rmsnorm(h, None, xn)
        qkv = xn @ self.wqkv[l].t()
        q = qkv[:, :self.qd].view(T, self.HEADS, self.HEAD_DIM)
        k = qkv[:, self.qd:self.qd + self.kd].view(T, self.KV_HEADS, self.HEAD_DIM)
        v = qkv[:, self.qd + self.kd:].view(T, self.KV_HEADS, self.HEAD_DIM)
        out = torch.empty((T, self.HEADS, self.HEAD_DIM), dtype=h.dtype, device=h.device)
        row = 0
        i = 0
        if self.Kp is not None:  # pooled: every decode row (leading spans) in one masked SDPA call
            if plan is None:
                plan = self._decode_plan(spans)
            if plan is not None:
                B, idx, ctx = plan
                slots, pos = idx[0], idx[1]
                mask = (self.arange[:ctx][None, :] <= pos[:, None])[:, None, None, :]     # [B, 1, 1, ctx]
                self.Kp[l, slots, pos] = k[:B]
                self.Vp[l, slots, pos] = v[:B]
                # GQA without repeating K/V: the 8 query heads of a KV head are 8 query rows of it
                qg = q[:B].view(B, self.KV_HEADS, self.HEADS // self.KV_HEADS, self.HEAD_DIM)
                kb = self.Kp[l, slots, :ctx].transpose(1, 2)                        # [B, 4, ctx, 128]
                vb = self.Vp[l, slots, :ctx].transpose(1, 2)
                o = F.scaled_dot_product_attention(qg, kb, vb, attn_mask=mask)     # [B, 4, 8, 128]
                out[:B] = o.reshape(B, self.HEADS, self.HEAD_DIM)
                row = i = B
        while i < len(spans):
            rid, pos0, n, clen = spans[i]
            if n == 1:  # a run of decode rows at the same position: one batched SDPA
                j = i
                while j < len(spans) and spans[j][2] == 1 and spans[j][1] == pos0:
                    j += 1
                ks, vs = [], []
                for b in range(i, j):
                    K, V = self.cache(spans[b][0], spans[b][3])
                    K[l, pos0] = k[row + b - i]
                    V[l, pos0] = v[row + b - i]
                    ks.append(K[l, :pos0 + 1])
                    vs.append(V[l, :pos0 + 1])
                B = j - i
                qb = q[row:row + B].unsqueeze(2).contiguous()                      # [B, 32, 1, 128]
                kb = self._heads(torch.stack(ks).transpose(1, 2))                  # [B, 32, ctx, 128]
                vb = self._heads(torch.stack(vs).transpose(1, 2))
                out[row:row + B] = F.scaled_dot_product_attention(qb, kb, vb)[:, :, 0]
                row += B
                i = j
                continue
            K, V = self.cache(rid, clen)
            K[l, pos0:pos0 + n] = k[row:row + n]
            V[l, pos0:pos0 + n] = v[row:row + n]
            qb = q[row:row + n].transpose(0, 1).unsqueeze(0).contiguous()          # [1, 32, n, 128]
            kb = self._heads(K[l, :pos0 + n].transpose(0, 1).unsqueeze(0))          # [1, 32, pos0 + n, 128]
            vb = self._heads(V[l, :pos0 + n].transpose(0, 1).unsqueeze(0))
            if pos0 == 0:
                o = F.scaled_dot_product_attention(qb, kb, vb, is_causal=True)
            else:  # a later chunk: query i (position pos0 + i) sees keys 0 .. pos0 + i (lower-right causal,
                # which SDPA's fused kernels take directly; an explicit mask falls back to the math path)
                from torch.nn.attention.bias import causal_lower_right

                o = F.scaled_dot_product_attention(qb, kb, vb, attn_mask=causal_lower_right(n, pos0 + n))
            out[row:row + n] = o[0].transpose(0, 1)
            row += n
            i += 1
        h += out.view(T, self.qd) @ self.wo[l].t()


class _IterationGraphs:
    """CUDA graphs of whole decode-only iterations in measured-attention mode: for every layer,
    pooled-KV attention + dense projections (AttentionDense) and then the MoE sublayer, all L layers
    in one graph, captured once per (decode rows, context bucket) on static buffers and replayed.
    Eagerly a decode iteration is ~16 small launches per layer, and the host cost of issuing them
    (~350 us per layer) would be what the engine's device-timed iteration measures; replay keeps it
    device-bound. The MoE layers run on their own fixed workspace (the stack's shared one grows for
    prefill batches, which would move its address under a captured graph)."""

    def __init__(self, stack: "MoEModel", att: AttentionDense, max_rows: int):
        require(att.Kp is not None, "iteration graphs need AttentionDense(pool_slots > 0)")
        self.stack, self.att, self.max_rows = stack, att, max_rows
        s = stack.shape
        self.workspace = Workspace(stack.device)
        self.layers = [GpuMoE(s, m.wr, m.w13, m.w2, workspace=self.workspace) for m in stack.layers]
        self.workspace.get(max(self.layers[0].workspace_bytes(t) for t in range(1, max_rows + 1)))
        for layer in self.layers:
            layer._bufs(max_rows)
        self.pool = torch.cuda.graph_pool_handle()
        self.graphs: dict[tuple, tuple] = {}

    def _step(self, x, xn, y, c, plan) -> None:
        for l in range(self.stack.num_layers):
            self.att.layer(l, x, [], plan)
            add_rmsnorm(x, None, xn)
            self.layers[l](xn, out=y, counts_out=c[l])
            add_rmsnorm(x, y, xn)

    def _graph(self, B: int, ctx: int):
        key = (B, ctx)
        g = self.graphs.get(key)
        if g is None:
            dev, H = self.stack.device, self.stack.shape.hidden
            x = torch.zeros((B, H), dtype=torch.bfloat16, device=dev)
            xn, y = torch.zeros_like(x), torch.zeros_like(x)
            c = torch.zeros((self.stack.num_layers, self.stack.shape.num_experts), dtype=torch.int32, device=dev)
            idx = torch.zeros((2, B), dtype=torch.int64, device=dev)
            plan = (B, idx, ctx)
            side = torch.cuda.Stream(dev)
            side.wait_stream(torch.cuda.current_stream(dev))
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.stream(side):
                # warm-up outside the capture (attention plans, kernel attributes) on slot 0 / position
                # 0 of the zero inputs: the replay that follows rewrites every KV row it reads
                kp0, vp0 = self.att.Kp[:, :1, :1].clone(), self.att.Vp[:, :1, :1].clone()
                self._step(x, xn, y, c, plan)
                graph.capture_begin(pool=self.pool)
                self._step(x, xn, y, c, plan)
                graph.capture_end()
                self.att.Kp[:, :1, :1] = kp0
                self.att.Vp[:, :1, :1] = vp0
            torch.cuda.current_stream(dev).wait_stream(side)
            g = (graph, x, c, idx)
            self.graphs[key] = g
        return g

    def run(self, dec: torch.Tensor, slots: list, pos: list, ctx: int, counts: torch.Tensor, events: list):
        graph, x, c, idx = self._graph(dec.shape[0], ctx)
        idx.copy_(torch.tensor([slots, pos], dtype=torch.int64), non_blocking=False)
        x.copy_(dec)
        e0, e1 = _timed(events)
        e0.record()
        graph.replay()
        e1.record()
        counts += c
        return x.clone()


class LayeredExecutor:
    """Runs a reference `BatchPlan` on the resident layer stack (duck-typed on moesim's SimState:
    `state.request(rid)` with `input_len` and `phase`)."""

    def __init__(self, stack: MoEModel, embed_seed: int = 0, keep_final_prompt: bool = False,
                 attention: AttentionDense | None = None, iteration_graphs: int = 0):
        self.stack = stack
        self.attention = attention  # measured attention + dense projections (None: modelled by the reference)
        # decode-only iterations of up to this many rows replay one CUDA graph of all layers
        # (measured attention with a pooled KV cache; single-GPU stack)
        self.igraphs = (_IterationGraphs(stack, attention, iteration_graphs)
                        if iteration_graphs > 0 and attention is not None else None)
        self.keep_final_prompt = keep_final_prompt
        self.final_prompt: dict[int, torch.Tensor] = {}
        self.final_decode: dict[int, torch.Tensor] = {}  # last decode hidden row of finished requests
        self.dev = stack.device
        self.H = stack.shape.hidden
        self.stash: dict[int, torch.Tensor] = {}    # rid -> [input_len, H] prompt activations
        self.decode_row: dict[int, torch.Tensor] = {}  # rid -> [H] current decode hidden
        self.embed_seed = embed_seed
        self.iter_log: list[dict] = []

    def _prompt(self, state, rid: int) -> torch.Tensor:
        h = self.stash.get(rid)
        if h is None:  # synthetic prompt embedding (no tokenizer / embedding table: out of scope)
            g = torch.Generator(device=self.dev).manual_seed(self.embed_seed * 1_000_003 + rid)
            h = torch.randn((state.request(rid).input_len, self.H), generator=g, device=self.dev).to(torch.bfloat16)
            self.stash[rid] = h
        return h

    def _decode_rows(self, plan) -> list[torch.Tensor]:
        rows = []
        for rid in plan.decode_ids:
            row = self.decode_row.get(rid)
            if row is None:  # prefill finished last iteration: its last prompt row seeds decoding
                h = self.stash.pop(rid)
                if self.keep_final_prompt:
                    self.final_prompt[rid] = h
                row = h[-1].clone()
                self.decode_row[rid] = row
            rows.append(row)
        return rows

    @staticmethod
    def _decode_span(state, rid: int) -> tuple:
        r = state.request(rid)  # the decode row is the token at position input_len + emitted - 1
        return rid, r.input_len + r.tokens_emitted - 1, 1, r.input_len + r.output_len

    def run_plan(self, state, plan) -> MoEIteration:
        L = self.stack.num_layers
        if self.attention is not None:  # KV caches of requests the engine retired since the last call
            for rid in [k for k in self.attention.kv if _finished(state.request(k))]:
                self.attention.drop(rid)
        for rid in [k for k in self.stash if _finished(state.request(k))]:
            h = self.stash.pop(rid)  # prompt finished without a decode step (output_len == 1)
            if self.keep_final_prompt:
                self.final_prompt[rid] = h
        dec_rows = self._decode_rows(plan)
        D = len(dec_rows)
        cuts = sorted({0, L} | {a.layer_start for a in plan.prefill_assignments}
                      | {a.layer_end for a in plan.prefill_assignments})
        counts = torch.zeros((L, self.stack.shape.num_experts), dtype=torch.int32, device=self.dev)
        routed = [D] * L
        for a in plan.prefill_assignments:
            for layer in range(a.layer_start, a.layer_end):
                routed[layer] += a.num_tokens
        events, attn_events = [], []
        dec = torch.stack(dec_rows) if D else torch.empty((0, self.H), dtype=torch.bfloat16, device=self.dev)
        graphed = False
        if self.igraphs is not None and 0 < D <= self.igraphs.max_rows and not plan.prefill_assignments:
            spans = [self._decode_span(state, rid) for rid in plan.decode_ids]
            B, slots, pos, ctx = self.attention.pool_plan(spans)
            dec = self.igraphs.run(dec, slots, pos, ctx, counts, events)
            graphed, cuts = True, []
        for l0, l1 in zip(cuts, cuts[1:]):
            act = [a for a in plan.prefill_assignments if a.layer_start <= l0 < a.layer_end]
            parts = [dec] + [self._prompt(state, a.request_id)[a.token_start:a.token_end] for a in act]
            if sum(p.shape[0] for p in parts) == 0:
                continue
            x = torch.cat(parts) if len(parts) > 1 else parts[0].clone()
            if self.attention is None:
                # only the MoE work is timed (not the embedding, the concatenation, the copy-back or an
                # expert-parallel stack's row gather): the stack records the events
                x = self.stack.run_segment(x, l0, l1, counts, events)
            else:  # per layer: attention + dense (measured), then the MoE sublayer
                spans = [self._decode_span(state, rid) for rid in plan.decode_ids]
                spans += [(a.request_id, a.token_start, a.num_tokens,
                           state.request(a.request_id).input_len + state.request(a.request_id).output_len)
                          for a in act]
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for layer in range(l0, l1):
                    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a0.record()
                    self.attention.layer(layer, x, spans)
                    a1.record()
                    attn_events.append((a0, a1))
                    x = self.stack.run_segment(x, layer, layer + 1, counts)
                e1.record()
                events.append((e0, e1))
            dec = x[:D]
            off = D
            for a in act:
                n = a.num_tokens
                self._prompt(state, a.request_id)[a.token_start:a.token_end].copy_(x[off:off + n])
                off += n
        for rid, row in zip(plan.decode_ids, dec):
            self.decode_row[rid] = row
        torch.cuda.synchronize(self.dev)
        moe_s = self.stack.reduce_max(sum(a.elapsed_time(b) for a, b in events) * 1e-3)
        nnz = (self.stack.reduce_counts(counts) > 0).sum(dim=1).cpu().tolist()
        self.iter_log.append({"moe_s": moe_s, "routed": routed, "experts_hit": nnz, "decode": D,
                              "prefill_tokens": plan.prefill_tokens,
                              "attn_s": sum(a.elapsed_time(b) for a, b in attn_events) * 1e-3,
                              "graphed": graphed})
        # drop finished requests' state (the engine retires them after this call)
        live = set(plan.decode_ids) | {r.id for r in state.decoding}
        for rid in [k for k in self.decode_row if k not in live]:
            row = self.decode_row.pop(rid)
            if self.keep_final_prompt:
                self.final_decode[rid] = row
        return MoEIteration(moe_s, routed, nnz, self.attention is not None)
