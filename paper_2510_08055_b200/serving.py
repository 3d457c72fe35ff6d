"""Iteration-level serving loop: layered / chunked / hybrid prefill planning,
KV-gated FCFS admission, clocked iterations and TTFT/TBT accounting.

A host-side restatement of the reference simulator's planner and engine
(moesim/scheduler.py:23-364, engine.py:120-351, metrics.py:11-157) so the
GPU executor can drive real MoE layers on the B200 box, where the reference
is not installed. Semantics reproduced (pinned by tests/test_serving.py
against plan streams and summaries recorded from the reference,
tests/golden/plans.json):

* groups G(L) = max(1, ceil(L / target)) capped at num_layers; balanced
  contiguous layer partition, larger groups first           (scheduler.py:23-60)
* chunked: up to C new prompt tokens per iteration through all layers,
  in-flight prefills first, FCFS admission while the prompt KV fits  (:157-198)
* layered: the cohort's whole prompts through exactly one layer group per
  iteration                                                   (:204-230)
* hybrid: chunk c of every cohort member sits in group (step - c)   (:236-283)
* every iteration carries all decoding requests; a prefill's last pass
  emits the first token, each decode iteration one token      (engine.py:179-256)

The per-iteration cost is pluggable: `ModelledCost` (reference roofline,
costmodel.py) or the measured executor (executor.py), which runs the MoE
layers on the GPU and charges their device time.
"""

from __future__ import annotations

import math
from collections import deque
from dataclasses import dataclass, field

import numpy as np

from . import costmodel as cm
from .types import ModelSpec, ValidationError, require

QUEUED, PREFILLING, DECODING, FINISHED = "queued", "prefilling", "decoding", "finished"


# ---------------------------------------------------------------------------- plan types
@dataclass(frozen=True)
class PrefillAssignment:
    request_id: int
    token_start: int
    token_end: int
    layer_start: int
    layer_end: int

    @property
    def num_tokens(self) -> int:
        return self.token_end - self.token_start

    @property
    def num_layers(self) -> int:
        return self.layer_end - self.layer_start


@dataclass(frozen=True)
class BatchPlan:
    decode_ids: tuple[int, ...]
    prefill_assignments: tuple[PrefillAssignment, ...]
    designated_group: int | None = None

    @property
    def prefill_tokens(self) -> int:
        return sum(a.num_tokens for a in self.prefill_assignments)

    def layer_token_counts(self, num_layers: int) -> list[int]:
        """Routed tokens through each MoE layer: all decodes + the prefill slices covering it."""
        n = [len(self.decode_ids)] * num_layers
        for a in self.prefill_assignments:
            for layer in range(a.layer_start, a.layer_end):
                n[layer] += a.num_tokens
        return n


@dataclass
class Request:
    id: int
    arrival_s: float
    input_len: int
    output_len: int
    phase: str = QUEUED
    prefill_progress: int = 0  # tokens (chunked), next group (layered), retired chunks (hybrid)
    first_token_s: float | None = None
    token_emit_times_s: list = field(default_factory=list)
    completion_s: float | None = None

    def __post_init__(self):
        require(self.input_len >= 1, f"input_len must be >= 1, got {self.input_len}")
        require(self.output_len >= 1, f"output_len must be >= 1, got {self.output_len}")
        require(self.arrival_s >= 0, f"arrival_s must be >= 0, got {self.arrival_s}")

    @property
    def tokens_emitted(self) -> int:
        return (self.first_token_s is not None) + len(self.token_emit_times_s)

    @property
    def emit_times(self) -> list[float]:
        return [] if self.first_token_s is None else [self.first_token_s, *self.token_emit_times_s]


def num_groups(prompt_len: int, group_token_target: int, num_layers: int | None = None) -> int:
    require(prompt_len >= 1, f"prompt_len must be >= 1, got {prompt_len}")
    require(group_token_target >= 1, f"group_token_target must be >= 1, got {group_token_target}")
    g = max(1, -(-prompt_len // group_token_target))
    return g if num_layers is None else min(g, num_layers)


def layer_boundaries(num_layers: int, groups: int) -> tuple[int, ...]:
    """Contiguous partition of [0, num_layers) into min(groups, L) groups, larger first."""
    require(num_layers >= 1 and groups >= 1, "num_layers and groups must be >= 1")
    g = min(groups, num_layers)
    q, extra = divmod(num_layers, g)
    out = [0]
    for i in range(g):
        out.append(out[-1] + q + (i < extra))
    return tuple(out)


@dataclass
class Cohort:
    member_ids: tuple[int, ...]
    bounds: tuple[int, ...]
    cursor: int = 0
    chunk_size: int | None = None  # None: whole prompts per group (layered)

    @property
    def groups(self) -> int:
        return len(self.bounds) - 1

    def chunks(self, input_len: int) -> int:
        return 1 if self.chunk_size is None else -(-input_len // self.chunk_size)

    def designated(self) -> int | None:
        return None if self.groups == 1 else min(self.cursor, self.groups - 1)


# ---------------------------------------------------------------------------- planner
class Planner:
    """Pure planning over a `ServingState` plus the matching commit step."""

    def __init__(self, policy: str, chunk_size: int = 512, group_token_target: int = 512):
        require(policy in ("chunked", "layered", "hybrid"), f"unknown policy {policy!r}")
        require(chunk_size >= 1, f"chunk_size must be >= 1, got {chunk_size}")
        require(group_token_target >= 1, f"group_token_target must be >= 1, got {group_token_target}")
        self.policy, self.chunk, self.target = policy, chunk_size, group_token_target

    # ---- helpers
    @staticmethod
    def _fcfs_fit(st) -> list[Request]:
        out, room = [], st.kv_headroom()
        for r in st.waiting:
            need = r.input_len * st.model.kv_bytes_per_token
            if need > room:
                break
            room -= need
            out.append(r)
        return out

    def _new_cohort(self, st, chunk: int | None) -> Cohort | None:
        members = self._fcfs_fit(st)
        if not members:
            return None
        g = num_groups(max(r.input_len for r in members), self.target, st.model.num_layers)
        return Cohort(tuple(r.id for r in members), layer_boundaries(st.model.num_layers, g), 0, chunk)

    def _chunked_slices(self, st, gate: int | None = None) -> tuple[PrefillAssignment, ...]:
        L = st.model.num_layers
        budget, out = self.chunk, []
        for r in st.prefilling:
            if budget == 0:
                break
            n = min(budget, r.input_len - r.prefill_progress)
            if n > 0:
                out.append(PrefillAssignment(r.id, r.prefill_progress, r.prefill_progress + n, 0, L))
                budget -= n
        room = st.kv_headroom()
        for r in st.waiting:
            if budget == 0 or (gate is not None and num_groups(r.input_len, gate, L) > 1):
                break
            need = r.input_len * st.model.kv_bytes_per_token
            if need > room:
                break
            room -= need
            n = min(budget, r.input_len)
            out.append(PrefillAssignment(r.id, 0, n, 0, L))
            budget -= n
        return tuple(out)

    @staticmethod
    def _layered_slices(st, c: Cohort) -> tuple[PrefillAssignment, ...]:
        ls, le = c.bounds[c.cursor], c.bounds[c.cursor + 1]
        return tuple(PrefillAssignment(rid, 0, st.by_id[rid].input_len, ls, le) for rid in c.member_ids)

    @staticmethod
    def _hybrid_slices(st, c: Cohort) -> tuple[PrefillAssignment, ...]:
        out = []
        for ci in range(max(0, c.cursor - c.groups + 1), c.cursor + 1):
            g = c.cursor - ci
            for rid in c.member_ids:
                r = st.by_id[rid]
                if ci < c.chunks(r.input_len):
                    out.append(PrefillAssignment(rid, ci * c.chunk_size, min((ci + 1) * c.chunk_size, r.input_len),
                                                 c.bounds[g], c.bounds[g + 1]))
        return tuple(out)

    # ---- plan (scheduler.py:192-291)
    def plan(self, st) -> BatchPlan:
        dec = tuple(sorted(r.id for r in st.decoding))
        if self.policy == "chunked":
            return BatchPlan(dec, self._chunked_slices(st))
        if self.policy == "layered":
            c = st.cohort or self._new_cohort(st, None)
            if c is None:
                return BatchPlan(dec, ())
            return BatchPlan(dec, self._layered_slices(st, c), c.designated())
        c = st.cohort
        if c is None and not st.prefilling:
            fit = self._fcfs_fit(st)
            if fit and num_groups(max(r.input_len for r in fit), self.target, st.model.num_layers) > 1:
                c = self._new_cohort(st, self.chunk)
        if c is not None:
            return BatchPlan(dec, self._hybrid_slices(st, c), c.designated())
        return BatchPlan(dec, self._chunked_slices(st, gate=self.target))

    # ---- commit (scheduler.py:305-364): activation, cursor advance, completions
    def commit(self, st, plan: BatchPlan) -> list[int]:
        if not plan.prefill_assignments:
            return []
        cohort_mode = self.policy == "layered" or (
            self.policy == "hybrid" and (st.cohort is not None or plan.designated_group is not None))
        if cohort_mode and st.cohort is None:
            st.cohort = self._new_cohort(st, self.chunk if self.policy == "hybrid" else None)
            assert st.cohort is not None, "cohort plan with no formable cohort"
        seen = []
        for a in plan.prefill_assignments:
            if a.request_id not in seen:
                seen.append(a.request_id)
        for rid in seen:
            r = st.by_id[rid]
            if r.phase == QUEUED:
                st.start_prefill(r)
        done: list[int] = []
        if not cohort_mode:
            for a in plan.prefill_assignments:
                r = st.by_id[a.request_id]
                assert a.token_start == r.prefill_progress, "chunked slice must resume at the cursor"
                r.prefill_progress = a.token_end
                if r.prefill_progress == r.input_len:
                    done.append(a.request_id)
            return done
        c = st.cohort
        step = c.cursor
        c.cursor += 1
        G = c.groups
        if c.chunk_size is None:
            for rid in c.member_ids:
                st.by_id[rid].prefill_progress = c.cursor
            if c.cursor == G:
                done.extend(c.member_ids)
                st.cohort = None
            return done
        finished_all = True
        for rid in c.member_ids:
            r = st.by_id[rid]
            nc = c.chunks(r.input_len)
            if step >= G - 1:
                r.prefill_progress = min(nc, step - G + 2)
            if step == nc + G - 2:
                done.append(rid)
            elif step < nc + G - 2:
                finished_all = False
        if finished_all:
            st.cohort = None
        return done


# ---------------------------------------------------------------------------- state + engine
class ServingState:
    def __init__(self, model: ModelSpec, hw: cm.HardwareSpec, requests: list[Request], seed: int):
        self.model, self.hw = model, hw
        self.clock = 0.0
        self.pending = deque(sorted(requests, key=lambda r: (r.arrival_s, r.id)))
        self.waiting: list[Request] = []
        self.prefilling: list[Request] = []
        self.decoding: list[Request] = []
        self.finished: list[Request] = []
        self.cohort: Cohort | None = None
        self.kv_cells = 0       # (token, layer) KV cells written
        self.kv_reserved = 0    # bytes reserved for admitted prompts and emitted tokens
        self.decode_tokens = 0
        self.by_id = {r.id: r for r in requests}
        self.rng = np.random.default_rng(seed + 0x5EED)  # engine.py:309

    def kv_headroom(self) -> float:
        return self.hw.kv_capacity_bytes - self.kv_reserved

    def kv_used_bytes(self) -> float:
        return self.kv_cells * self.model.kv_bytes_per_token / self.model.num_layers

    def start_prefill(self, r: Request) -> None:
        self.waiting.remove(r)
        r.phase = PREFILLING
        self.prefilling.append(r)
        self.kv_reserved += r.input_len * self.model.kv_bytes_per_token

    def release(self, r: Request) -> None:
        held = r.input_len + r.tokens_emitted
        self.kv_cells -= held * self.model.num_layers
        self.kv_reserved -= held * self.model.kv_bytes_per_token


@dataclass
class IterationRecord:
    index: int
    start_s: float
    runtime_s: float
    expert_load_bytes: float
    moe_runtime_s: float
    decode_batch_size: int
    prefill_tokens: int
    designated_group: int | None


class ModelledCost:
    """Reference roofline for every kernel (engine.py:120-176 cost assembly)."""

    def __init__(self, coverage=None):
        self.coverage = coverage if coverage is not None else TableCoverage()

    def moe_kernels(self, st: ServingState, plan: BatchPlan) -> list[cm.Kernel]:
        m = st.model
        dec = len(plan.decode_ids)
        scopes: dict[tuple[int, int], int] = {}
        for a in plan.prefill_assignments:
            key = (a.layer_start, a.layer_end)
            scopes[key] = scopes.get(key, 0) + a.num_tokens
        out, covered = [], 0
        for (ls, le), pf in sorted(scopes.items()):
            covered += le - ls
            routed = dec + pf
            out.append(("scope", routed, le - ls, self.coverage.coverage(routed, st.rng)))
        if m.num_layers - covered > 0 and dec > 0:
            out.append(("rest", dec, m.num_layers - covered, self.coverage.coverage(dec, st.rng)))
        return out

    def iteration(self, st: ServingState, plan: BatchPlan, decode_ctx: int) -> list[cm.Kernel]:
        m = st.model
        ks = []
        for _, routed, layers, cov in self.moe_kernels(st, plan):
            ks.append(cm.moe_cost(m, routed, cov, layers))
            ks.append(cm.dense_cost(m, routed, layers))
        ks.extend(attention_kernels(m, plan, decode_ctx))
        return ks


def attention_kernels(m: ModelSpec, plan: BatchPlan, decode_ctx: int) -> list[cm.Kernel]:
    ks = [cm.attention_cost(m, a.num_tokens, a.token_start, 0, 0, a.num_layers) for a in plan.prefill_assignments]
    if plan.decode_ids:
        ks.append(cm.attention_cost(m, 0, 0, decode_ctx, len(plan.decode_ids)))
    return ks


class TableCoverage:
    def __init__(self, table=cm.DEFAULT_COVERAGE_TABLE):
        cm.check_table(table)
        self.table = table

    def coverage(self, routed_tokens: int, rng=None) -> float:
        return cm.coverage_from_table(routed_tokens, self.table)


class SimulationHorizonError(RuntimeError):
    pass


def run(model: ModelSpec, hw: cm.HardwareSpec, planner: Planner, requests: list[Request], cost=None,
        seed: int = 0, max_sim_s: float = 86_400.0) -> tuple[list[IterationRecord], list[Request], float]:
    """Serve `requests` to completion. Returns (records, finished requests by id, makespan)."""
    cost = cost if cost is not None else ModelledCost()
    reqs = [Request(r.id, r.arrival_s, r.input_len, r.output_len) for r in requests]
    for r in reqs:
        if r.input_len * model.kv_bytes_per_token > hw.kv_capacity_bytes:
            raise ValidationError(f"request {r.id}: prompt KV exceeds kv_capacity_bytes; it could never be admitted")
    st = ServingState(model, hw, reqs, seed)
    records: list[IterationRecord] = []
    while st.pending or st.waiting or st.prefilling or st.decoding:
        while st.pending and st.pending[0].arrival_s <= st.clock:
            st.waiting.append(st.pending.popleft())
        if not (st.waiting or st.prefilling or st.decoding):
            st.clock = st.pending[0].arrival_s
            continue
        plan = planner.plan(st)
        if not plan.decode_ids and not plan.prefill_assignments:
            raise AssertionError("scheduler produced an empty plan with work outstanding")
        records.append(_step(st, planner, plan, cost, len(records)))
        if st.clock > max_sim_s:
            raise SimulationHorizonError(f"simulation exceeded max_sim_s={max_sim_s}")
    return records, sorted(st.finished, key=lambda r: r.id), st.clock


def _step(st: ServingState, planner: Planner, plan: BatchPlan, cost, index: int) -> IterationRecord:
    m = st.model
    expected = tuple(sorted(r.id for r in st.decoding))
    if plan.decode_ids != expected:
        raise AssertionError(f"plan/state mismatch: decode_ids {plan.decode_ids} != decoding {expected}")
    decode_ctx = 0
    for rid in plan.decode_ids:
        r = st.by_id[rid]
        decode_ctx += r.input_len + r.tokens_emitted
    kernels = cost.iteration(st, plan, decode_ctx)
    runtime = cm.iteration_runtime(kernels, st.hw) + st.hw.iteration_overhead_s
    if runtime <= 0.0:
        raise AssertionError("planned iteration has no work")
    start = st.clock
    st.clock = now = start + runtime
    completed = planner.commit(st, plan)
    for a in plan.prefill_assignments:
        st.kv_cells += a.num_tokens * a.num_layers
    for rid in plan.decode_ids:
        r = st.by_id[rid]
        r.token_emit_times_s.append(now)
        st.kv_cells += m.num_layers
        st.kv_reserved += m.kv_bytes_per_token
        if r.tokens_emitted == r.output_len:
            r.phase, r.completion_s = FINISHED, now
            st.decoding.remove(r)
            st.release(r)
            st.finished.append(r)
    st.decode_tokens += len(plan.decode_ids)
    for rid in completed:
        r = st.by_id[rid]
        r.first_token_s = now
        st.kv_cells += m.num_layers
        st.kv_reserved += m.kv_bytes_per_token
        st.prefilling.remove(r)
        if r.tokens_emitted == r.output_len:
            r.phase, r.completion_s = FINISHED, now
            st.release(r)
            st.finished.append(r)
        else:
            r.phase = DECODING
            st.decoding.append(r)
    if st.kv_used_bytes() > st.hw.kv_capacity_bytes:
        raise ValidationError(f"KV capacity exceeded at t={now:.3f}s")
    moe_s = sum(cm.kernel_runtime(k, st.hw) for k in kernels if k.kind == cm.MOE)
    return IterationRecord(index, start, runtime, sum(k.expert_weight_bytes for k in kernels), moe_s,
                           len(plan.decode_ids), plan.prefill_tokens, plan.designated_group)


# ---------------------------------------------------------------------------- trace I/O (workload.py:14, :145-178)
TRACE_HEADER = "id,arrival_s,input_len,output_len"


def export_trace(requests: list[Request], path) -> None:
    """Write requests as the reference's trace CSV (header + one `id,arrival_s,input_len,output_len` line
    per request, arrival written with repr so it round-trips exactly; workload.py:145-150)."""
    with open(path, "w", encoding="utf-8") as f:
        f.write(TRACE_HEADER + "\n")
        for r in requests:
            f.write(f"{r.id},{r.arrival_s!r},{r.input_len},{r.output_len}\n")


def load_trace(path) -> list[Request]:
    """Read a trace CSV (reference format); errors name the offending line (workload.py:153-178)."""
    out: list[Request] = []
    with open(path, "r", encoding="utf-8") as f:
        for lineno, line in enumerate(f, start=1):
            line = line.strip()
            if not line:
                continue
            if lineno == 1 and line == TRACE_HEADER:
                continue
            parts = line.split(",")
            if len(parts) != 4:
                raise ValidationError(f"{path}: line {lineno}: expected 4 comma-separated fields, got {len(parts)}")
            try:
                out.append(Request(int(parts[0]), float(parts[1]), int(parts[2]), int(parts[3])))
            except ValueError as exc:  # ValidationError is a ValueError: field checks report the line too
                raise ValidationError(f"{path}: line {lineno}: {exc}") from exc
    return out


# ---------------------------------------------------------------------------- summary (metrics.py)
def percentile(samples: list[float], p: float) -> float:
    """Nearest rank: sorted[ceil(p/100 * n) - 1]."""
    require(len(samples) > 0, "percentile of empty sample set")
    require(0 < p <= 100, f"p must be in (0, 100], got {p}")
    s = sorted(samples)
    return s[math.ceil(p / 100.0 * len(s)) - 1]


def summarize(records: list[IterationRecord], requests: list[Request], makespan: float) -> dict:
    ttfts = [r.first_token_s - r.arrival_s for r in requests]
    tbts = [b - a for r in requests for a, b in zip(r.emit_times, r.emit_times[1:])]
    return {
        "ttft_mean_s": sum(ttfts) / len(ttfts) if ttfts else 0.0,
        "ttft_p99_s": percentile(ttfts, 99) if ttfts else 0.0,
        "tbt_mean_s": sum(tbts) / len(tbts) if tbts else 0.0,
        "tbt_p99_s": percentile(tbts, 99) if tbts else 0.0,
        "total_expert_load_bytes": sum(rec.expert_load_bytes for rec in records),
        "moe_time_s": sum(rec.moe_runtime_s for rec in records),
        "mean_decode_batch": sum(rec.decode_batch_size for rec in records) / len(records) if records else 0.0,
        "e2e_latency_mean_s": sum(r.completion_s - r.arrival_s for r in requests) / len(requests) if requests else 0.0,
        "num_requests": len(requests),
        "num_iterations": len(records),
        "makespan_s": makespan,
    }
