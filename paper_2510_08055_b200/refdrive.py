"""The reference simulator drives the B200 MoE layer.

The reference (`moesim`) is run UNMODIFIED: its engine (`engine.run` ->
`scheduler.plan_for` -> `engine.step` -> `_iteration_kernels`, engine.py:120-256,
:272-351) plans every iteration and keeps the clock, KV and token bookkeeping;
its chunk bench (`cli.chunk_bench_rows`, cli.py:211-243) sweeps chunk sizes.
The GPU enters only at the call sites SURVEY §8(b) names:

* **coverage** — any object with `.coverage(routed_tokens, rng) -> float` is a
  `CoverageModel` (coverage.py:216-254); `coverage.MeasuredCoverage` routes
  real tokens through a `GpuMoE` layer and returns nnz(counts)/E (engine.py:147,
  :152; cli.py:222).
* **MoE cost** — the names `moe_cost`, `kernel_runtime` and
  `iteration_runtime` (costmodel.py:57, :148-157) that engine.py:148/:153/:197
  and cli.py:223-227 look up in their own module globals. `measured_costs()`
  rebinds those names for the duration of a with-block (and restores them):
  a MoE kernel then carries its measured device seconds (`measured_s`) and the
  runtime sum charges them instead of the roofline; every other kernel keeps
  the reference's roofline formula. Bytes and flops stay the reference's
  formulas with the measured coverage, so `IterationRecord.expert_load_bytes`
  (engine.py:251) is Σ nnz·bytes_per_expert of what the GPU really loaded.
* **the whole MoE stack** — with `executor=` (executor.LayeredExecutor), the
  engine's `_iteration_kernels` is wrapped: the iteration's BatchPlan
  (scheduler.py:82-92) runs through the resident layer stack on the GPU
  (decode tokens through every layer, each prefill slice through its layer
  range), and its measured MoE kernel replaces the modelled ones; dense and
  attention kernels stay the reference's modelled costs (out of scope).

A maintainer adding this to the reference would pass a `cost_hook` into
`engine.step` / `chunk_bench_rows` instead (INTEGRATION.md shows the 6-line
patch); rebinding the module names gives the same effect without editing the
read-only reference. Like the reference, one run is
single-threaded: do not run two measured runs concurrently in one process.
"""

from __future__ import annotations

import contextlib
import dataclasses
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# where tools/vendor_reference.sh installs the reference (git-ignored, travels to the GPU box)
VENDORED = os.path.join(ROOT, "baseline", "_ref")
SOURCE_TREE = "/root/reference/pkg/src"  # the read-only upstream checkout (build container only)


class ReferenceMissing(ImportError):
    pass


def import_moesim():
    """Import the unmodified reference package: already importable, else the vendored copy under
    baseline/_ref, else the upstream source tree. Raises ReferenceMissing if none exists."""
    try:
        import moesim  # noqa: F401
    except ImportError:
        for p in (VENDORED, SOURCE_TREE):
            if os.path.isdir(os.path.join(p, "moesim")):
                sys.path.insert(0, p)
                break
        else:
            raise ReferenceMissing("moesim (the reference) is not importable: run tools/vendor_reference.sh "
                                   "to install it under baseline/_ref") from None
    import moesim
    import moesim.cli
    import moesim.costmodel
    import moesim.engine

    return moesim


def reference_available() -> bool:
    try:
        import_moesim()
        return True
    except ReferenceMissing:
        return False


_MEASURED_CLS = {}


def measured_kernel_cls():
    """`KernelCost` (costmodel.py:21-36) plus the device seconds the kernel measured."""
    ms = import_moesim()
    cls = _MEASURED_CLS.get(id(ms.costmodel.KernelCost))
    if cls is None:
        cls = dataclasses.make_dataclass("MeasuredKernelCost", [("measured_s", float, dataclasses.field(default=0.0))],
                                         bases=(ms.costmodel.KernelCost,), frozen=True)
        cls.__doc__ = "A KernelCost that was run on the GPU: runtime = measured_s, not the roofline."
        _MEASURED_CLS[id(ms.costmodel.KernelCost)] = cls
    return cls


def measured_moe_kernel(model, routed_per_layer, experts_hit_per_layer, device_s: float):
    """The MoE kernel of one iteration as moe_cost (costmodel.py:57-85) would state it, with the
    coverage the routing really produced: expert bytes = Σ_layers nnz·bytes_per_expert,
    activations 2·T·H·dtype per layer, flops T·k·flops_per_token_per_expert per layer."""
    ms = import_moesim()
    expert = float(sum(experts_hit_per_layer) * model.bytes_per_expert)
    act = float(sum(2.0 * n * model.hidden_dim * model.dtype_bytes for n in routed_per_layer))
    flops = float(sum(n * model.top_k * model.flops_per_token_per_expert for n in routed_per_layer))
    return measured_kernel_cls()(kind=ms.costmodel.KernelKind.MOE_FFN, flops=flops, hbm_bytes=expert + act,
                                 expert_weight_bytes=expert, measured_s=float(device_s))


@contextlib.contextmanager
def measured_costs(coverage=None, executor=None):
    """Bind the measured-cost adapter at the reference's MoE call sites for one with-block.

    coverage: a `MeasuredCoverage`; MoE kernels that engine.py / cli.py cost right after a
              coverage call on the same routed-token count are charged that call's device time
              x layers_in_scope (the same batch runs through each layer in scope).
    executor: a `LayeredExecutor` (or any object with `run_plan(state, plan) -> MoEIteration`);
              the engine's iteration MoE work runs through it (whole plan, real hidden states).
    """
    ms = import_moesim()
    eng, cli, cmod = ms.engine, ms.cli, ms.costmodel
    MK = measured_kernel_cls()
    saved = {(eng, "iteration_runtime"): eng.iteration_runtime, (eng, "moe_cost"): eng.moe_cost,
             (eng, "_iteration_kernels"): eng._iteration_kernels,
             (cli, "kernel_runtime"): cli.kernel_runtime, (cli, "moe_cost"): cli.moe_cost}
    base_runtime, base_moe, base_iter = cmod.kernel_runtime, cmod.moe_cost, eng._iteration_kernels

    def kernel_runtime(kernel, hw):
        return kernel.measured_s if isinstance(kernel, MK) else base_runtime(kernel, hw)

    def iteration_runtime(kernels, hw):
        return sum(kernel_runtime(k, hw) for k in kernels)

    def moe_cost(model, routed_tokens, coverage_fraction, layers_in_scope=None):
        layers = model.num_layers if layers_in_scope is None else layers_in_scope
        k = base_moe(model, routed_tokens, coverage_fraction, layers)
        if coverage is not None and getattr(coverage, "last_routed", None) == routed_tokens:
            return MK(kind=k.kind, flops=k.flops, hbm_bytes=k.hbm_bytes, expert_weight_bytes=k.expert_weight_bytes,
                      measured_s=coverage.last_device_s * layers)
        return k

    def iteration_kernels(state, plan, coverage_model):
        kernels, decode_ctx = base_iter(state, plan, coverage_model)
        it = executor.run_plan(state, plan)
        moe = measured_moe_kernel(state.model, it.routed, it.experts_hit, it.device_s)
        rest = [k for k in kernels if k.kind != cmod.KernelKind.MOE_FFN]
        if getattr(it, "includes_attention", False):
            # attention + dense projections ran on the GPU and are inside device_s: keep their
            # modelled flops / bytes (energy, reporting) but charge no modelled time for them
            measured = (cmod.KernelKind.DENSE_PROJ, cmod.KernelKind.ATTENTION_PREFILL,
                        cmod.KernelKind.ATTENTION_DECODE)
            rest = [MK(kind=k.kind, flops=k.flops, hbm_bytes=k.hbm_bytes,
                       expert_weight_bytes=k.expert_weight_bytes, measured_s=0.0) if k.kind in measured else k
                    for k in rest]
        return [moe] + rest, decode_ctx

    eng.iteration_runtime = iteration_runtime
    cli.kernel_runtime = kernel_runtime
    if coverage is not None:
        eng.moe_cost = moe_cost
        cli.moe_cost = moe_cost
    if executor is not None:
        eng._iteration_kernels = iteration_kernels
    try:
        yield
    finally:
        for (mod, name), fn in saved.items():
            setattr(mod, name, fn)


def b200_hardware(kv_capacity_bytes: float = 100e9, iteration_overhead_s: float = 0.0):
    """The reference's HardwareSpec (types.py:75-112) with this pool's measured B200 peaks
    (MEASURED_PEAKS.json when present) for the modelled, non-MoE kernels of measured runs;
    KV budget: 180 GB minus 58 GB of resident expert weights, rounded down."""
    import json

    ms = import_moesim()
    flops, bw = 1643.2e12, 6550.7e9
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        flops, bw = d.get("bf16_tflops", 1643.2) * 1e12, d.get("hbm_gbs", 6550.7) * 1e9
    return ms.types.HardwareSpec(name="b200", peak_flops=flops, peak_hbm_bw=bw, mfu=0.6, mbu=0.8,
                                 kv_capacity_bytes=kv_capacity_bytes, iteration_overhead_s=iteration_overhead_s)


def reference_model(shape_model):
    """Our ModelSpec (types.py mirror) as the reference's ModelSpec."""
    ms = import_moesim()
    return ms.types.ModelSpec(**{f.name: getattr(shape_model, f.name) for f in dataclasses.fields(ms.types.ModelSpec)})


def reference_config(name: str) -> str:
    """Path of one of the reference's run configs (pkg/configs/<name>), vendored copy first."""
    for d in (os.path.join(VENDORED, "configs"), os.path.join(os.path.dirname(SOURCE_TREE), "configs")):
        p = os.path.join(d, name)
        if os.path.exists(p):
            return p
    raise ReferenceMissing(f"reference config {name} not found: run tools/vendor_reference.sh")
