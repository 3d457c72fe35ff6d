#!/bin/bash
# round-2 first GPU call: tests, smoke, bench lines at the decode / headline / compute-bound sizes
set -x
O=gpurun_out/r02a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench.jsonl 2>$O/bench.err
for T in 1 8 32 2048 8224; do timeout 300 python bench.py --tokens $T --steps 30 --no-cpu-baseline; done > $O/bench_sweep.jsonl 2>$O/bench_sweep.err
timeout 300 python tools/host_overhead.py > $O/host_overhead.txt 2>&1
