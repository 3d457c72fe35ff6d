#!/bin/bash
# one gpurun call: build check, gpu tests, smoke, bench, token sweep, serving c3
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
for T in 32 2048 4608 8224; do timeout 300 python bench.py --tokens $T --steps 20 --no-cpu-baseline; done > gpurun_out/sweep.log 2>&1
timeout 1200 python tools/serving_bench.py --config c3 > gpurun_out/c3.log 2>&1
