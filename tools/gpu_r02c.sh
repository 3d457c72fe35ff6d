#!/bin/bash
# round-2 evidence after the EP protocol / decode changes: full GPU suite, bench sweep, shared-GPU
# EP protocol runs (bench + serving), measured serving C3/C4/C5
set -x
O=gpurun_out/r02c; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench.jsonl 2>$O/bench.err
for T in 1 2 4 8 16 32 64 2048 8224; do timeout 300 python bench.py --tokens $T --steps 30 --no-cpu-baseline; done > $O/bench_sweep.jsonl 2>$O/bench_sweep.err
LPMOE_BENCH_SHARED_GPU=1 timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_ep2_shared.jsonl 2>$O/bench_ep2_shared.err
LPMOE_BENCH_SHARED_GPU=1 timeout 1200 python tools/serving_bench.py --config c5 --gpus 2 --requests 4 > $O/serving_c5_ep2_shared.jsonl 2>$O/serving_c5_ep2_shared.err
timeout 1200 python tools/serving_bench.py --config c3 > $O/serving_c3.jsonl 2>$O/serving_c3.err
timeout 1200 python tools/serving_bench.py --config c4 > $O/serving_c4.jsonl 2>$O/serving_c4.err
timeout 2400 python tools/serving_bench.py --config c5 --requests 100 > $O/serving_c5.jsonl 2>$O/serving_c5.err
