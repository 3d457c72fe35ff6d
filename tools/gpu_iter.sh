#!/bin/bash
# quick GPU iteration: decode + EP tests, decode bench lines, decode traces. Usage: tools/gpu_iter.sh TAG
set -x
O=gpurun_out/$1; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_moe.py -x -q -k "decode or qwen_layer or tiny_config or launch_count or batch_invariance or graph" > $O/pytest_decode.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ep_p2p.py tests/test_gpu_ep.py -x -q > $O/pytest_ep.log 2>&1
for T in 1 2 4 8 16; do timeout 120 python bench.py --tokens $T --steps 30 --no-cpu-baseline; done > $O/bench_decode.jsonl 2> $O/bench_decode.err
for T in 1 2 8; do LP_T=$T timeout 120 python tools/trace_layer.py > $O/trace_T$T.txt 2>&1; done
