#!/bin/bash
# decode-size layers: parity tests, bench lines T=1..16, one item-level trace at T=1
O=gpurun_out/$1; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_moe.py -x -q -k "decode or tiny_config or qwen_layer or launch_count or batch_invariance" > $O/pytest_decode.log 2>&1
for T in 1 2 3 4 8 16; do timeout 120 python bench.py --tokens $T --steps 40 --no-cpu-baseline; done > $O/bench_decode.jsonl 2> $O/bench_decode.err
LP_TINY_ITEMS=1 LP_T=1 timeout 120 python tools/trace_layer.py > $O/trace_T1.txt 2>&1
