#!/bin/bash
set -x
O=gpurun_out/$1; mkdir -p $O
for d in 1 0; do for T in 1 1 2; do LPMOE_DECODE_DNC=$d timeout 120 python bench.py --tokens $T --steps 30 --no-cpu-baseline; done; done > $O/bench_decode.jsonl 2> $O/bench_decode.err
for d in 1; do for T in 1; do LPMOE_DECODE_DNC=$d LP_TINY_ITEMS=1 LP_T=$T timeout 120 python tools/trace_layer.py > $O/trace_T${T}_dnc$d.txt 2>&1; done; done
timeout 900 python -m pytest tests/test_gpu_ep_p2p.py tests/test_gpu_ep_executor.py tests/test_gpu_executor.py -x -q > $O/pytest_ep.log 2>&1
timeout 600 python -m pytest tests/test_gpu_moe.py -x -q -k "decode" > $O/pytest_decode.log 2>&1
