#!/bin/bash
set -x
O=gpurun_out/$1; mkdir -p $O
timeout 400 python -m pytest tests/test_gpu_ep_p2p.py -x -q -k "skewed" > $O/pytest_ep.log 2>&1
for d in 1 0; do for T in 1 2; do LPMOE_DECODE_DNC=$d timeout 120 python bench.py --tokens $T --steps 30 --no-cpu-baseline; done; done > $O/bench_decode.jsonl 2> $O/bench_decode.err
for d in 1 0; do for T in 1 2; do LPMOE_DECODE_DNC=$d LP_TINY_ITEMS=1 LP_T=$T timeout 120 python tools/trace_layer.py > $O/trace_T${T}_dnc$d.txt 2>&1; done; done
