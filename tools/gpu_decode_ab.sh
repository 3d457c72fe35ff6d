#!/bin/bash
set -x
O=gpurun_out/$1; mkdir -p $O
for g in 1 0; do for d in 1 0; do LPMOE_DECODE_ACT_GATHER=$g LPMOE_DECODE_W2_WARM=0 LPMOE_DECODE_DNC=$d LP_TINY_ITEMS=1 LP_T=1 timeout 120 python tools/trace_layer.py > $O/trace_T1_dnc${d}_g$g.txt 2>&1; done; done
for g in 1 0; do for d in 1 0; do for T in 1 2 8; do LPMOE_DECODE_ACT_GATHER=$g LPMOE_DECODE_W2_WARM=0 LPMOE_DECODE_DNC=$d timeout 120 python bench.py --tokens $T --steps 30 --no-cpu-baseline; done; done; done > $O/bench_decode.jsonl 2> $O/bench_decode.err
timeout 600 python -m pytest tests/test_gpu_moe.py -x -q -k "decode" > $O/pytest_decode.log 2>&1
