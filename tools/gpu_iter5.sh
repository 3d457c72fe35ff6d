#!/bin/bash
set -x
O=gpurun_out/$1; mkdir -p $O
for w in 1 0; do for d in 1 0; do LPMOE_DECODE_W2_WARM=$w LPMOE_DECODE_DNC=$d LP_TINY_ITEMS=1 LP_T=1 timeout 120 python tools/trace_layer.py > $O/trace_T1_dnc${d}_warm$w.txt 2>&1; done; done
for w in 1 0; do for d in 1 0; do LPMOE_DECODE_W2_WARM=$w LPMOE_DECODE_DNC=$d timeout 120 python bench.py --tokens 1 --steps 30 --no-cpu-baseline; done; done > $O/bench_decode.jsonl 2> $O/bench_decode.err
