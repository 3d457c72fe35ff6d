#!/bin/bash
# Serving runs (MoE measured, attention/dense modelled) on the final tree: C3, C4, C5.
O=gpurun_out/serv; mkdir -p $O
for c in c3 c4 c5; do timeout 1200 python tools/serving_bench.py --config $c > $O/serving_$c.jsonl 2>$O/serving_$c.err; done
