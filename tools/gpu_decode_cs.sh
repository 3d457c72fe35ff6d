#!/bin/bash
# decode kernel cluster size A/B (routing partials per CTA vs SMs streaming)
O=gpurun_out/$1; mkdir -p $O
for cs in 4 2; do for T in 1 2 3 4; do LPMOE_DECODE_CS=$cs timeout 120 python bench.py --tokens $T --steps 40 --no-cpu-baseline; done; done > $O/bench_cs.jsonl 2> $O/bench_cs.err
