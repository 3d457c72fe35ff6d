#!/bin/bash
mkdir -p gpurun_out
for T in 576 8224; do
 for v in "LPMOE_PDL=1" "LPMOE_PDL=0" "LPMOE_MAX_N=128" "LPMOE_PDL=0 LPMOE_MAX_N=128"; do
  echo "T=$T $v"; env $v timeout 300 python bench.py --tokens $T --steps 20 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['stages_us'], d['clocks']['sm_mhz'])"
 done
done > gpurun_out/variants.log 2>&1
timeout 900 python tools/serving_bench.py --config c5 --requests 40 > gpurun_out/c5.log 2>&1
