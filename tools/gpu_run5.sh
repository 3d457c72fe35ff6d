#!/bin/bash
mkdir -p gpurun_out
for T in 8224 576; do
 for v in "LPMOE_PDL=1" "LPMOE_WEVICT_FIRST=0" "LPMOE_LOOKAHEAD=4" "LPMOE_LOOKAHEAD=8" "LPMOE_LOOKAHEAD=8 LPMOE_WEVICT_FIRST=0" "LPMOE_MAX_N=128 LPMOE_LOOKAHEAD=8"; do
  echo "T=$T $v"; env $v timeout 300 python bench.py --tokens $T --steps 20 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['stages_us'], d['clocks']['sm_mhz'])"
 done
done > gpurun_out/variants2.log 2>&1
