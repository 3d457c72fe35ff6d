#!/bin/bash
# bench variants: gpu_var.sh "T1 T2" "ENV1" "ENV2" ...
Ts=$1; shift
for T in $Ts; do
 for v in "$@"; do
  echo "T=$T $v"; env $v timeout 300 python bench.py --tokens $T --steps 20 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['value'],1), {k: round(v,1) for k,v in d['stages_us'].items()}, d['clocks']['sm_mhz'])"
 done
done
