#!/bin/bash
# A/B bench with interleaved repeats: gpu_ab.sh "T1 T2" REPS "ENV_A" "ENV_B" ...
Ts=$1; shift; R=$1; shift
for T in $Ts; do
 for rep in $(seq $R); do
  for v in "$@"; do
   echo -n "T=$T [$v] "; env $v timeout 120 python bench.py --tokens $T --steps 40 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['value'],1), round(d['e2e']['value'],1), {k: round(v,1) for k,v in d['stages_us'].items()}, d['clocks']['sm_mhz'])"
  done
 done
done
