#!/bin/bash
# quick check: GPU tests + bench at a few T (args: token counts)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for T in "$@"; do
  echo "T=$T"; timeout 300 python bench.py --tokens $T --steps 20 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['value'],1), {k: round(v,1) for k,v in d['stages_us'].items()}, d['clocks']['sm_mhz'])"
done
