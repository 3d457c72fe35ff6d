#!/bin/bash
# Decode ring A/B on one B200: KS=2 (5 x 36 KiB stages, default) vs KS=1 (11 x 18 KiB), parity first.
O=gpurun_out/ks; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_moe.py -q -x -k "decode or experimental or size_sweep or graph" > $O/pytest_decode.log 2>&1
echo "pytest rc=$?" >> $O/pytest_decode.log
for rep in 1 2; do
  for T in 1 2 4 8 16; do
    for KS in 2 1; do
      LPMOE_DECODE_KS=$KS timeout 300 python bench.py --tokens $T --steps 30 --no-cpu-baseline 2>/dev/null | sed "s/^/KS=$KS /"
    done
  done
done > $O/bench_ks.txt
