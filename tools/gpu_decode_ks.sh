#!/bin/bash
# Decode ring A/B on one B200: k-blocks per ring stage KS = 1 (11 x 18 KiB) .. 4 (2 x 72 KiB); parity first.
O=gpurun_out/ks2; mkdir -p $O
for KS in 3 4; do
  LPMOE_DECODE_KS=$KS timeout 600 python -m pytest tests/test_gpu_moe.py -q -x -k "decode_kernel" > $O/pytest_ks$KS.log 2>&1
  echo "pytest rc=$?" >> $O/pytest_ks$KS.log
done
for rep in 1 2; do
  for T in 1 2 4 8 16; do
    for KS in 2 3 4; do
      LPMOE_DECODE_KS=$KS timeout 300 python bench.py --tokens $T --steps 30 --no-cpu-baseline 2>/dev/null | sed "s/^/KS=$KS /"
    done
  done
done > $O/bench_ks.txt
