#!/bin/bash
# Large-tile router with 16 gating warps (one top-k round for 64 tokens) vs 10: parity, A/B, trace.
O=gpurun_out/rab2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_moe.py -q -x -k "qwen_layer or batch_invariance or size_sweep or back_to_back or skewed or compute_bound or experimental" > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
OLD=$PWD/paper_2510_08055_b200/_lib/liblpmoe_old.so
for rep in 1 2; do for T in 4100 8224; do
  timeout 300 python bench.py --tokens $T --steps 30 --no-cpu-baseline 2>/dev/null | sed "s/^/new /"
  LPMOE_LIB=$OLD timeout 300 python bench.py --tokens $T --steps 30 --no-cpu-baseline 2>/dev/null | sed "s/^/old /"
done; done > $O/bench.txt
