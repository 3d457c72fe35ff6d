#!/bin/bash
# Router TMEM drain with all partials in flight (CS=1 tiles, T >= 2048): parity, then A/B against the
# previous build (paper_2510_08055_b200/_lib/liblpmoe_old.so) and phase traces.
O=gpurun_out/rab; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_moe.py -q -x -k "qwen_layer or batch_invariance or size_sweep or back_to_back or skewed" > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
OLD=$PWD/paper_2510_08055_b200/_lib/liblpmoe_old.so
for rep in 1 2; do for T in 2048 8224; do
  timeout 300 python bench.py --tokens $T --steps 30 --no-cpu-baseline 2>/dev/null | sed "s/^/new /"
  LPMOE_LIB=$OLD timeout 300 python bench.py --tokens $T --steps 30 --no-cpu-baseline 2>/dev/null | sed "s/^/old /"
done; done > $O/bench.txt
for T in 2048 8224; do LP_T=$T timeout 200 python tools/trace_layer.py > $O/trace_T$T.txt 2>&1; done
