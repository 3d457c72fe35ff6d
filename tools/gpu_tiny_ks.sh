#!/bin/bash
# k_experts_tiny (GPT-OSS decode sizes; Qwen with LPMOE_DECODE=0) with two k-blocks per ring stage:
# parity, then A/B against the one-k-block build (paper_2510_08055_b200/_lib/liblpmoe_tinyold.so).
O=gpurun_out/tiny; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_moe.py -q -x -k "gpt_oss or tiny or decode_kernel_bit or LPMOE_DECODE=0 or LPMOE_TINY" > $O/pytest_tiny.log 2>&1
echo "pytest rc=$?" >> $O/pytest_tiny.log
OLD=$PWD/paper_2510_08055_b200/_lib/liblpmoe_tinyold.so
for rep in 1 2; do
  for T in 1 4 8; do
    timeout 300 python bench.py --shape gptoss --tokens $T --steps 30 --no-cpu-baseline 2>/dev/null | sed "s/^/new gptoss /"
    LPMOE_LIB=$OLD timeout 300 python bench.py --shape gptoss --tokens $T --steps 30 --no-cpu-baseline 2>/dev/null | sed "s/^/old gptoss /"
  done
  for T in 1 8; do
    LPMOE_DECODE=0 timeout 300 python bench.py --tokens $T --steps 30 --no-cpu-baseline 2>/dev/null | sed "s/^/new qwen-tiny /"
    LPMOE_DECODE=0 LPMOE_LIB=$OLD timeout 300 python bench.py --tokens $T --steps 30 --no-cpu-baseline 2>/dev/null | sed "s/^/old qwen-tiny /"
  done
done > $O/bench_tiny.txt
