#!/bin/bash
O=gpurun_out/tiny; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_moe.py -q -x -k "gpt_oss or tiny_config or decode_kernel_bit or experimental_paths_match_oracle or size_sweep" > $O/pytest_tiny.log 2>&1
echo "pytest rc=$?" >> $O/pytest_tiny.log
