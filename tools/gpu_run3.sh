#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
LP_T=8224 LP_ITERS=4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_experts -s 2 -c 1 -o gpurun_out/prof_experts_8224 python tools/prof_layer.py > gpurun_out/ncu_full_8224.log 2>&1
LP_T=8224 LP_ITERS=4 timeout 600 ncu --set full --clock-control none -k regex:"k_router|k_scan|k_scatter|k_combine" -s 4 -c 4 -o gpurun_out/prof_small_8224 python tools/prof_layer.py > gpurun_out/ncu_small_8224.log 2>&1
