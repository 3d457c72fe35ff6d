#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
LP_T=8224 LP_ITERS=8 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_8224.csv python tools/prof_layer.py > gpurun_out/ncu_8224.log 2>&1
timeout 900 python tools/serving_bench.py --config c3 > gpurun_out/c3.log 2>&1
timeout 900 python tools/serving_bench.py --config c4 > gpurun_out/c4.log 2>&1
