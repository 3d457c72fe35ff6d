#!/bin/bash
O=gpurun_out/ge; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_moe.py -q -x -k "graphed_host or host_pipeline or cuda_graph" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for T in 1 2 4 8 16 64 576; do timeout 300 python bench.py --tokens $T --steps 30 --no-cpu-baseline; done > $O/bench.jsonl 2>$O/bench.err
