#!/bin/bash
O=gpurun_out/dc; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_moe.py -q -x -k "decode or graphed_host or size_sweep or experimental" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for T in 1 2 4 8 16; do timeout 300 python bench.py --tokens $T --steps 30 --no-cpu-baseline; done > $O/bench.jsonl 2>$O/bench.err
