#!/bin/bash
# Round-2 re-validation of the final tree on one B200 (outputs under gpurun_out/fin/):
# GPU suite, smoke, config-2 bench line, and measured-attention serving (pooled KV cache +
# whole-iteration decode graphs) for C3 and C5.
set -x
O=gpurun_out/fin; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench.jsonl 2>$O/bench.err
timeout 1500 python tools/serving_bench.py --config c3 --attention > $O/serving_c3_attention.jsonl 2>$O/serving_c3_attention.err
timeout 1800 python tools/serving_bench.py --config c5 --requests 100 --attention > $O/serving_c5_attention.jsonl 2>$O/serving_c5_attention.err
