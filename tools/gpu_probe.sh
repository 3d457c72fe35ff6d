#!/bin/bash
# Probes on one B200: per-SM TMA streaming with the host launch latency kept out of the events
# (SPIN=1), and %globaltimer phase timelines of the large-batch layer (router phases).
set -x
O=gpurun_out/probe; mkdir -p $O
SPIN=1 timeout 300 ./tools/sm_stream_bench > $O/sm_stream_spin.txt 2>&1
timeout 300 ./tools/sm_stream_bench > $O/sm_stream_nospin.txt 2>&1
for T in 2048 8224; do LP_T=$T timeout 200 python tools/trace_layer.py > $O/trace_T$T.txt 2>&1; done
timeout 600 python -m pytest tests/test_gpu_executor.py -q -x > $O/pytest_executor.log 2>&1
timeout 2400 python tools/serving_bench.py --config c5 --requests 100 --attention > $O/serving_c5_attention.jsonl 2>$O/serving_c5_attention.err
