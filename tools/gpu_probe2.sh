#!/bin/bash
# Decode-regime streaming probe on one B200: plain TMA ring vs the same ring consumed by
# decode-item MMAs (tools/sm_stream_bench.cu MMA_AB), and the T=1 decode item timeline.
set -x
O=gpurun_out/probe2; mkdir -p $O
SPIN=1 MMA_AB=1 timeout 300 ./tools/sm_stream_bench > $O/sm_stream_mma.txt 2>&1
LP_TINY_ITEMS=1 LP_T=1 timeout 200 python tools/trace_layer.py > $O/trace_decode_T1.txt 2>&1
