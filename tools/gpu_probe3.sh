#!/bin/bash
O=gpurun_out/probe3; mkdir -p $O
SPIN=1 MMA_AB=1 SK_ONLY=1 timeout 300 ./tools/sm_stream_bench > $O/sm_stream_stage_size.txt 2>&1
