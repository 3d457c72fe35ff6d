#!/bin/bash
# C5 (100-request arXiv trace) with measured attention + dense + MoE, pooled KV sized by memory.
O=gpurun_out/c5att; mkdir -p $O
timeout 3000 python tools/serving_bench.py --config c5 --requests 100 --attention > $O/serving_c5_attention.jsonl 2>$O/serving_c5_attention.err
echo "rc=$?" >> $O/serving_c5_attention.err
