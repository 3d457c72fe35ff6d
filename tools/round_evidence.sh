#!/bin/bash
# Round evidence on one B200 (outputs under gpurun_out/ev/, summaries copied into profiles/rNN/ by hand):
# full GPU suite, smoke, bench lines (config 2 + size sweep), the reference arm, ncu launch list of the
# config-2 bench, ncu --set full of the expert kernel (T=576, 8224) and of the decode kernel (T=1).
set -x
O=gpurun_out/ev; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench.jsonl 2>$O/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_ref.jsonl 2>$O/bench_ref.err
for T in 1 2 4 8 16 32 64 2048 8224; do timeout 300 python bench.py --tokens $T --steps 30 --no-cpu-baseline; done > $O/bench_sweep.jsonl 2>$O/bench_sweep.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline > $O/ncu_bench.log 2>&1
LP_T=1 LP_ITERS=6 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_decode -s 2 -c 1 -o $O/k_decode_1 python tools/prof_layer.py > $O/ncu_full.log 2>&1
LP_T=576 LP_ITERS=6 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_experts -s 2 -c 1 -o $O/k_experts_576 python tools/prof_layer.py >> $O/ncu_full.log 2>&1
LP_T=8224 LP_ITERS=4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_experts -s 2 -c 1 -o $O/k_experts_8224 python tools/prof_layer.py >> $O/ncu_full.log 2>&1
LP_TINY_ITEMS=1 LP_T=1 timeout 120 python tools/trace_layer.py > $O/trace_decode_T1.txt 2>&1
LP_T=576 timeout 120 python tools/trace_layer.py > $O/trace_T576.txt 2>&1
timeout 600 python tools/ep_overhead.py 1 64 576 2048 > $O/ep_overhead_world1.jsonl 2>$O/ep_overhead.err
timeout 1500 python tools/serving_bench.py --config c3 > $O/serving_c3.jsonl 2>$O/serving_c3.err
timeout 1500 python tools/serving_bench.py --config c4 > $O/serving_c4.jsonl 2>$O/serving_c4.err
timeout 2400 python tools/serving_bench.py --config c5 --requests 100 > $O/serving_c5.jsonl 2>$O/serving_c5.err
timeout 2000 python tools/serving_bench.py --config c4 --attention > $O/serving_c4_attention.jsonl 2>$O/serving_c4_attention.err
