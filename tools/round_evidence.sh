#!/bin/bash
# Round evidence on one B200: tests, bench lines, ncu launch list + full capture, serving runs.
# Outputs under gpurun_out/ev/.
set -x
O=gpurun_out/ev; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench.jsonl 2>$O/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_ref.jsonl 2>$O/bench_ref.err
for T in 64 2048 8224; do timeout 300 python bench.py --tokens $T --steps 30 --no-cpu-baseline; done > $O/bench_sweep.jsonl 2>$O/bench_sweep.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline > $O/ncu_bench.log 2>&1
LP_T=576 LP_ITERS=6 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_experts -s 2 -c 1 -o $O/k_experts_576 python tools/prof_layer.py > $O/ncu_full.log 2>&1
LP_T=8224 LP_ITERS=4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_experts -s 2 -c 1 -o $O/k_experts_8224 python tools/prof_layer.py >> $O/ncu_full.log 2>&1
[ -f paper_2510_08055_b200/_lib/liblpmoe_trace.so ] || python -m paper_2510_08055_b200.build --trace > /dev/null 2>&1
LP_T=576 timeout 300 python tools/trace_layer.py > $O/trace_T576.txt 2>&1
timeout 1200 python tools/serving_bench.py --config c3 > $O/serving_c3.jsonl 2>$O/serving_c3.err
timeout 1200 python tools/serving_bench.py --config c4 > $O/serving_c4.jsonl 2>$O/serving_c4.err
timeout 1800 python tools/serving_bench.py --config c5 --requests 100 > $O/serving_c5.jsonl 2>$O/serving_c5.err
