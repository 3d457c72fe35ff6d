#!/bin/bash
# Round-2 closing evidence on one B200 (outputs under gpurun_out/fin2/): GPU suite, smoke, config-2
# bench line, reference arm, size sweep, ncu launch list of the config-2 bench, ncu --set full of the
# decode kernel (T=1, new ring) and of the expert kernel (T=576).
set -x
O=gpurun_out/fin2; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench.jsonl 2>$O/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_ref.jsonl 2>$O/bench_ref.err
for T in 1 2 4 8 16 32 64 2048 8224; do timeout 300 python bench.py --tokens $T --steps 30 --no-cpu-baseline; done > $O/bench_sweep.jsonl 2>$O/bench_sweep.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline > $O/ncu_bench.log 2>&1
LP_T=1 LP_ITERS=6 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_decode -s 2 -c 1 -o $O/k_decode_1 python tools/prof_layer.py > $O/ncu_full.log 2>&1
LP_T=576 LP_ITERS=6 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_experts -s 2 -c 1 -o $O/k_experts_576 python tools/prof_layer.py >> $O/ncu_full.log 2>&1
