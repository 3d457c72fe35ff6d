#!/bin/bash
# compute-sanitizer over the two-k-block decode ring (T = 1..16: 4-CTA and pair routing clusters,
# block-diagonal and per-expert DN items), plus an ncu --set full capture of the pair kernel at T=2048.
O=gpurun_out/san2; mkdir -p $O
for tool in memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/san_driver.py 1 2 3 4 8 16 \
    > $O/$tool.log 2>&1; echo "$tool rc=$?" >> $O/summary.txt
  tail -3 $O/$tool.log >> $O/summary.txt
done
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/san_driver.py 1 8 16 \
  > $O/racecheck.log 2>&1; echo "racecheck rc=$?" >> $O/summary.txt; tail -3 $O/racecheck.log >> $O/summary.txt
LP_T=2048 LP_ITERS=6 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_experts -s 2 -c 1 -o $O/k_experts_2048 python tools/prof_layer.py > $O/ncu_2048.log 2>&1
cat $O/summary.txt
