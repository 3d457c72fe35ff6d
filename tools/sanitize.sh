#!/bin/bash
# compute-sanitizer passes over the layer paths (memory-bound gather kernel, CTA-pair kernel,
# staged API) and the executor glue; outputs under gpurun_out/san/.
O=gpurun_out/san; mkdir -p $O
for tool in memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/san_driver.py 1 2 8 64 576 2048 \
    > $O/$tool.log 2>&1; echo "$tool rc=$?" >> $O/summary.txt
  tail -3 $O/$tool.log >> $O/summary.txt
done
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/san_driver.py 1 2 8 64 576 2048 \
  > $O/racecheck.log 2>&1; echo "racecheck rc=$?" >> $O/summary.txt; tail -3 $O/racecheck.log >> $O/summary.txt
cat $O/summary.txt
