#!/bin/bash
# per-kernel device time (cold-cache, serialised) of a few layer forwards at T tokens
T=${1:-576}
LP_T=$T LP_ITERS=6 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"lp::|k_" --csv python tools/prof_layer.py 2>/dev/null | grep -v "^==" > gpurun_out/launches_$T.csv
