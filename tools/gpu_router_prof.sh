#!/bin/bash
# ncu --set full of the large-tile router (T=8224: 64-token tiles, CS=1) with source for the hot-line view.
O=gpurun_out/rprof; mkdir -p $O
LP_T=8224 LP_ITERS=4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_router -s 2 -c 1 -o $O/k_router_8224 python tools/prof_layer.py > $O/ncu.log 2>&1
LP_T=2048 LP_ITERS=4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_router -s 2 -c 1 -o $O/k_router_2048 python tools/prof_layer.py >> $O/ncu.log 2>&1
