#!/bin/bash
# tensor-pipe utilisation of k_experts at T tokens (clock-independent ratio)
T=${1:-8224}
LP_T=$T LP_ITERS=6 timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex.sum.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_experts -s 2 -c 3 --csv python tools/prof_layer.py 2>/dev/null | grep -v "^==" 
