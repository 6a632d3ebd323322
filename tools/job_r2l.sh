#!/bin/bash
# round-2: conv_lab after the wgrad converter change, tcgen05 pipe counters per conv kernel, wgrad capture
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2l
timeout 300 python tools/conv_lab.py 50 > gpurun_out/r2l/conv_lab.txt 2>&1
export PST_GRAPHS=0
M=sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32.sum,sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32.sum.peak_sustained,sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_hmma.sum,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg,gpu__time_duration.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:"conv_wgrad_ts|conv_ts_kernel" -c 9 --csv \
   python tools/conv_lab.py 1 > gpurun_out/r2l/tc_counters.csv 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_wgrad_ts -c 1 \
   -o gpurun_out/r2l/prof_wgrad_g1 python tools/conv_lab.py 1 > gpurun_out/r2l/ncu_wgrad.log 2>&1
cat gpurun_out/r2l/conv_lab.txt
