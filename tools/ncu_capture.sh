#!/bin/bash
# Run on the GPU box: launch list (time + DRAM bytes per launch) and full captures of the hot
# conv kernels.  Eager launches (PST_GRAPHS=0): ncu's per-kernel replay of graph nodes fails for
# the wgrad kernel.  Numbers printed by bench under ncu are never bench values.
OUT=${1:-gpurun_out}
mkdir -p $OUT
export PST_GRAPHS=0
BENCH="python bench.py --steps 1 --warmup 1 --profile-steps 0 --no-e2e --no-cpu-baseline"
# launch list: the --clock-control none duration pass of B200_PROFILING.md
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches.csv \
  $BENCH > $OUT/ncu_launch_bench.log 2>&1
# DRAM traffic of every launch of the same command (per-class bytes per launch -> profiles/traffic.json)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 3000 --csv --log-file $OUT/traffic.csv $BENCH > $OUT/ncu_traffic_bench.log 2>&1
# one full capture each of a mid-network forward conv, dgrad conv and wgrad (ResNet-110, stage 2 convs)
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:conv_fwd_kernel<\(bool\)0, \(bool\)0>' -s 150 -c 1 \
  -o $OUT/prof_fwd $BENCH > $OUT/ncu_fwd.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:conv_fwd_kernel<\(bool\)0, \(bool\)1>' -s 150 -c 1 \
  -o $OUT/prof_dgrad $BENCH > $OUT/ncu_dgrad.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_wgrad -s 100 -c 1 \
  -o $OUT/prof_wgrad $BENCH > $OUT/ncu_wgrad.log 2>&1
ls -la $OUT
