#!/bin/bash
# Run on the GPU box: launch list + full captures of the hot conv kernels (eager launches:
# PST_GRAPHS=0, since ncu's per-kernel replay of graph nodes fails for the wgrad kernel).
OUT=${1:-gpurun_out}
mkdir -p $OUT
export PST_GRAPHS=0
BENCH="python bench.py --steps 2 --warmup 1 --profile-steps 0 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches.csv $BENCH > $OUT/ncu_launch_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_fwd -s 12 -c 1 -o $OUT/prof_fwd $BENCH > $OUT/ncu_fwd.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_wgrad -s 100 -c 1 -o $OUT/prof_wgrad $BENCH > $OUT/ncu_wgrad.log 2>&1
ls -la $OUT
