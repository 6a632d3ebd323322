#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2o
timeout 120 python tools/conv_lab.py 50 > gpurun_out/r2o/conv_lab_default.txt 2>&1
export PST_LIB=exp
for cfg in "PST_WT_SETS3_ROWS=256" "PST_WT_SETS3_ROWS=320" "PST_WT_SETS3_ROWS=640" "PST_WT_SETS=2"; do
  env $cfg LAB_TAG="$cfg" timeout 120 python tools/conv_lab.py 50 >> gpurun_out/r2o/wgrad_knobs.txt 2>&1
done
unset PST_LIB
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2o/bench_n1.log 2>&1
cat gpurun_out/r2o/conv_lab_default.txt gpurun_out/r2o/wgrad_knobs.txt; grep -o '"value": [0-9.]*' gpurun_out/r2o/bench_n1.log | head -2
