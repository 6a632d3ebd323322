#!/bin/bash
# round-2 job: FFMA wgrad experiment + 1-GPU bench with the memory report + shared-GPU N=2 bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 ./tools/ffma_wgrad_bench > gpurun_out/r2d_ffma_wgrad.txt 2>&1; echo "rc=$?" >> gpurun_out/r2d_ffma_wgrad.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2d_bench_n1.log 2>&1; echo "rc=$?" >> gpurun_out/r2d_bench_n1.log
cat gpurun_out/r2d_ffma_wgrad.txt
tail -c 1500 gpurun_out/r2d_bench_n1.log
