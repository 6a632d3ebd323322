#!/bin/bash
# round-2 job: distributed-mode parity over NCCL (ranks share cuda:0), shared-GPU N=2 bench, N=1 bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/r2a_smi.txt
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q -s > gpurun_out/r2a_dist.log 2>&1; echo "dist rc=$?" >> gpurun_out/r2a_dist.log
PST_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_bench_n2_shared.log 2>&1; echo "rc=$?" >> gpurun_out/r2a_bench_n2_shared.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2a_bench_n1.log 2>&1; echo "rc=$?" >> gpurun_out/r2a_bench_n1.log
tail -3 gpurun_out/r2a_dist.log gpurun_out/r2a_bench_n2_shared.log gpurun_out/r2a_bench_n1.log
