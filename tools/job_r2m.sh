#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2m
rm -f gpurun_out/parity_margins.jsonl
timeout 2400 python -m pytest tests/test_gpu_fsbks.py tests/test_gpu_configs.py -q -rA -k "fsbks or 100_steps" --durations=10 > gpurun_out/r2m/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2m/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2m/bench_n1.log 2>&1
tail -25 gpurun_out/r2m/pytest.log; tail -c 800 gpurun_out/r2m/bench_n1.log
