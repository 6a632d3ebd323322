#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2t
rm -f gpurun_out/parity_margins.jsonl
timeout 1200 python -m pytest tests/test_gpu_dist.py -q -rA > gpurun_out/r2t/dist.log 2>&1; echo "rc=$?" >> gpurun_out/r2t/dist.log
PST_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2t/bench_n2_shared.json 2> gpurun_out/r2t/bench.err
timeout 1500 python -m pytest tests/test_gpu_configs.py -q -rA -k segments_100 > gpurun_out/r2t/seg.log 2>&1; echo "rc=$?" >> gpurun_out/r2t/seg.log
cp gpurun_out/parity_margins.jsonl gpurun_out/r2t/
tail -5 gpurun_out/r2t/dist.log; tail -4 gpurun_out/r2t/seg.log; tail -c 300 gpurun_out/r2t/bench_n2_shared.json
