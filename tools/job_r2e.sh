#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/midblock_probe.py > gpurun_out/r2e_midblock_probe.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_dist.py -q -k "midblock or tiny_resnet" > gpurun_out/r2e_dist.log 2>&1
cat gpurun_out/r2e_midblock_probe.txt; tail -5 gpurun_out/r2e_dist.log
