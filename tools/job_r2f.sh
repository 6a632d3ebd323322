#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/midblock_probe.py "" 1 3 5 7 3,5 3,7 5,7 2,3 1,2,3 > gpurun_out/r2f_probe.txt 2>&1
timeout 600 python tools/momentum_probe.py > gpurun_out/r2f_momentum_probe.txt 2>&1
cat gpurun_out/r2f_probe.txt gpurun_out/r2f_momentum_probe.txt
