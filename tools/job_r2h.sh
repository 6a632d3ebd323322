#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/step_probe.py > gpurun_out/r2h_step_probe.txt 2>&1
cat gpurun_out/r2h_step_probe.txt
