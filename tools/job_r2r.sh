#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2r
timeout 900 python tools/stage_times.py 20 > gpurun_out/r2r/stage_times.jsonl 2> gpurun_out/r2r/stage_times.err
cat gpurun_out/r2r/stage_times.jsonl
