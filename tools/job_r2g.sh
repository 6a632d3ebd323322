#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PST_FUSE_PRE=0 timeout 600 python tools/momentum_probe.py > gpurun_out/r2g_nofuse.txt 2>&1
cat gpurun_out/r2g_nofuse.txt | grep -E "seed|layer[123]\.(W|beta)"
