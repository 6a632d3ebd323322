#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python tools/midblock_probe.py 1,2,3,6 1,2,3 2,3,6 1,3,6 3,6 7 3,5 3,7 5,7 1,2,3,4 > gpurun_out/r2i_probe.txt 2>&1
cat gpurun_out/r2i_probe.txt
