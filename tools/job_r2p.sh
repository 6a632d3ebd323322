#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2p
timeout 600 python tools/measure_layer_costs.py > gpurun_out/r2p/b200_costs.json 2> gpurun_out/r2p/costs.err
cat gpurun_out/r2p/b200_costs.json
