#!/bin/bash
OUT=gpurun_out/${TAG:-costs}; mkdir -p $OUT
timeout 300 python tools/measure_layer_costs.py > $OUT/b200_costs.json 2> $OUT/costs.err
