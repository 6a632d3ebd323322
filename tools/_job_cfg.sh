#!/bin/bash
OUT=gpurun_out/${TAG:-cfg}; mkdir -p $OUT
timeout 1400 python -m pytest tests/test_gpu_configs.py -m gpu -q -k "resnet362 or balanced" > $OUT/t.log 2>&1; echo rc=$? >> $OUT/t.log
