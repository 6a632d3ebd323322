#!/bin/bash
OUT=gpurun_out/${TAG:-ab}; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_ops.py tests/test_gpu_pipeline.py -m gpu -x -q > $OUT/t.log 2>&1; echo rc=$? >> $OUT/t.log
LAB_TAG=A timeout 120 python tools/conv_lab.py 50 > $OUT/lab.txt 2>&1
PST_LIB_PATH=$PWD/$PST_B LAB_TAG=B timeout 120 python tools/conv_lab.py 50 >> $OUT/lab.txt 2>&1
bash tools/_job_ab.sh
