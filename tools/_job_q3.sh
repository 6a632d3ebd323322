#!/bin/bash
OUT=gpurun_out/${TAG:-q3}; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_ops.py tests/test_gpu_pipeline.py -m gpu -x -q > $OUT/t.log 2>&1; echo rc=$? >> $OUT/t.log
LAB_TAG=sets3 timeout 120 python tools/conv_lab.py 50 > $OUT/lab.txt 2>&1
PST_LIB_PATH=$PWD/paper_1912_12675_b200/libpst_ts4.so LAB_TAG=sets4 timeout 120 python tools/conv_lab.py 50 >> $OUT/lab.txt 2>&1
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --profile-steps 0 > $OUT/bench.json 2> $OUT/bench.err
PST_LIB_PATH=$PWD/paper_1912_12675_b200/libpst_ts4.so timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --profile-steps 0 > $OUT/bench_ts4.json 2> $OUT/bench_ts4.err
