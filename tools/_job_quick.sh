#!/bin/bash
# quick iteration: kernel parity tests, conv timings, short bench
OUT=gpurun_out/${TAG:-q}; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_ops.py tests/test_gpu_pipeline.py -m gpu -x -q > $OUT/t.log 2>&1; echo rc=$? >> $OUT/t.log
timeout 120 python tools/conv_lab.py 50 > $OUT/lab.txt 2>&1
PST_DBG_TL=1 timeout 120 python tools/tl_probe.py g1 wgrad 2>&1 | grep TLW > $OUT/tl_wgrad.txt
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --profile-steps 0 > $OUT/bench.json 2> $OUT/bench.err
PST_FUSE_PRE=0 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --profile-steps 0 > $OUT/bench_nofuse.json 2>&1
