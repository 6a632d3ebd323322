#!/bin/bash
# A/B on one box: default (A) vs the env assignment in $B_ENV (B); parity tests run under B
OUT=gpurun_out/${TAG:-abenv}; mkdir -p $OUT
env $B_ENV timeout 300 python -m pytest tests/test_gpu_ops.py tests/test_gpu_pipeline.py -m gpu -x -q > $OUT/t.log 2>&1; echo rc=$? >> $OUT/t.log
LAB_TAG=A timeout 120 python tools/conv_lab.py 50 > $OUT/lab.txt 2>&1
env $B_ENV LAB_TAG=B timeout 120 python tools/conv_lab.py 50 >> $OUT/lab.txt 2>&1
for i in 1 2 3; do
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --profile-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('A', round(d['ms_per_step'],4), round(d['value']))" >> $OUT/ab.txt
  env $B_ENV timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --profile-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('B', round(d['ms_per_step'],4), round(d['value']))" >> $OUT/ab.txt
done
