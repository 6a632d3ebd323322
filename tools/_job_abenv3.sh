#!/bin/bash
# default (A) vs $B_ENV (B) vs $C_ENV (C): parity tests under B and C, then alternating benches
OUT=gpurun_out/${TAG:-abenv3}; mkdir -p $OUT
env $B_ENV timeout 300 python -m pytest tests/test_gpu_ops.py tests/test_gpu_pipeline.py -m gpu -x -q > $OUT/tB.log 2>&1; echo rc=$? >> $OUT/tB.log
env $C_ENV timeout 300 python -m pytest tests/test_gpu_ops.py tests/test_gpu_pipeline.py -m gpu -x -q > $OUT/tC.log 2>&1; echo rc=$? >> $OUT/tC.log
for i in 1 2 3; do
  for v in A B C; do
    case $v in A) E="X=0";; B) E="$B_ENV";; C) E="$C_ENV";; esac
    env $E timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --profile-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), round(d['value']))" >> $OUT/ab.txt
  done
done
