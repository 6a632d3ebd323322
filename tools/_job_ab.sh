#!/bin/bash
# A/B on one box: libpst.so (A) vs $PST_B (B), alternating, ms per step
OUT=gpurun_out/${TAG:-ab}; mkdir -p $OUT
for i in 1 2 3 4; do
  for v in A B; do
    if [ $v = B ]; then export PST_LIB_PATH=$PWD/$PST_B; else unset PST_LIB_PATH; fi
    timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --profile-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), round(d['value']))" >> $OUT/ab.txt
  done
done
