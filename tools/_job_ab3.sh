#!/bin/bash
# A/B/C on one box: libpst.so vs $PST_B vs $PST_C (bench ms per step, alternating)
OUT=gpurun_out/${TAG:-ab3}; mkdir -p $OUT
for i in 1 2 3; do
  for v in A B C; do
    case $v in A) unset PST_LIB_PATH;; B) export PST_LIB_PATH=$PWD/$PST_B;; C) export PST_LIB_PATH=$PWD/$PST_C;; esac
    timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --profile-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), round(d['value']))" >> $OUT/ab.txt
  done
done
