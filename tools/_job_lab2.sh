#!/bin/bash
# In-graph marginal cost of each kernel class (PST_SKIP) and TS-conv knob experiments (conv_lab).
OUT=gpurun_out/${TAG:-lab}; mkdir -p $OUT
for sk in none fwd bnapply bnbwd wgrad dgrad sgd fwd,bnapply,bwdpre,bnbwd,wgrad,dgrad,sgd; do
  PST_SKIP=$sk timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --profile-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$sk', round(d['ms_per_step'],3))" >> $OUT/skip.txt
done
PST_WSTREAM=0 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --profile-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nowstream', round(d['ms_per_step'],3))" >> $OUT/skip.txt
for kn in 0 16 2 1 3 8 64 4; do
  PST_TS_KNOB=$kn LAB_TAG=knob$kn timeout 300 python tools/conv_lab.py 50 >> $OUT/lab.txt 2>&1
done
PST_LIB=bf16 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --profile-steps 2 > $OUT/bench_bf16.json 2>&1
