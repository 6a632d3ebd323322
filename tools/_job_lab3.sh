#!/bin/bash
OUT=gpurun_out/${TAG:-lab3}; mkdir -p $OUT
for g in g1 g3; do PST_DBG_TL=1 timeout 120 python tools/tl_probe.py $g > $OUT/tl_$g.txt 2>&1; done
for kn in 2 3 32 34; do
  PST_TS_KNOB=$kn LAB_TAG=knob$kn timeout 120 python tools/conv_lab.py 50 >> $OUT/lab.txt 2>&1
done
for sk in wgrad fwd,bnapply,bwdpre,bnbwd,wgrad,dgrad,sgd; do
  PST_SKIP=$sk timeout 120 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --profile-steps 0 2>$OUT/skip_err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$sk', round(d['ms_per_step'],3))" >> $OUT/skip.txt
done
timeout 1400 python -m pytest tests/test_gpu_configs.py -m gpu -q --durations=0 > $OUT/t.log 2>&1; echo rc=$? >> $OUT/t.log
