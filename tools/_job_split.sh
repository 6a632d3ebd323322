#!/bin/bash
# wgrad / dgrad SM split sweep (forked wgrad stream): ms per step
OUT=gpurun_out/${TAG:-split}; mkdir -p $OUT
for cfg in "PST_WG_SMS=84 PST_DG_CTAS=64" "PST_WG_SMS=84 PST_DG_CTAS=64" "X=0" "PST_WG_SMS=84 PST_DG_CTAS=64" "PST_WG_SMS=84 PST_DG_CTAS=64" "PST_WG_SMS=84 PST_DG_CTAS=64" "PST_WG_SMS=84 PST_DG_CTAS=64" "X=0" "PST_WG_SMS=84 PST_DG_CTAS=64" "PST_WG_SMS=84 PST_DG_CTAS=64"; do
  env $cfg timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --profile-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', round(d['ms_per_step'],3), round(d['value']))" >> $OUT/split.txt
done
