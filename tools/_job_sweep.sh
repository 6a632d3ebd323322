#!/bin/bash
# TS conv planning sweep (conv_lab per-launch times) + the single-rank distributed test
OUT=gpurun_out/${TAG:-sw}; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_pipeline.py -m gpu -x -q > $OUT/t.log 2>&1; echo rc=$? >> $OUT/t.log
for cfg in "" "PST_TS_WMAX=150" "PST_TS_WMAX=150 PST_TS_TPS=1" "PST_TS_TPS=1" "PST_TS_NACC=2" "PST_TS_NACC=3" \
           "PST_TS_WMAX=150 PST_TS_NACC=2" "PST_TS_TPS=1 PST_TS_NACC=2" "PST_TS_TPS=1 PST_TS_NACC=3"; do
  env $cfg LAB_TAG="[$cfg]" timeout 120 python tools/conv_lab.py 50 >> $OUT/lab.txt 2>&1
done
