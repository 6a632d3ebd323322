#!/bin/bash
OUT=gpurun_out/${TAG:-lab4}; mkdir -p $OUT
for kn in 3 2 1; do PST_TS_KNOB=$kn PST_DBG_TL=1 timeout 120 python tools/tl_probe.py g1 > $OUT/tl_g1_k$kn.txt 2>&1; done
PST_DBG_TL=1 timeout 120 python tools/tl_probe.py g1 wgrad > $OUT/tl_g1_wgrad.txt 2>&1
