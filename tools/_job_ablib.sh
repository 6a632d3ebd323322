#!/bin/bash
# A/B on one box: libpst.so (A) vs the library $PST_B (B): parity tests (A), conv_lab (+knob16), benches
OUT=gpurun_out/${TAG:-ablib}; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_ops.py tests/test_gpu_pipeline.py -m gpu -x -q > $OUT/t.log 2>&1; echo rc=$? >> $OUT/t.log
LAB_TAG=A timeout 120 python tools/conv_lab.py 50 > $OUT/lab.txt 2>&1
PST_LIB_PATH=$PWD/$PST_B LAB_TAG=B timeout 120 python tools/conv_lab.py 50 >> $OUT/lab.txt 2>&1
PST_TS_KNOB=16 LAB_TAG=A16 timeout 120 python tools/conv_lab.py 50 >> $OUT/lab.txt 2>&1
PST_TS_KNOB=16 PST_LIB_PATH=$PWD/$PST_B LAB_TAG=B16 timeout 120 python tools/conv_lab.py 50 >> $OUT/lab.txt 2>&1
for i in 1 2 3; do
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --profile-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('A', round(d['ms_per_step'],4), round(d['value']))" >> $OUT/ab.txt
  PST_LIB_PATH=$PWD/$PST_B timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --profile-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('B', round(d['ms_per_step'],4), round(d['value']))" >> $OUT/ab.txt
done
