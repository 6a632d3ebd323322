#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2q
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_ops.py -q -x > gpurun_out/r2q/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2q/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2q/bench1.json 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2q/bench2.json 2>&1
tail -3 gpurun_out/r2q/pytest.log
for f in bench1 bench2; do python -c "
import json,sys; l=json.loads(open('gpurun_out/r2q/$f.json').read().strip().splitlines()[-1]); print(l['value'], l['ms_per_step'], l['clocks'], {k:round(v['ms_per_step'],3) for k,v in l['kernels'].items()})"; done
