#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2s
rm -f gpurun_out/parity_margins.jsonl
timeout 3500 python -m pytest tests -m gpu -q -rA --durations=30 > gpurun_out/r2s/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2s/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2s/smoke.log
cp gpurun_out/parity_margins.jsonl gpurun_out/r2s/ 2>/dev/null
tail -n 45 gpurun_out/r2s/pytest_gpu.log; cat gpurun_out/r2s/smoke.log
