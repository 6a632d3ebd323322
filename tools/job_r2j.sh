#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/parity_margins.jsonl
timeout 3300 python -m pytest tests -m gpu -q -rA --durations=25 > gpurun_out/r2j_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2j_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_smoke.log
tail -n 40 gpurun_out/r2j_pytest_gpu.log
