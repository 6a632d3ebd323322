#!/bin/bash
# round-2 job: full GPU suite (spread-derived tolerances everywhere, mid-block, dropout), smoke
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/parity_margins.jsonl
timeout 3000 python -m pytest tests -m gpu -q -rA --durations=20 > gpurun_out/r2c_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_smoke.log
tail -n 30 gpurun_out/r2c_pytest_gpu.log
