#!/bin/bash
# The GPU test suite with the parity-margin log, then the smoke test (run under gpurun on one B200).
# usage: tools/gpu_suite.sh [outdir]
cd $GRAFT_REPO_ROOT
OUT=${1:-gpurun_out/suite}
mkdir -p $OUT
rm -f gpurun_out/parity_margins.jsonl
timeout 3500 python -m pytest tests -m gpu -q -rA --durations=30 > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
cp gpurun_out/parity_margins.jsonl $OUT/ 2>/dev/null
tail -n 45 $OUT/pytest_gpu.log; cat $OUT/smoke.log
