#!/bin/bash
# bench step time alternating between library builds (A/B on one box): usage tools/ab_libs.sh outdir lib1.so lib2.so ...
cd $GRAFT_REPO_ROOT
OUT=$1; shift
mkdir -p $OUT
for rep in 1 2; do
  for lib in "$@"; do
    PST_LIB_PATH=$lib timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 20 --warmup 5 > $OUT/b.json 2> $OUT/b.err
    echo "$lib $(python -c "import json; d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items() if k.startswith('conv')})")" >> $OUT/summary.txt
  done
done
cat $OUT/summary.txt
