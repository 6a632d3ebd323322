#!/bin/bash
# bench step time under experiment knobs (libpst_exp.so): usage tools/ab_knobs.sh outdir "VAR=val VAR2=val" ...
cd $GRAFT_REPO_ROOT
OUT=$1; shift
mkdir -p $OUT
i=0
for kv in "$@"; do
  env PST_LIB=exp $kv timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 20 --warmup 5 > $OUT/b$i.json 2> $OUT/b$i.err
  echo "$kv $(python -c "import json,sys; d=json.loads(open('$OUT/b$i.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items() if k.startswith('conv')})")" >> $OUT/summary.txt
  i=$((i+1))
done
cat $OUT/summary.txt
