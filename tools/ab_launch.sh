#!/bin/bash
# one-step ncu launch lists (experiment build) under several knob settings, grouped by kernel + grid.
# usage: tools/ab_launch.sh outdir "VAR=val" ...
cd $GRAFT_REPO_ROOT
OUT=$1; shift
mkdir -p $OUT
i=0
for kv in "$@"; do
  env PST_LIB=exp PST_GRAPHS=0 $kv timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -c 1200 --csv \
    --log-file $OUT/l$i.csv python bench.py --steps 1 --warmup 1 --profile-steps 0 --no-e2e --no-cpu-baseline --spin-seconds 0 > $OUT/ncu$i.log 2>&1
  echo "== $kv" >> $OUT/groups.txt
  python tools/launch_groups.py $OUT/l$i.csv | head -14 >> $OUT/groups.txt
  i=$((i+1))
done
cat $OUT/groups.txt
