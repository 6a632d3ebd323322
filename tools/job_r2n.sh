#!/bin/bash
# round-2 wgrad experiments on the experiment build: M tiles per CTA, unit size, converter sets
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2n
export PST_LIB=exp
for cfg in "PST_WT_GMAX=4" "PST_WT_GMAX=1" "PST_WT_GMAX=2" "PST_WT_GMAX=1 PST_WT_SETS=2" "PST_WT_PTARGET=16" "PST_WT_PTARGET=16 PST_WT_GMAX=1" "PST_WT_PTARGET=64 PST_WT_GMAX=1"; do
  env $cfg LAB_TAG="$cfg" timeout 120 python tools/conv_lab.py 50 >> gpurun_out/r2n/wgrad_knobs.txt 2>&1
done
cat gpurun_out/r2n/wgrad_knobs.txt
