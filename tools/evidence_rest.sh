#!/bin/bash
cd $GRAFT_REPO_ROOT
OUT=${1:-gpurun_out/evd}
mkdir -p $OUT
PST_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_n2_shared_gpu.json 2>> $OUT/bench.err
timeout 900 python tools/stage_times.py 20 > $OUT/stage_times.jsonl 2>> $OUT/bench.err
export PST_GRAPHS=0
BENCH="python bench.py --steps 1 --warmup 1 --profile-steps 0 --no-e2e --no-cpu-baseline --spin-seconds 0"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 3000 --csv --log-file $OUT/traffic.csv $BENCH > $OUT/ncu_traffic_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_wgrad -s 100 -c 1 \
  -o $OUT/prof_wgrad $BENCH > $OUT/ncu_wgrad.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_ts_kernel -s 200 -c 1 \
  -o $OUT/prof_ts $BENCH > $OUT/ncu_ts.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bn_apply -s 50 -c 1 \
  -o $OUT/prof_bn_apply $BENCH > $OUT/ncu_bn_apply.log 2>&1
ls -la $OUT
tail -c 400 $OUT/bench.json; cat $OUT/stage_times.jsonl
