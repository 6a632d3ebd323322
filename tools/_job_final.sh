#!/bin/bash
# Round-end evidence: gpu tests, smoke, bench (default contract) + reference arm, ncu launch list with
# DRAM bytes per launch, full captures of the wgrad and TS conv kernels.
OUT=gpurun_out/${TAG:-final}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > $OUT/tg.log 2>&1; echo rc=$? >> $OUT/tg.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo rc=$? >> $OUT/smoke.log
timeout 400 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 400 python bench.py > $OUT/bench2.json 2> $OUT/bench2.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
export PST_GRAPHS=0
BENCH="python bench.py --steps 1 --warmup 1 --profile-steps 0 --no-e2e --no-cpu-baseline --spin-seconds 0"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 3000 --csv --log-file $OUT/traffic.csv $BENCH > $OUT/ncu_traffic_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_wgrad -s 100 -c 1 \
  -o $OUT/prof_wgrad $BENCH > $OUT/ncu_wgrad.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_ts_kernel -s 150 -c 1 \
  -o $OUT/prof_ts $BENCH > $OUT/ncu_ts.log 2>&1
