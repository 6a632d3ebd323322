#!/bin/bash
# round-2: tcgen05 pipe counters available to ncu on B200, conv_lab baseline, full wgrad/TS captures
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2k
ncu --query-metrics --chip gb100 > gpurun_out/r2k/query_metrics.txt 2>&1 || ncu --query-metrics > gpurun_out/r2k/query_metrics.txt 2>&1
grep -i -E "tensor|umma|utc|tmem|tc_" gpurun_out/r2k/query_metrics.txt > gpurun_out/r2k/tensor_metrics.txt
timeout 300 python tools/conv_lab.py 50 > gpurun_out/r2k/conv_lab.txt 2>&1
export PST_GRAPHS=0
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_wgrad_ts -c 1 \
   -o gpurun_out/r2k/prof_wgrad_g1 python tools/conv_lab.py 1 > gpurun_out/r2k/ncu_wgrad.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_ts_kernel -c 1 \
   -o gpurun_out/r2k/prof_ts_g1 python tools/conv_lab.py 1 > gpurun_out/r2k/ncu_ts.log 2>&1
# every tensor-pipe-looking metric on one wgrad and one TS launch
M=$(grep -o -E "^[a-z0-9_]*(tensor|tmem|utc|umma)[a-z0-9_.]*" gpurun_out/r2k/tensor_metrics.txt | sort -u | head -60 | paste -sd, -)
echo "$M" > gpurun_out/r2k/tensor_metric_names.txt
timeout 600 ncu --metrics "$M" --clock-control none -k regex:"conv_wgrad_ts|conv_ts_kernel" -c 2 --csv \
   python tools/conv_lab.py 1 > gpurun_out/r2k/tensor_metrics_values.csv 2>&1
cat gpurun_out/r2k/conv_lab.txt; wc -l gpurun_out/r2k/*.txt
timeout 1500 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_fsbks.py tests/test_gpu_dist.py tests/test_gpu_midblock.py -q -x -k "not resnet110 and not table3" > gpurun_out/r2k/pytest_subset.log 2>&1; echo "rc=$?" >> gpurun_out/r2k/pytest_subset.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2k/bench_n1.log 2>&1
tail -5 gpurun_out/r2k/pytest_subset.log; tail -c 3000 gpurun_out/r2k/bench_n1.log
