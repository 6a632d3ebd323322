OUT=gpurun_out/p1
mkdir -p $OUT
export PST_GRAPHS=0
BENCH="python bench.py --steps 1 --warmup 1 --profile-steps 0 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -c 3000 --csv --log-file $OUT/launches.csv $BENCH > $OUT/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_ts_kernel -s 20 -c 1 -o $OUT/prof_fwd $BENCH > $OUT/ncu_fwd.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_wgrad_ts -s 20 -c 1 -o $OUT/prof_wgrad $BENCH > $OUT/ncu_wgrad.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bwd_pre -s 20 -c 1 -o $OUT/prof_bwdpre $BENCH > $OUT/ncu_bwdpre.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bn_apply -s 20 -c 1 -o $OUT/prof_bnapply $BENCH > $OUT/ncu_bnapply.log 2>&1
ls -la $OUT
