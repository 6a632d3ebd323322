OUT=gpurun_out/p2; mkdir -p $OUT
export PST_GRAPHS=0
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 1 --profile-steps 0 --no-e2e --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
