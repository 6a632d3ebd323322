export PST_GRAPHS=0
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches7.csv python bench.py --steps 1 --warmup 1 --profile-steps 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu7.log 2>&1
