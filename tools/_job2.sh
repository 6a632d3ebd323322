./build/mma_bench > gpurun_out/mma_bench.txt 2>&1
export PST_GRAPHS=0
BENCH="python bench.py --steps 1 --warmup 1 --profile-steps 0 --no-e2e --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:conv_fwd_kernel<\(bool\)0, \(bool\)0>' -s 150 -c 1 -o gpurun_out/prof_fwd2 $BENCH > gpurun_out/ncu_fwd2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:conv_fwd_kernel<\(bool\)0, \(bool\)1>' -s 150 -c 1 -o gpurun_out/prof_dgrad2 $BENCH > gpurun_out/ncu_dgrad2.log 2>&1
