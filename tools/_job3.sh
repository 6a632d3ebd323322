./build/mma_bench > gpurun_out/mma_bench2.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_ops.py tests/test_gpu_pipeline.py -x -q > gpurun_out/t3.log 2>&1; echo rc=$? >> gpurun_out/t3.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b3.json 2> gpurun_out/b3.err
