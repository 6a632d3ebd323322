timeout 600 python -m pytest tests/test_gpu_ops.py tests/test_gpu_pipeline.py -x -q > gpurun_out/t8.log 2>&1; echo rc=$? >> gpurun_out/t8.log
timeout 300 python tools/tl_probe.py > gpurun_out/tl9.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b8.json 2> gpurun_out/b8.err
