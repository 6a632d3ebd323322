set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tg.log 2>&1; echo rc=$? >> gpurun_out/tg.log
timeout 300 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
