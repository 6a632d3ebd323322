timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/tg.log 2>&1; echo rc=$? >> gpurun_out/tg.log
for f in 1 0; do
  PST_FUSE_PRE=$f timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --profile-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fuse=$f', round(d['ms_per_step'],3), round(d['value']))"
done
