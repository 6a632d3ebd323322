for sk in none fwd bnapply bwdpre bnbwd wgrad dgrad sgd fwd,bnapply,bwdpre,bnbwd,wgrad,dgrad,sgd; do
  PST_SKIP=$sk timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --profile-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$sk', round(d['ms_per_step'],3))"
done
