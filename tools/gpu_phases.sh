# cumulative phase times of the search kernel (variants/hooks.so: COOP_SEARCH_PHASE_HOOKS build)
for d in 1 2 4 3 5 6 0; do
  COOP_LIB_OVERRIDE=variants/hooks.so COOP_SEARCH_DBG=$d timeout 300 python bench.py --no-replay --no-cpu-baseline --e2e-pools 0 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dbg $d', round(d['ms_per_step'],2))"
done
