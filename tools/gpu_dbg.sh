for m in ${DBG_MODES:-0}; do
  COOP_SEARCH_DBG=$m timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-pools 0 --no-replay 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dbg', $m, 'ms', round(d['ms_per_step'],2), 'GB/s', round(d['roofline']['achieved'],1))"
done
