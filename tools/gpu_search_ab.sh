# A/B timing of search-kernel variants (env settings) on config 4, device-timed
for v in "" "COOP_SEARCH_TWO_CTA=1" "COOP_SEARCH_DBG=2" "COOP_SEARCH_TWO_CTA=1 COOP_SEARCH_DBG=2" $EXTRA; do
  env $v timeout 300 python bench.py --no-replay --no-cpu-baseline --e2e-pools 0 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$v]', round(d['ms_per_step'],2), round(d['roofline']['frac'],3))"
done
