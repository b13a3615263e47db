COOP_SEARCH_DBG=9 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-pools 0 --no-replay 2>&1 | grep dbg9 | tail -1
COOP_SEARCH_ONE_CTA=1 COOP_SEARCH_DBG=9 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-pools 0 --no-replay 2>&1 | grep dbg9 | tail -1
