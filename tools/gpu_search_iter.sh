# search-kernel iteration: parity tests, then device timing of config 4 (search only)
timeout 900 python -m pytest tests/test_search_gpu.py tests/test_snapshots_gpu.py tests/test_shard_determinism_gpu.py -x -q -k "not stream" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_full_parity_gpu.py -x -q -k config4 2>&1 | tail -1
for v in "" $EXTRA; do
  env $v timeout 300 python bench.py --no-replay --no-cpu-baseline --e2e-pools 0 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$v]', round(d['ms_per_step'],2), round(d['roofline']['frac'],3))"
done
