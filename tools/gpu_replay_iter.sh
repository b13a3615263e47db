# replay iteration: parity tests, then the bench's replay configs (with the oracle beside them)
timeout 1200 python -m pytest tests/test_replay_gpu.py tests/test_pool_gpu.py tests/test_budget_gpu.py tests/test_snapshots_gpu.py -x -q 2>&1 | tail -2
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-pools 0 $BENCH_EXTRA 2>/dev/null > gpurun_out/bench_replay.json
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_replay.json'))
for k,v in d['replay'].items():
    if isinstance(v,dict) and 'ms_per_sweep' in v:
        print(k, round(v['ms_per_sweep'],2), 'oracle', round(v.get('oracle_ms_per_sweep') or 0,2), 'x', round(v.get('gpu_vs_oracle') or 0,3), 'mism', (v.get('parity') or {}).get('mismatches'))
PY
