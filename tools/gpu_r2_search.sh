# round 2: search kernel parity + timing (streaming kernel + CTA fallback)
set -x
timeout 900 python -m pytest tests/test_search_gpu.py tests/test_full_parity_gpu.py tests/test_shard_determinism_gpu.py -x -q -k "not config5" 2>&1 | tail -15
timeout 600 python bench.py --no-replay --no-cpu-baseline --e2e-pools 0 --steps 10 > gpurun_out/bench_s.json 2> gpurun_out/bench_s.err; tail -3 gpurun_out/bench_s.err; cut -c1-900 gpurun_out/bench_s.json
COOP_SEARCH_IMPL=cta timeout 600 python bench.py --no-replay --no-cpu-baseline --e2e-pools 0 --steps 10 > gpurun_out/bench_cta.json 2>&1; cut -c1-600 gpurun_out/bench_cta.json
