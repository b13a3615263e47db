set -x
timeout 600 python -m pytest tests/test_replay_gpu.py -x -q 2>&1 | tail -30
timeout 600 python -m pytest tests/test_search_gpu.py -x -q 2>&1 | tail -5
timeout 300 python bench.py --no-cpu-baseline --e2e-pools 0 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cut -c1-700 gpurun_out/bench.json
