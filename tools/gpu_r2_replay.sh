# round 2: replay parity (all GPU replay tests incl. the 2048-cell config-5 test) + timing
set -x
timeout 900 python -m pytest tests/test_replay_gpu.py tests/test_budget_gpu.py tests/test_pool_gpu.py -x -q 2>&1 | tail -5
timeout 600 python tools/replay_timing.py 2>&1
timeout 900 python -m pytest tests/test_full_parity_gpu.py -x -q -k config5 2>&1 | tail -5
