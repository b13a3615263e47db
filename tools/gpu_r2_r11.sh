set -x
timeout 900 python -m pytest tests/test_replay_gpu.py tests/test_snapshots_gpu.py -x -q 2>&1 | tail -2
COOP_REPLAY_WALK=warp timeout 600 python -m pytest tests/test_replay_gpu.py -x -q -k "dnn or fig2 or random" 2>&1 | tail -2
COOP_REPLAY_WALK=lane timeout 600 python -m pytest tests/test_replay_gpu.py -x -q -k "dnn or fig2 or random" 2>&1 | tail -2
timeout 1200 python tools/replay_timing.py 256 2>&1 | grep cells
