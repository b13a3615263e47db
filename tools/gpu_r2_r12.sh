set -x
timeout 900 python -m pytest tests/test_replay_gpu.py tests/test_snapshots_gpu.py -x -q 2>&1 | tail -2
COOP_REPLAY_PHASES=1 COOP_REPLAY_WALK=Group python tools/replay_one.py bilstm 0.216 1 16
COOP_REPLAY_WALK=Group timeout 1200 python tools/replay_timing.py 256 2>&1 | grep cells
