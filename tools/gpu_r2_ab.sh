# A/B of the replay closure walk variants on a reduced BiLSTM cell and two full sweeps + snapshot tests
set -x
timeout 600 python -m pytest tests/test_snapshots_gpu.py -x -q 2>&1 | tail -3
python tools/replay_one.py bilstm 0.216 1 16
COOP_REPLAY_GSMEM=0 python tools/replay_one.py bilstm 0.216 1 16
COOP_REPLAY_WALK=generic python tools/replay_one.py bilstm 0.216 1 16
python tools/replay_timing.py 256 inception_v3,gpt3_2.7b
COOP_REPLAY_GSMEM=0 python tools/replay_timing.py 256 inception_v3,gpt3_2.7b
COOP_REPLAY_WALK=generic python tools/replay_timing.py 256 inception_v3,gpt3_2.7b
