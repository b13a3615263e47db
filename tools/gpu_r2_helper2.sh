set -x
COOP_REPLAY_HELPER=3 timeout 900 python -m pytest tests/test_replay_gpu.py -x -q -k "dnn or random or fig2 or dtr" 2>&1 | tail -2
COOP_REPLAY_HELPER=2 timeout 900 python -m pytest tests/test_replay_gpu.py -x -q -k "dnn_traces or config3" 2>&1 | tail -2
for h in 1 2 3; do COOP_REPLAY_HELPER=$h timeout 1200 python tools/replay_timing.py 256 bilstm 2>&1 | grep -A1 cells; done
for h in 1 2 3; do COOP_REPLAY_HELPER=$h python tools/replay_one.py gpt3_2.7b 0.476 64; done
