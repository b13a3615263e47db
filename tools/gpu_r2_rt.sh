# replay timing on the heavy traces + parity of the replay tests
set -x
timeout 900 python -m pytest tests/test_replay_gpu.py -x -q 2>&1 | tail -2
timeout 900 python tools/replay_timing.py 256 bilstm,inception_v3,gpt3_2.7b,resnet50 2>&1
python tools/replay_one.py resnet50 0.5 1
