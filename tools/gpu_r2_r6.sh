set -x
timeout 900 python -m pytest tests/test_replay_gpu.py tests/test_pool_gpu.py tests/test_snapshots_gpu.py -x -q 2>&1 | tail -2
python tools/replay_one.py resnet50 0.5 1
timeout 900 python tools/replay_timing.py 256 gpt3_2.7b,inception_v3 2>&1 | grep cells
