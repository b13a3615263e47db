set -x
timeout 900 python -m pytest tests/test_replay_gpu.py tests/test_snapshots_gpu.py -x -q 2>&1 | tail -2
COOP_REPLAY_PHASES=1 python tools/replay_one.py bilstm 0.216 1 16
COOP_REPLAY_PHASES=1 python tools/replay_one.py resnet50 0.5 1
timeout 900 python tools/replay_timing.py 256 gpt3_2.7b,inception_v3,resnet50,spos,bert_large,swin_t,unet 2>&1 | grep cells
COOP_REPLAY_PHASES=1 timeout 900 python tools/replay_one.py bilstm 0.2156 1
