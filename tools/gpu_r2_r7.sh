set -x
python tools/replay_one.py bilstm 0.216 1 16
COOP_REPLAY_GSMEM=0 python tools/replay_one.py bilstm 0.216 1 16
COOP_REPLAY_GSMEM=0 timeout 900 python tools/replay_timing.py 256 gpt3_2.7b,inception_v3,resnet50,spos 2>&1 | grep cells
timeout 900 python tools/replay_timing.py 256 spos 2>&1 | grep cells
COOP_REPLAY_PHASES=1 timeout 900 python tools/replay_one.py bilstm 0.2156 1
