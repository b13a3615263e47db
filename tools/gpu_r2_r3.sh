set -x
COOP_REPLAY_PHASES=1 python tools/replay_one.py bilstm 0.216 1 16
COOP_REPLAY_PHASES=1 python tools/replay_one.py resnet50 0.5 1
COOP_REPLAY_PHASES=1 python tools/replay_one.py inception_v3 0.291 1
timeout 600 python -m pytest tests/test_replay_gpu.py tests/test_snapshots_gpu.py -x -q 2>&1 | tail -2
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_small.py replay > gpurun_out/san_racecheck_replay.txt 2>&1; tail -2 gpurun_out/san_racecheck_replay.txt
