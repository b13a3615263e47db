# replay kernel source profile on a GPT-3 cell (warp BFS) + phases; R37 test
set -x
timeout 600 python -m pytest tests/test_replay_gpu.py -x -q -k r37 2>&1 | tail -2
COOP_REPLAY_PHASES=1 python tools/replay_one.py gpt3_2.7b 0.476 1
COOP_REPLAY_PHASES=1 COOP_REPLAY_WALK=lane python tools/replay_one.py gpt3_2.7b 0.476 1
COOP_REPLAY_PHASES=1 COOP_REPLAY_WALK=Group python tools/replay_one.py gpt3_2.7b 0.476 1
timeout 1500 ncu --section SourceCounters --section WarpStateStats --clock-control none --import-source on -k regex:replay_kernel -s 1 -c 1 -o gpurun_out/replay_g3 -f python tools/replay_one.py gpt3_2.7b 0.476 1 > gpurun_out/ncu_replay_g3.out 2>&1
tail -1 gpurun_out/ncu_replay_g3.out
ncu -i gpurun_out/replay_g3.ncu-rep --page source --csv --print-source sass > gpurun_out/replay_g3_sass.csv 2>/dev/null
ncu -i gpurun_out/replay_g3.ncu-rep --page raw --csv > gpurun_out/replay_g3_raw.csv 2>/dev/null
