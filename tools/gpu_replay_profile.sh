# source-level ncu capture of the replay kernel on one inception_v3 cell (30 % budget)
timeout 1200 ncu --section SourceCounters --section WarpStateStats --section LaunchStats --section Occupancy --clock-control none --import-source on -k regex:replay_kernel -c 1 -o gpurun_out/replay_src -f python tools/replay_one.py inception_v3 0.3 1 > gpurun_out/ncu_replay.out 2>&1
tail -3 gpurun_out/ncu_replay.out
ncu -i gpurun_out/replay_src.ncu-rep --page source --csv --print-source sass > gpurun_out/replay_src_sass.csv 2>/dev/null
ncu -i gpurun_out/replay_src.ncu-rep --page raw --csv > gpurun_out/replay_src_raw.csv 2>/dev/null
ls -la gpurun_out/replay_src*
