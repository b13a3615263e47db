# source-level profile of the replay kernel (current build) on the reduced BiLSTM cell
set -x
timeout 1500 ncu --section SourceCounters --section WarpStateStats --section LaunchStats --section Occupancy --clock-control none --import-source on -k regex:replay_kernel -s 1 -c 1 -o gpurun_out/replay_bl2 -f python tools/replay_one.py bilstm 0.216 1 16 > gpurun_out/ncu_replay_bl2.out 2>&1
tail -2 gpurun_out/ncu_replay_bl2.out
ncu -i gpurun_out/replay_bl2.ncu-rep --page source --csv --print-source sass > gpurun_out/replay_bl2_sass.csv 2>/dev/null
ncu -i gpurun_out/replay_bl2.ncu-rep --page raw --csv > gpurun_out/replay_bl2_raw.csv 2>/dev/null
ls -la gpurun_out/replay_bl2*
