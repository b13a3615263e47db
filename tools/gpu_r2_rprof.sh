# source-level stall profile of the replay kernel on a reduced BiLSTM cell (seq 16-18, 21.6 % of peak)
set -x
python tools/replay_one.py bilstm 0.216 1 16
timeout 1500 ncu --section SourceCounters --section WarpStateStats --section LaunchStats --clock-control none --import-source on -k regex:replay_kernel -s 1 -c 1 -o gpurun_out/replay_bl -f python tools/replay_one.py bilstm 0.216 1 16 > gpurun_out/ncu_replay_bl.out 2>&1
tail -2 gpurun_out/ncu_replay_bl.out
ncu -i gpurun_out/replay_bl.ncu-rep --page source --csv --print-source sass > gpurun_out/replay_bl_sass.csv 2>/dev/null
python tools/sass_lines.py gpurun_out/replay_bl_sass.csv paper_2311_00591_b200/libcoop.so replay_kernel 50 > gpurun_out/replay_bl_lines.txt 2>&1
head -55 gpurun_out/replay_bl_lines.txt
