# round 2: source-level stall profile of the replay kernel on BASELINE config 2 (ResNet-50 @ 50 %, one cell)
set -x
python tools/replay_one.py resnet50 0.5 1
timeout 1200 ncu --section SourceCounters --section WarpStateStats --section LaunchStats --section Occupancy --clock-control none --import-source on -k regex:replay_kernel -s 1 -c 1 -o gpurun_out/replay_c2 -f python tools/replay_one.py resnet50 0.5 1 > gpurun_out/ncu_replay_c2.out 2>&1
tail -3 gpurun_out/ncu_replay_c2.out
ncu -i gpurun_out/replay_c2.ncu-rep --page source --csv --print-source sass > gpurun_out/replay_c2_sass.csv 2>/dev/null
python tools/sass_lines.py gpurun_out/replay_c2_sass.csv paper_2311_00591_b200/libcoop.so replay_kernel 70 > gpurun_out/replay_c2_lines.txt 2>&1
head -75 gpurun_out/replay_c2_lines.txt
