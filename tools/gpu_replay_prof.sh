# source-level ncu capture of the replay kernel on config 2 (one cell) + per-line report
timeout 900 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -s 1 -c 1 -o gpurun_out/replay_src -f python tools/replay_cfg2.py > gpurun_out/ncu_rsrc.out 2>&1
tail -1 gpurun_out/ncu_rsrc.out
ncu -i gpurun_out/replay_src.ncu-rep --page source --csv --print-source sass > gpurun_out/replay_src_sass.csv 2>/dev/null
ncu -i gpurun_out/replay_src.ncu-rep --page raw --csv > gpurun_out/replay_src_raw.csv 2>/dev/null
SORT=stall python tools/sass_lines.py gpurun_out/replay_src_sass.csv paper_2311_00591_b200/libcoop.so replay_kernel 70 > gpurun_out/replay_lines_stall.txt 2>&1
