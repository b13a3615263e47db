timeout 600 ncu --section SourceCounters --section WarpStateStats --clock-control none --import-source on -k regex:replay_kernel -c 1 -o gpurun_out/replay_bilstm -f python tools/replay_one.py bilstm 0.401 > gpurun_out/ncu_bilstm.out 2>&1
tail -2 gpurun_out/ncu_bilstm.out
ncu -i gpurun_out/replay_bilstm.ncu-rep --page source --csv --print-source sass > gpurun_out/replay_bilstm_sass.csv 2>/dev/null
ls -la gpurun_out/replay_bilstm*
