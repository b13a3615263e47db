set -x
timeout 900 python -m pytest tests/test_search_gpu.py tests/test_full_parity_gpu.py -x -q -k "not config5" 2>&1 | tail -4
python tools/stream_stats.py 262144
COOP_SEARCH_IMPL=stream_only python tools/stream_stats.py 262144
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search_stream -s 2 -c 1 -o gpurun_out/stream_src -f env COOP_SEARCH_IMPL=stream_only python tools/stream_stats.py 65536 > gpurun_out/ncu_stream.out 2>&1
ncu -i gpurun_out/stream_src.ncu-rep --page source --csv --print-source sass > gpurun_out/stream_sass.csv 2>/dev/null
ncu -i gpurun_out/stream_src.ncu-rep --page raw --csv > gpurun_out/stream_raw.csv 2>/dev/null
python tools/sass_lines.py gpurun_out/stream_sass.csv paper_2311_00591_b200/libcoop.so search_stream 45 > gpurun_out/stream_lines.txt 2>&1
head -48 gpurun_out/stream_lines.txt
