set -x
python tools/stream_stats.py 262144
COOP_SEARCH_IMPL=stream_only python tools/stream_stats.py 262144
COOP_SEARCH_IMPL=cta python tools/stream_stats.py 262144
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search_stream -s 2 -c 1 -o gpurun_out/stream_src -f env COOP_SEARCH_IMPL=stream_only python tools/stream_stats.py 65536 > gpurun_out/ncu_stream.out 2>&1
tail -2 gpurun_out/ncu_stream.out
ncu -i gpurun_out/stream_src.ncu-rep --page source --csv --print-source sass > gpurun_out/stream_sass.csv 2>/dev/null
ncu -i gpurun_out/stream_src.ncu-rep --page raw --csv > gpurun_out/stream_raw.csv 2>/dev/null
python tools/sass_lines.py gpurun_out/stream_sass.csv paper_2311_00591_b200/libcoop.so search_stream 60 > gpurun_out/stream_lines.txt 2>&1
head -64 gpurun_out/stream_lines.txt
