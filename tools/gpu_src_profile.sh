# source-level ncu capture of the search kernel (131072 pools) for tools/sass_lines.py
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 1 -c 1 -o gpurun_out/search_src -f python bench.py --pools 131072 --steps 2 --warmup 1 --no-cpu-baseline --e2e-pools 0 --no-replay > gpurun_out/ncu_src.out 2>&1
tail -2 gpurun_out/ncu_src.out
ncu -i gpurun_out/search_src.ncu-rep --page source --csv --print-source sass > gpurun_out/search_src_sass.csv 2>/dev/null
ncu -i gpurun_out/search_src.ncu-rep --page raw --csv > gpurun_out/search_src_raw.csv 2>/dev/null
ls -la gpurun_out/search_src*
