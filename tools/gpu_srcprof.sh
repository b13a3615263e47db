# source-level ncu capture of the search kernel (131072 pools) + per-line report
set -x
KSUB=${KSUB:-search_kernelILi8ELi512ELi2E}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 1 -c 1 -o gpurun_out/search_src -f python bench.py --pools 131072 --steps 2 --warmup 1 --no-cpu-baseline --e2e-pools 0 --no-replay > gpurun_out/ncu_src.out 2>&1
tail -2 gpurun_out/ncu_src.out
ncu -i gpurun_out/search_src.ncu-rep --page source --csv --print-source sass > gpurun_out/search_src_sass.csv 2>/dev/null
ncu -i gpurun_out/search_src.ncu-rep --page raw --csv > gpurun_out/search_src_raw.csv 2>/dev/null
python tools/sass_lines.py gpurun_out/search_src_sass.csv paper_2311_00591_b200/libcoop.so $KSUB 120 > gpurun_out/search_lines.txt 2>&1
SORT=stall python tools/sass_lines.py gpurun_out/search_src_sass.csv paper_2311_00591_b200/libcoop.so $KSUB 60 > gpurun_out/search_lines_stall.txt 2>&1
for d in 1 2; do COOP_SEARCH_DBG=$d timeout 300 python bench.py --no-replay --no-cpu-baseline --e2e-pools 0 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dbg', $d, d['ms_per_step'])"; done
