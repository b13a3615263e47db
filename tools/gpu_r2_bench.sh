# round 2: full default bench + launch list + ncu --set full of the search kernel
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; tail -3 gpurun_out/bench_r02.err
head -c 600 gpurun_out/bench_r02.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_r02_ref.json 2>&1; tail -c 400 gpurun_out/bench_r02_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 3 --warmup 1 --no-cpu-baseline --e2e-pools 0 --no-config5 > gpurun_out/ncu_list_r02.out 2>&1
tail -2 gpurun_out/ncu_list_r02.out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 1 -c 1 -o gpurun_out/search_full_r02 -f python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-pools 0 --no-replay > gpurun_out/ncu_full_r02.out 2>&1
tail -2 gpurun_out/ncu_full_r02.out
ncu -i gpurun_out/search_full_r02.ncu-rep --page raw --csv > gpurun_out/search_full_r02_raw.csv 2>/dev/null
ls -la gpurun_out/ | tail -20
