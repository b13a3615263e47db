# evidence run: smoke, full GPU tests, default bench, launch list + one full ncu capture of the search kernel
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -q -m gpu -x --durations=8 > gpurun_out/pytest_gpu.log 2>&1; tail -12 gpurun_out/pytest_gpu.log
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; head -c 300 gpurun_out/bench.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-pools 0 > gpurun_out/ncu_list.out 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 3 -c 1 -o gpurun_out/search_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-pools 0 --no-replay > gpurun_out/ncu_full.out 2>&1; echo "ncu full rc=$?"
ncu -i gpurun_out/search_full.ncu-rep --page raw --csv > gpurun_out/search_full_raw.csv 2>/dev/null
