# round evidence: gpu tests, default bench, ncu launch list + full capture of the search kernel, replay capture
set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 1 --no-cpu-baseline --e2e-pools 0 --replay-steps 1 --no-config5 > gpurun_out/ncu_list.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 1 -c 1 -o gpurun_out/search_full -f python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-pools 0 --no-replay > gpurun_out/ncu_full.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -s 1 -c 1 -o gpurun_out/replay_full -f python tools/replay_one.py resnet50 0.5 > gpurun_out/ncu_replay.out 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python tools/pool_latency.py > gpurun_out/pool_latency.txt 2>&1
tail -c 600 gpurun_out/bench.json; cat gpurun_out/bench_ref.json | head -c 400; cat gpurun_out/pool_latency.txt
