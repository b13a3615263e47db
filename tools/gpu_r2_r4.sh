set -x
timeout 900 python -m pytest tests/test_replay_gpu.py tests/test_snapshots_gpu.py tests/test_pool_gpu.py tests/test_budget_gpu.py -x -q 2>&1 | tail -2
python tools/replay_one.py resnet50 0.5 1
timeout 900 python bench.py --steps 3 --warmup 3 --no-config5 --e2e-pools 0 --cpu-seconds 2 > gpurun_out/b4.json 2> gpurun_out/b4.err; tail -2 gpurun_out/b4.err
python -c "
import json; d=json.load(open('gpurun_out/b4.json'))
for k in ('config2','config3'): v=d['replay'][k]; print(k, v['ms_per_sweep'], v['oracle_ms_per_sweep'], v['parity'])
"
timeout 900 python tools/replay_timing.py 256 resnet50,inception_v3,gpt3_2.7b,spos 2>&1 | grep cells
