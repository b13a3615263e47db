set -x
timeout 900 python -m pytest tests/test_replay_gpu.py tests/test_snapshots_gpu.py tests/test_budget_gpu.py -x -q 2>&1 | tail -3
COOP_REPLAY_HELPER=1 timeout 900 python -m pytest tests/test_replay_gpu.py -x -q -k "dnn or random or fig2" 2>&1 | tail -2
COOP_REPLAY_PHASES=1 python tools/replay_one.py resnet50 0.5 1
COOP_REPLAY_PHASES=1 python tools/replay_one.py gpt3_2.7b 0.476 1
timeout 900 python bench.py --steps 3 --warmup 3 --no-config5 --e2e-pools 0 --cpu-seconds 2 > gpurun_out/b6.json 2> gpurun_out/b6.err; tail -2 gpurun_out/b6.err
python -c "
import json; d=json.load(open('gpurun_out/b6.json'))
for k in ('config2','config3'): v=d['replay'][k]; print(k, v['ms_per_sweep'], v['oracle_ms_per_sweep'], v['parity']['mismatches'])
"
timeout 1200 python tools/replay_timing.py 256 bilstm,gpt3_2.7b 2>&1 | grep cells
