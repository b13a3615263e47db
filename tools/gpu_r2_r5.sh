set -x
python tools/replay_one.py resnet50 0.5 1
timeout 900 python tools/replay_timing.py 256 gpt3_2.7b,inception_v3,resnet50 2>&1 | grep cells
timeout 900 python bench.py --steps 3 --warmup 3 --no-config5 --e2e-pools 0 --cpu-seconds 2 > gpurun_out/b5.json 2> gpurun_out/b5.err; tail -2 gpurun_out/b5.err
python -c "
import json; d=json.load(open('gpurun_out/b5.json'))
for k in ('config2','config3'): v=d['replay'][k]; print(k, v['ms_per_sweep'], v['oracle_ms_per_sweep'], v['parity']['mismatches'])
"
