# quick state check: gpu tests + default bench
set -x
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
head -c 1500 gpurun_out/bench.json
