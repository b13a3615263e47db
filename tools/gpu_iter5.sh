set -x
timeout 900 python -m pytest tests/test_pool_gpu.py -q -x 2>&1 | tail -5
timeout 300 python tools/pool_latency.py > gpurun_out/pool_latency.txt 2>&1; cat gpurun_out/pool_latency.txt
