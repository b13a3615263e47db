timeout 900 python -m pytest tests/test_search_gpu.py -q -x 2>&1 | tail -3
VARIANTS="cur head2cta cur" bash tools/gpu_ab.sh
