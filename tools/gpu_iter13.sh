timeout 900 python -m pytest tests/test_search_gpu.py -q -x 2>&1 | tail -3
VARIANTS="cur prune2 cur prune2" bash tools/gpu_ab.sh
