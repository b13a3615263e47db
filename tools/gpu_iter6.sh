set -x
timeout 900 python -m pytest tests/test_search_gpu.py -q -x 2>&1 | tail -5
VARIANTS="cur" bash tools/gpu_ab.sh
