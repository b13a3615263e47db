COOP_LIB_OVERRIDE=variants/k4.so timeout 900 python -m pytest tests/test_search_gpu.py -q -x 2>&1 | tail -3
VARIANTS="headnh k4 prune2 headnh k4" bash tools/gpu_ab.sh
