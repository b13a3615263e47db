COOP_LIB_OVERRIDE=variants/zero2.so timeout 900 python -m pytest tests/test_search_gpu.py -q -x 2>&1 | tail -3
VARIANTS="final zero2 final zero2" bash tools/gpu_ab.sh
