COOP_LIB_OVERRIDE=variants/constT.so timeout 900 python -m pytest tests/test_search_gpu.py -q -x 2>&1 | tail -3
VARIANTS="final constT final constT" bash tools/gpu_ab.sh
