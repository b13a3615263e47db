timeout 600 python -m pytest tests/test_search_gpu.py -x -q 2>&1 | tail -3
bash tools/gpu_dbg.sh
echo "--- one CTA per SM"
COOP_SEARCH_ONE_CTA=1 bash tools/gpu_dbg.sh
