VARIANTS="prune2 inplace prune2 inplace" bash tools/gpu_ab.sh
