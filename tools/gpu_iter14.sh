VARIANTS="ballot prune2 ballot prune2" bash tools/gpu_ab.sh
