VARIANTS="prune2 smemre prune2 smemre" bash tools/gpu_ab.sh
