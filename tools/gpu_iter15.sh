VARIANTS="prune2 prune2R ballotR prune2 prune2R ballotR" bash tools/gpu_ab.sh
