VARIANTS="cur2 warpver cur2 warpver" bash tools/gpu_ab.sh
