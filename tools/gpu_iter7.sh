for d in 1 2 0; do DBG=$d VARIANTS="head2cta prune" bash tools/gpu_ab.sh | sed "s/^/dbg$d /"; done
