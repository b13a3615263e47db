for d in 2 3 4 5 6 0; do DBG=$d VARIANTS="prunedbg" bash tools/gpu_ab.sh | sed "s/^/dbg$d /"; done
