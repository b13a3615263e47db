for d in 1 2 4 5 6 0; do DBG=$d VARIANTS="cur" bash tools/gpu_ab.sh | sed "s/^/dbg$d /"; done
bash tools/gpu_src_profile.sh
