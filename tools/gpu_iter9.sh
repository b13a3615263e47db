VARIANTS="cur head2cta" bash tools/gpu_ab.sh
bash tools/gpu_src_profile.sh
