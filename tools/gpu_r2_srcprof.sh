nproc; lscpu | grep "Model name"
bash tools/gpu_src_profile.sh
python tools/sass_lines.py gpurun_out/search_src_sass.csv paper_2311_00591_b200/libcoop.so search_kernelILi8ELi512ELi2E 80 > gpurun_out/search_lines.txt 2>&1
