timeout 1200 python tools/ablation.py > gpurun_out/ablation.txt 2>&1; cat gpurun_out/ablation.txt
timeout 900 python -m pytest tests/test_replay_gpu.py -q -x -k "ablation" 2>&1 | tail -3
