timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python tools/pool_latency.py 2>&1
timeout 600 python tools/replay_timing.py 256 resnet50,inception_v3,swin_t,gpt3_2.7b,spos 2>&1 | grep -v slowest
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
