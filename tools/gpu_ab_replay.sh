# A/B of a replay-engine variant: parity tests with the variant, then sweep timings of both
# usage: V=variants/<name>.so bash tools/gpu_ab_replay.sh
COOP_LIB_OVERRIDE=$V timeout 1200 python -m pytest tests/test_replay_gpu.py tests/test_pool_gpu.py tests/test_budget_gpu.py -q -x 2>&1 | tail -3
for lib in "" $V; do
  echo "lib=$lib"
  COOP_LIB_OVERRIDE=$lib timeout 600 python tools/replay_timing.py 256 resnet50,inception_v3,swin_t,gpt3_2.7b,spos 2>&1 | grep -v slowest
  COOP_LIB_OVERRIDE=$lib timeout 600 python tools/replay_timing.py 16 bilstm 2>&1
done
