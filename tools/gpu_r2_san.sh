set -x
COOP_REPLAY_PHASES=1 python tools/replay_one.py bilstm 0.216 1 16
COOP_REPLAY_PHASES=1 python tools/replay_one.py resnet50 0.5 1
COOP_REPLAY_PHASES=1 python tools/replay_one.py inception_v3 0.291 1
for tool in memcheck racecheck synccheck; do
  for w in search replay pool; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py $w > gpurun_out/san_${tool}_${w}.txt 2>&1
    echo "$tool $w rc=$?"; tail -3 gpurun_out/san_${tool}_${w}.txt
  done
done
