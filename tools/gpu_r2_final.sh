# round 2 final: smoke, full GPU tests, default bench, reference arm, sanitizers
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; tail -2 gpurun_out/smoke_final.log
timeout 1800 python -m pytest tests -q -m gpu -x --durations=10 > gpurun_out/pytest_gpu_final.log 2>&1; tail -16 gpurun_out/pytest_gpu_final.log
timeout 1500 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -3 gpurun_out/bench_final.err; head -c 400 gpurun_out/bench_final.json
timeout 600 python bench.py --impl reference > gpurun_out/bench_final_ref.json 2>&1; tail -c 300 gpurun_out/bench_final_ref.json
for tool in memcheck racecheck synccheck; do
  for w in search replay pool; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py $w > gpurun_out/san_${tool}_${w}.txt 2>&1
    echo "$tool $w rc=$?"; tail -1 gpurun_out/san_${tool}_${w}.txt
  done
done
