# compute-sanitizer on the search kernel (small invocations incl. the rare tie path)
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py search > gpurun_out/san_${tool}_search.txt 2>&1
  echo "$tool search rc=$?"; tail -2 gpurun_out/san_${tool}_search.txt
done
