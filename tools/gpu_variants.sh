# device timing of config 4 for variant libraries (variants/<name>.so)
for v in $VARIANTS; do
  COOP_LIB_OVERRIDE=variants/$v.so timeout 300 python bench.py --no-replay --no-cpu-baseline --e2e-pools 0 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],2))"
done
