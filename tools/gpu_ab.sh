# A/B timing of libcoop variants: VARIANTS="head cur cur:K4" bash tools/gpu_ab.sh
# (<name>[:K4|:TWO] -- variants/<name>.so, "cur" = the in-tree build; suffix sets an env knob)
for spec in ${VARIANTS:-head}; do
  v=${spec%%:*}; knob=${spec#*:}; [ "$knob" = "$spec" ] && knob=""
  if [ "$v" = cur ]; then lib=""; else lib=variants/$v.so; fi
  k4=0; two=0; [ "$knob" = K4 ] && k4=1; [ "$knob" = TWO ] && two=1
  COOP_SEARCH_K4=$k4 COOP_SEARCH_TWO_CTA=$two COOP_LIB_OVERRIDE=$lib COOP_SEARCH_DBG=${DBG:-0} timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-pools 0 --no-replay 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$spec', 'ms', round(d['ms_per_step'],2), 'GB/s', round(d['roofline']['achieved'],1))"
done
