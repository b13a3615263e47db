set -x
VARIANTS="cur two512" bash tools/gpu_ab.sh
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pool_kernel -c 300 --csv --log-file gpurun_out/pool_ncu.csv python tools/pool_latency.py > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.DictReader(l for l in open('gpurun_out/pool_ncu.csv') if not l.startswith('==')) if r.get('Metric Name')=='gpu__time_duration.sum']
v=sorted(float(r['Metric Value'].replace(',','')) for r in rows)
print('pool_kernel launches', len(v), 'median', v[len(v)//2], rows[0]['Metric Unit'] if rows else '', 'min', v[0], 'max', v[-1])
PY
