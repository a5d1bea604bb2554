# step kernels (divergence, correction, diffusion, advection): parity tests, then an ncu launch list
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_box.py tests/test_gpu_physics_ext.py tests/test_gpu_dist.py -x -q -m gpu -k "diverg or correct or step or cavity or box or physics or slab or advect or diffus" 2>&1 | tail -4
CF_CG_DIRECT=2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"divergence|correct|diffuse|advect" --csv --log-file gpurun_out/stepk.csv python tools/ncu_table.py 256 step > gpurun_out/stepk.log 2>&1; echo ncu=$?
python - <<'PY'
import csv, io, collections
t = open('gpurun_out/stepk.csv').read()
rows = list(csv.DictReader(io.StringIO(t[t.index('"ID"'):])))
agg = collections.defaultdict(lambda: collections.defaultdict(float)); cnt = collections.Counter()
for r in rows:
    k = r['Kernel Name'].split('(')[0]
    agg[k][r['Metric Name']] += float(r['Metric Value'].replace(',', ''))
    if r['Metric Name'].startswith('gpu__time'): cnt[k] += 1; unit = r['Metric Unit']
for k, m in agg.items():
    n = cnt[k]
    print(k, n, 'launches avg', round(m['gpu__time_duration.sum'] / n / (1000 if unit in ('ns', 'nsecond') else 1), 1), 'us')
PY
