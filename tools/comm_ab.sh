for m in 0 1; do KPO_COMM_BULK=$m timeout 200 python tools/comm_bench.py --sizes-mb 16,32,64,128 --ctas 8,16,32 > gpurun_out/cb$m.json; done
python - <<'PY'
import json
a=json.load(open('gpurun_out/cb0.json'))['rows']; b=json.load(open('gpurun_out/cb1.json'))['rows']
for x,y in zip(a,b):
    if x['op']!='reduce_scatter': print(x['op'], x['bytes']>>20, 'MB', x['ncta'], 'lsu', x['busbw_gbs'], 'bulk', y['busbw_gbs'], 'MB/cta', round(x['bytes']/x['ncta']/2**20,2))
PY
