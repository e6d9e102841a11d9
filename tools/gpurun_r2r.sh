# attention backward hybrid grid (first key tiles one CTA per q head): same-box A/B, tests, in-step effect
set -x
timeout 900 python tools/attn_bwd_ab.py --variants 2+h0,2,2+h2,2+h6,2+h0,2 --shapes 4096:24:8,4096:64:8 > gpurun_out/r2r_ab.log 2>&1
echo "ab rc=$?"; grep -v "^{" gpurun_out/r2r_ab.log
timeout 900 python -m pytest tests/test_kernels_gpu.py -m gpu -q -p no:cacheprovider -k "attention" > gpurun_out/r2r_test.log 2>&1
echo "test rc=$?"; tail -3 gpurun_out/r2r_test.log
for h in 0 auto 0 auto; do
  if [ $h = auto ]; then unset KPO_ATTN_BWD_HYBRID; else export KPO_ATTN_BWD_HYBRID=$h; fi
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-sweep > gpurun_out/r2r_bench_h$h.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/r2r_bench_h$h.json')); r=d['roofline']
print('h=$h', d['ms_per_step'], d['sustained']['ms_per_step'], r['kernel'], r['avg_launch_ms'], r['frac'], json.dumps(r['solo']))"
done
unset KPO_ATTN_BWD_HYBRID
