set -x
KPO_ATTN_FWD=3 timeout 600 python -m pytest tests/test_kernels_gpu.py -q -p no:cacheprovider -k "attention" -x --timeout 240 > gpurun_out/r2g_attn_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/r2g_attn_tests.log
timeout 600 python tools/attn_bwd_ab.py --variants 2+f2,2+f3,2+f2,2+f3 --shapes 4096:24:8,4096:4:1,4096:64:8,2048:16:16:64 > gpurun_out/r2g_ab.log 2>&1
echo "ab rc=$?"; grep -v "^{" gpurun_out/r2g_ab.log
KPO_ATTN_FWD=3 timeout 300 ncu --set full --import-source on --clock-control none -k regex:attn_fwd_tc3 -s 3 -c 1 \
  -o gpurun_out/attn_fwd_tc3 -f python tools/attn_bwd_ab.py --child 4096:24:8 --reps 2 > gpurun_out/r2g_ncu.log 2>&1
echo "ncu rc=$?"
