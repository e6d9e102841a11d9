set -x
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -p no:cacheprovider -k "attention" -x > gpurun_out/attn_tests3.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/attn_tests3.log
KPO_ATTN_BWD=3 timeout 900 python -m pytest tests/test_kernels_gpu.py -q -p no:cacheprovider -k "attention" -x > gpurun_out/attn_tests3v3.log 2>&1
echo "tests v3 rc=$?"; tail -3 gpurun_out/attn_tests3v3.log
timeout 900 python tools/attn_bwd_ab.py --variants 2,3,2,3 --shapes 4096:24:8,4096:4:1,4096:64:8 > gpurun_out/attn_ab3.log 2>&1
echo "ab rc=$?"; grep -v "^{" gpurun_out/attn_ab3.log
timeout 300 python tools/attn_bwd_ab.py --variants 1,3 --shapes 2048:16:16:64 > gpurun_out/attn_ab3_64.log 2>&1; grep -v "^{" gpurun_out/attn_ab3_64.log
KPO_ATTN_BWD=3 timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_bwd_tc3 -s 3 -c 1 \
  -o gpurun_out/attn_bwd_tc3c -f python tools/attn_bwd_ab.py --child 4096:24:8 --reps 2 > gpurun_out/ncu_attn3.log 2>&1
echo "ncu rc=$?"
