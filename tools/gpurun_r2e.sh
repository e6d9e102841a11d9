set -x
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -p no:cacheprovider -k "attention" -x > gpurun_out/r2e_attn_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/r2e_attn_tests.log
timeout 900 python tools/attn_bwd_ab.py --variants 2@base,2,2@base,2 --shapes 4096:24:8,4096:4:1,4096:64:8 > gpurun_out/r2e_ab.log 2>&1
echo "ab rc=$?"; grep -v "^{" gpurun_out/r2e_ab.log
timeout 1200 python tools/unit_sm_sweep.py --out gpurun_out/r2e_unit_sm_sweep.json > gpurun_out/r2e_sweep.log 2>&1
echo "sweep rc=$?"; tail -5 gpurun_out/r2e_sweep.log
