set -x
timeout 600 python tools/attn_bwd_ab.py --variants 2+f2,2+f1,2,2+f2,2+f1,2 --shapes 4096:4:1,4096:24:8,4096:64:8 > gpurun_out/r2m_ab.log 2>&1
echo "ab rc=$?"; grep -v "^{" gpurun_out/r2m_ab.log
