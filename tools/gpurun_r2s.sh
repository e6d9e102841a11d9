# same-box A/B: mbarrier watchdog on (current) vs off (-DKPO_NO_MBAR_WATCHDOG), and the builds at the r2 ncu
# capture (b62ffe9) and after the paired-fp32 softmax (628af3b); attention fwd + bwd, then the layer GEMMs
set -x
timeout 900 python tools/attn_bwd_ab.py --variants 2@nowd,2,2@628af3b,2@b62ffe9,2@nowd,2,2@628af3b,2@b62ffe9 --shapes 4096:24:8,4096:64:8 > gpurun_out/r2s_ab.log 2>&1
echo "ab rc=$?"; grep -v "^{" gpurun_out/r2s_ab.log
for v in cur nowd cur nowd; do
  if [ $v = nowd ]; then export KPO_LIB_PATH=$PWD/tools/ab/libkpo_nowd.so; else unset KPO_LIB_PATH; fi
  timeout 300 python tools/gemm_bench.py --config 1 > gpurun_out/r2s_gemm_$v.log 2>&1
  echo "gemm $v"; tail -3 gpurun_out/r2s_gemm_$v.log
done
unset KPO_LIB_PATH
