#!/bin/bash
# One gpurun call: the step's ncu launch list plus --set full captures of the step's main kernels.
# usage: bash tools/profile_round.sh <tag>   (outputs under gpurun_out/)
tag=${1:-r}
only=${2:-}
out=gpurun_out
NCU="ncu --clock-control none --profile-from-start off"
[ -z "$only" ] && timeout 300 $NCU --metrics gpu__time_duration.sum --csv --log-file $out/launches_$tag.csv \
  python tools/profile_step.py > $out/launches_$tag.log 2>&1
cap() {  # name regex
  [ -n "$only" ] && [[ "$1" != $only* ]] && return
  timeout 400 $NCU --set full --import-source on --kernel-name-base demangled -k "regex:$2" -c 1 \
    -o $out/full_${tag}_$1 -f python tools/profile_step.py > $out/full_${tag}_$1.log 2>&1
}
cap attn_bwd_tc 'attn_bwd_tc_kernel'
cap attn_fwd_tc2 'attn_fwd_tc2_kernel'
cap gemm2_swiglu 'gemm2_kernel<\(int\)256, \(bool\)0, \(bool\)0, \(int\)1>'
cap gemm2_swiglu_bwd 'gemm2_kernel<\(int\)256, \(bool\)0, \(bool\)1, \(int\)2>'
cap gemm2_wgrad 'gemm2_kernel<\(int\)256, \(bool\)1, \(bool\)1, \(int\)0>'
cap rmsnorm_fwd 'rmsnorm_fwd_row'
cap rmsnorm_bwd 'rmsnorm_bwd_rows'
ls -la $out | tail -20
