# attention-backward kernel: correctness, same-box A/B vs the 64-query kernel, peers, one ncu capture
set -x
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -p no:cacheprovider -k "attention" -x > gpurun_out/attn_tests.log 2>&1
echo "tests rc=$?"; tail -5 gpurun_out/attn_tests.log
timeout 900 python tools/attn_bwd_ab.py --variants 2,3 --shapes 4096:24:8,4096:4:1,4096:64:8,1000:8:2 > gpurun_out/attn_ab.log 2>&1
echo "ab rc=$?"; tail -3 gpurun_out/attn_ab.log
timeout 300 python tools/attn_bwd_ab.py --variants 1,3 --shapes 2048:16:16:64 > gpurun_out/attn_ab64.log 2>&1; tail -2 gpurun_out/attn_ab64.log
timeout 900 python tools/attn_ablate.py --modes 0 > gpurun_out/attn_peers.log 2>&1; tail -1 gpurun_out/attn_peers.log
KPO_ATTN_BWD=3 timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_bwd_tc3 -s 3 -c 1 \
  -o gpurun_out/attn_bwd_tc3 -f python tools/attn_bwd_ab.py --child 4096:24:8 --reps 2 > gpurun_out/ncu_attn.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_attn.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-sweep > gpurun_out/bench_attn3.json 2> gpurun_out/bench_attn3.err
echo "bench rc=$?"; tail -c 600 gpurun_out/bench_attn3.json
