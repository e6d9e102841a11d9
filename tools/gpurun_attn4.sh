set -x
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -p no:cacheprovider -k "attention" -x > gpurun_out/attn_tests4.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/attn_tests4.log
timeout 900 python tools/attn_bwd_ab.py --variants 2,4,2,4 --shapes 4096:24:8,4096:4:1,4096:64:8,1000:8:2 > gpurun_out/attn_ab4.log 2>&1
echo "ab rc=$?"; grep -v "^{" gpurun_out/attn_ab4.log
timeout 300 python tools/attn_bwd_ab.py --variants 3,4 --shapes 2048:16:16:64 > gpurun_out/attn_ab4_64.log 2>&1; grep -v "^{" gpurun_out/attn_ab4_64.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_bwd_d -s 2 -c 2 \
  -o gpurun_out/attn_bwd_split -f python tools/attn_bwd_ab.py --child 4096:24:8 --reps 2 > gpurun_out/ncu_attn4.log 2>&1
echo "ncu rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 -x > gpurun_out/attn4_gputest.log 2>&1
echo "gpu tests rc=$?"; tail -3 gpurun_out/attn4_gputest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-sweep > gpurun_out/bench_attn4.json 2> gpurun_out/bench_attn4.err
echo "bench rc=$?"
