set -x
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 -rf > gpurun_out/r2d_gputest.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/r2d_gputest.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err
echo "bench rc=$?"; tail -c 800 gpurun_out/r2d_bench.json
