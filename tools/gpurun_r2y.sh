# the driver's default bench invocation on the final commit
set -x
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r2y_bench.json 2> gpurun_out/r2y_bench.err
echo "bench rc=$?"; tail -c 300 gpurun_out/r2y_bench.err
