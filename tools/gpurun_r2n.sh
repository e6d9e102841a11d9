# final round check on the committed code: GPU tests, default bench, TP8 bench line
set -x
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 -rf > gpurun_out/r2n_gputest.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/r2n_gputest.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r2n_bench.json 2> gpurun_out/r2n_bench.err
echo "bench rc=$?"; tail -c 600 gpurun_out/r2n_bench.json
timeout 900 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu --no-sweep > gpurun_out/r2n_bench_config2.json 2> gpurun_out/r2n_bench_config2.err
echo "cfg2 rc=$?"
