set -x
timeout 600 python tools/e2e_probe.py --n 40 > gpurun_out/r2h_e2e_probe.json 2> gpurun_out/r2h_e2e_probe.err
echo "probe rc=$?"; cat gpurun_out/r2h_e2e_probe.json; tail -3 gpurun_out/r2h_e2e_probe.err
timeout 900 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu --no-sweep > gpurun_out/r2h_bench_config2.json 2> gpurun_out/r2h_bench_config2.err
echo "cfg2 rc=$?"; tail -c 400 gpurun_out/r2h_bench_config2.json
timeout 900 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu --no-sweep > gpurun_out/r2h_bench_config3.json 2> gpurun_out/r2h_bench_config3.err
echo "cfg3 rc=$?"; tail -c 400 gpurun_out/r2h_bench_config3.json
