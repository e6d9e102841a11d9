# config 2 (TP8) bench line with its MBO sets executed (incl. the set with the default among the candidates)
set -x
timeout 900 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu > gpurun_out/r2w_bench_config2.json 2> gpurun_out/r2w_bench_config2.err
echo "cfg2 rc=$?"; tail -c 400 gpurun_out/r2w_bench_config2.err
