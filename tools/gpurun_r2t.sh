# final code (mbarrier watchdog off in the product build): GPU tests, smoke, default bench line, ncu of the step
set -x
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2t_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 -rf > gpurun_out/r2t_gputest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r2t_gputest.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r2t_bench.json 2> gpurun_out/r2t_bench.err
echo "bench rc=$?"; tail -c 300 gpurun_out/r2t_bench.json
timeout 900 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu --no-sweep > gpurun_out/r2t_bench_config2.json 2> gpurun_out/r2t_bench_config2.err
echo "cfg2 rc=$?"
timeout 1200 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu > gpurun_out/r2t_bench_config3.json 2> gpurun_out/r2t_bench_config3.err
echo "cfg3 rc=$?"
bash tools/profile_round.sh r2t > gpurun_out/r2t_profile.log 2>&1
echo "profile rc=$?"
