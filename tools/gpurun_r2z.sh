# final code: GPU tests, the default bench line, ncu launch list + --set full captures of the step's kernels
set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 -rf > gpurun_out/r2z_gputest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r2z_gputest.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r2z_bench.json 2> gpurun_out/r2z_bench.err
echo "bench rc=$?"; tail -c 300 gpurun_out/r2z_bench.json
bash tools/profile_round.sh r2z > gpurun_out/r2z_profile.log 2>&1
echo "profile rc=$?"
