# full round check: gpu tests, default bench (MBO frontier, microbatch, CPU baseline), reference arm,
# smoke() under the ncu launch list (the launch gate must survive the profiler), protocol sweep (20 trials)
set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 -rf > gpurun_out/r2b_gputest.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/r2b_gputest.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
echo "bench rc=$?"; tail -c 1500 gpurun_out/r2b_bench.json; tail -5 gpurun_out/r2b_bench.err
/usr/bin/time -v timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2b_ref.json 2> gpurun_out/r2b_ref.err
echo "ref rc=$?"; cat gpurun_out/r2b_ref.json; grep -i "elapsed" gpurun_out/r2b_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_smoke_launches.csv \
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke_ncu.log 2>&1
echo "ncu smoke rc=$?"; tail -3 gpurun_out/r2b_smoke_ncu.log
timeout 1500 python tools/protocol_sweep.py --trials 20 --out gpurun_out/r2b_protocol_sweep.json > gpurun_out/r2b_protocol.log 2>&1
echo "sweep rc=$?"; tail -5 gpurun_out/r2b_protocol.log
