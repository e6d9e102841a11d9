# the reference optimizer on hardware for config 3 (Llama-3-70B FSDP8: the BASELINE "full time-energy frontier" config)
set -x
mkdir -p gpurun_out/tables_o
timeout 5400 python tools/mbo_hardware.py --config 3 --window 2.0 --warmup 0.3 --repeat 3 --trials 5 \
  --iter-window 4.0 --table-dir gpurun_out/tables_o --tag r2w2 --out gpurun_out/r2o_mbo_config3.json \
  > gpurun_out/r2o_mbo.log 2>&1
echo "mbo rc=$?"; tail -14 gpurun_out/r2o_mbo.log
