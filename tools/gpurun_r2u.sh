# the reference optimizer on hardware for config 2 (Llama-3-8B TP8: all-reduce overlapped with the nanobatched GEMMs)
set -x
mkdir -p gpurun_out/tables_u
timeout 2700 python tools/mbo_hardware.py --config 2 --window 1.0 --warmup 0.3 --repeat 3 --trials 5 \
  --iter-window 2.0 --table-dir gpurun_out/tables_u --tag r2w1 --resume --out gpurun_out/r2u_mbo_config2.json \
  > gpurun_out/r2u_mbo.log 2>&1
echo "mbo rc=$?"; tail -14 gpurun_out/r2u_mbo.log
