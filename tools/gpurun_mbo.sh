# MBO on hardware, every partition of config 1; outputs merged back via gpurun_out/
set -x
mkdir -p gpurun_out/tables
timeout 5000 python tools/mbo_hardware.py --config 1 --window 1.0 --warmup 0.3 --repeat 3 --trials 5 \
  --iter-window 2.0 --table-dir gpurun_out/tables --tag r2 --out gpurun_out/r2_mbo_config1.json \
  > gpurun_out/r2_mbo.log 2>&1
echo "mbo rc=$?"
tail -20 gpurun_out/r2_mbo.log
