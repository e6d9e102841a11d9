# MBO on hardware with the 2 s windows of the validated protocol (0.6% energy CV, profiles/r2_protocol_sweep_20trials.json)
set -x
mkdir -p gpurun_out/tables_l
timeout 6000 python tools/mbo_hardware.py --config 1 --window 2.0 --warmup 0.3 --repeat 3 --trials 5 \
  --iter-window 2.0 --table-dir gpurun_out/tables_l --tag r2w2 --out gpurun_out/r2l_mbo_config1.json \
  > gpurun_out/r2l_mbo.log 2>&1
echo "mbo rc=$?"; tail -14 gpurun_out/r2l_mbo.log
