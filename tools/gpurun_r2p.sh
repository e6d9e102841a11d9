# the reference optimizer on hardware for config 3 (Llama-3-70B FSDP8: the BASELINE "full time-energy frontier" config),
# 1 s windows (protocol sweep: CV 1.2-2.2% at 1 s); --resume picks up tables a cut-off call left in tables_o
set -x
mkdir -p gpurun_out/tables_o
timeout 3300 python tools/mbo_hardware.py --config 3 --window 1.0 --warmup 0.3 --repeat 3 --trials 5 \
  --iter-window 3.0 --table-dir gpurun_out/tables_o --tag r2w1 --resume --out gpurun_out/r2p_mbo_config3.json \
  > gpurun_out/r2p_mbo.log 2>&1
echo "mbo rc=$?"; tail -14 gpurun_out/r2p_mbo.log
