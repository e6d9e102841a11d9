set -x
timeout 900 python tools/switch_sweep.py --out gpurun_out/r2k_switch_sweep.json > gpurun_out/r2k_switch.log 2>&1
echo "sweep rc=$?"; cat gpurun_out/r2k_switch.log | tail -5
