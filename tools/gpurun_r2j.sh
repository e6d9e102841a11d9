set -x
timeout 600 python tools/e2e_probe.py --n 200 > gpurun_out/r2j_e2e_probe.json 2> gpurun_out/r2j_e2e_probe.err
echo "probe rc=$?"; cat gpurun_out/r2j_e2e_probe.json; tail -3 gpurun_out/r2j_e2e_probe.err
