# reference arm timing, smoke() under the ncu launch list, the step's ncu profile set, then MBO with
# the energy-outlier re-measurement
set -x
start=$(date +%s)
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2c_ref.json 2> gpurun_out/r2c_ref.err
echo "ref rc=$? wall $(( $(date +%s) - start )) s"; cat gpurun_out/r2c_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c_smoke_launches.csv \
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c_smoke_ncu.log 2>&1
echo "ncu smoke rc=$?"; grep -v "^==PROF==" gpurun_out/r2c_smoke_ncu.log | tail -3
bash tools/profile_round.sh r2 > gpurun_out/r2c_profile.log 2>&1
echo "profile rc=$?"
mkdir -p gpurun_out/tables_c
timeout 4000 python tools/mbo_hardware.py --config 1 --window 1.0 --warmup 0.3 --repeat 3 --trials 5 \
  --iter-window 2.0 --table-dir gpurun_out/tables_c --tag r2c --out gpurun_out/r2c_mbo_config1.json \
  > gpurun_out/r2c_mbo.log 2>&1
echo "mbo rc=$?"; tail -14 gpurun_out/r2c_mbo.log
