# config 1 iteration-level sets again from the committed 2 s-window tables (--resume: replayed, nothing re-profiled),
# now with the set that keeps the measured default among each partition's candidates
set -x
timeout 1500 python tools/mbo_hardware.py --config 1 --window 2.0 --warmup 0.3 --repeat 3 --trials 5 \
  --iter-window 2.0 --table-dir profiles/tables --tag r2w2 --resume --out gpurun_out/r2x_mbo_config1.json \
  > gpurun_out/r2x_mbo.log 2>&1
echo "mbo rc=$?"; tail -16 gpurun_out/r2x_mbo.log
