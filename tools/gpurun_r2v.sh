# config 2 (TP8) iteration-level sets again from the committed tables (--resume replays them bit-exactly,
# nothing re-profiled), with the set that adds the measured default to each partition's candidates
set -x
timeout 1500 python tools/mbo_hardware.py --config 2 --window 1.0 --warmup 0.3 --repeat 3 --trials 5 \
  --iter-window 2.0 --table-dir profiles/tables --tag r2w1 --resume --out gpurun_out/r2v_mbo_config2.json \
  > gpurun_out/r2v_mbo.log 2>&1
echo "mbo rc=$?"; tail -16 gpurun_out/r2v_mbo.log
