"""Does the profiling warm-up matter when consecutive measurements switch schedules (as the optimizer's
batches do)?  For each warm-up in --warmups: --trials rounds of [config A (a 3-CTA schedule: slow,
low power), then config B (the default-like schedule)], recording B's energy per execution with a
1 s window and no cooldown -- the protocol tools/mbo_hardware.py used.  Compared with the same-config
spread of tools/protocol_sweep.py, a larger spread at a short warm-up means the window still sees the
previous schedule's power state.
python tools/switch_sweep.py [--partition fwd_mlp0] --out gpurun_out/switch_sweep.json"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--partition", default="fwd_mlp0")
    ap.add_argument("--warmups", default="0.3,1.0,2.0")
    ap.add_argument("--window", type=float, default=1.0)
    ap.add_argument("--trials", type=int, default=10)
    ap.add_argument("--out", default="gpurun_out/switch_sweep.json")
    a = ap.parse_args()

    import torch

    from paper_2601_17654_b200.comm import Communicator
    from paper_2601_17654_b200.device import b200_model_measured as b200_model
    from paper_2601_17654_b200.domain import LaunchTiming, ScheduleConfig
    from paper_2601_17654_b200.engine import Engine
    from paper_2601_17654_b200.layer import PartitionedLayer, sym_bytes_for
    from paper_2601_17654_b200.model import baseline_workload

    dev = torch.device("cuda", 0)
    wl = baseline_workload(a.config)
    comm = Communicator.loopback_group(wl.world, sym_bytes_for(wl), device=dev)
    L = PartitionedLayer(wl, comm)
    gpu = b200_model()
    eng = Engine.for_layer(L, gpu, clock_control=False, energy_outlier_frac=None)
    prog = L.programs[a.partition]
    n = len(prog.units)
    cfg_a = ScheduleConfig(gpu.f_max_mhz, 3, LaunchTiming.overlap(0, 1))
    cfg_b = ScheduleConfig(gpu.f_max_mhz, 24, LaunchTiming.overlap(0, n))
    out = {"workload": wl.tag, "partition": a.partition, "window_s": a.window,
           "config_a": f"{cfg_a.timing.encode()}@{cfg_a.sm_alloc}", "config_b": f"{cfg_b.timing.encode()}@{cfg_b.sm_alloc}",
           "rows": []}
    for w in [float(x) for x in a.warmups.split(",")]:
        es, ts, pw = [], [], []
        for _ in range(a.trials):
            eng.measure_local(prog.name, cfg_a, w, a.window, 0.0)
            t_ms, e_j, _ = eng.measure_local(prog.name, cfg_b, w, a.window, 0.0)
            es.append(e_j)
            ts.append(t_ms)
            pw.append(e_j / (t_ms / 1e3))
        row = {"warmup_s": w, "energy_mean_j": statistics.mean(es), "energy_std_j": statistics.stdev(es),
               "energy_cv": statistics.stdev(es) / statistics.mean(es), "energy_range_j": [min(es), max(es)],
               "time_mean_ms": statistics.mean(ts), "power_w": [round(x, 1) for x in pw]}
        out["rows"].append(row)
        print(f"warmup {w}: E {row['energy_mean_j']:.5f} J cv {row['energy_cv']:.4f} range {row['energy_range_j']}",
              flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)
    eng.close()
    comm.close()


if __name__ == "__main__":
    main()
