"""Hardware validation of the thermally-stable profiling protocol (reference cli.py:552-605
`thermal_window_sweep` / `thermal_cooldown_sweep`, protocol PAPER.md:700-708, cooling
simgpu.py:311-318), run against the real `Engine.measure` instead of the simulator.

  window sweep    10 trials x windows {0.3, 1, 2, 5} s of one partition: the spread (std and CV)
                  of the measured energy per execution must be non-increasing with the window
                  (reference criterion: each std <= 1.15x the previous, last <= 0.6x the first).
  cooldown sweep  a heater window (the heaviest partition for 5 s), then the target partition after
                  cooldowns {0, 1, 2, 5} s and after a temperature target (idle + 3 C): the mean
                  energy must stop changing (reference: plateau within 2e-3 -- here judged against
                  the window sweep's measured spread, since real counters are noisier).
Every sample records the median SM clock, throttle reasons and GPU temperature; samples that saw a
hardware/thermal slowdown are flagged (engine.BAD_REASONS).

python tools/protocol_sweep.py [--config 1] [--partition fwd_mlp0] [--trials 10]
Writes gpurun_out/protocol_sweep.json."""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--partition", default="fwd_mlp0")
    ap.add_argument("--heater", default="bwd_mlp0")
    ap.add_argument("--trials", type=int, default=10)
    ap.add_argument("--windows", default="0.3,1,2,5")
    ap.add_argument("--cooldowns", default="0,1,2,5")
    ap.add_argument("--cool-trials", type=int, default=5)
    ap.add_argument("--out", default="gpurun_out/protocol_sweep.json")
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
    eng = Engine.for_layer(L, gpu, clock_control=True)
    prog = L.programs[a.partition]
    n = len(prog.units)
    cfg = ScheduleConfig(gpu.f_max_mhz, 16, LaunchTiming.overlap(0, n))
    heat = L.programs[a.heater]
    hcfg = ScheduleConfig(gpu.f_max_mhz, 16, LaunchTiming.overlap(0, len(heat.units)))
    out = {"workload": wl.tag, "partition": a.partition, "config": cfg.encode() if hasattr(cfg, "encode")
           else f"{cfg.timing.encode()}@{cfg.sm_alloc}", "heater": a.heater,
           "clock_control": eng.freq.reason, "p_static_w": gpu.p_static_w}
    time.sleep(5.0)
    out["idle_temperature_c"] = eng.nvml.temperature_c()

    def sample(prog_, cfg_, warm, win, cool):
        t_ms, e_j, temp = eng.measure_local(prog_.name, cfg_, warm, win, cool)
        o = eng.last
        return {"time_ms": t_ms, "energy_j": e_j, "dyn_j": e_j - gpu.p_static_w * t_ms / 1e3, "reps": o.reps,
                "window_s": round(o.window_s, 4), "sm_mhz": o.sm_mhz, "temp_start_c": o.temperature_start_c,
                "temp_end_c": temp, "flags": list(o.flags), "retried": o.retried}

    # ---------------------------------------------------------------- window sweep
    windows = [float(x) for x in a.windows.split(",")]
    ws = []
    for w in windows:
        rows = [sample(prog, cfg, 0.5, w, 1.0) for _ in range(a.trials)]
        es = [r["energy_j"] for r in rows]
        ts = [r["time_ms"] for r in rows]
        ws.append({"window_s": w, "energy_mean_j": statistics.mean(es), "energy_std_j": statistics.stdev(es),
                   "energy_cv": statistics.stdev(es) / statistics.mean(es), "time_mean_ms": statistics.mean(ts),
                   "time_cv": statistics.stdev(ts) / statistics.mean(ts),
                   "sm_mhz_median": statistics.median(r["sm_mhz"] for r in rows),
                   "flagged": sum(1 for r in rows if r["flags"] and r["flags"] != ["power_capped"]),
                   "power_capped": sum(1 for r in rows if "power_capped" in r["flags"]), "trials": rows})
        print(f"window {w}: E {ws[-1]['energy_mean_j']:.5f} J cv {ws[-1]['energy_cv']:.4f}  "
              f"t {ws[-1]['time_mean_ms']:.4f} ms cv {ws[-1]['time_cv']:.4f}", flush=True)
    stds = [r["energy_std_j"] for r in ws]
    out["window_sweep"] = {"rows": ws, "energy_std": stds,
                           "nonincreasing": all(b <= x * 1.15 for x, b in zip(stds, stds[1:])),
                           "trend": stds[-1] <= 0.6 * stds[0]}
    out["window_sweep"]["passed"] = out["window_sweep"]["nonincreasing"] and out["window_sweep"]["trend"]

    # ---------------------------------------------------------------- cooldown sweep
    cools = [float(x) for x in a.cooldowns.split(",")]
    target_c = out["idle_temperature_c"] + 3.0
    cs = []
    for c in cools + ["target"]:
        rows = []
        for _ in range(a.cool_trials):
            sample(heat, hcfg, 0.5, 5.0, 0.0)  # heater
            if c == "target":
                eng.cooldown_target_c = target_c
                t0 = time.perf_counter()
                eng._cooldown(0.0)
                waited = time.perf_counter() - t0
                eng.cooldown_target_c = None
            else:
                time.sleep(c)
                waited = c
            r = sample(prog, cfg, 0.2, 2.0, 0.0)
            r["cooldown_s"] = round(waited, 3)
            rows.append(r)
        es = [r["energy_j"] for r in rows]
        cs.append({"cooldown": c, "energy_mean_j": statistics.mean(es), "energy_std_j": statistics.stdev(es),
                   "temp_start_mean_c": statistics.mean(r["temp_start_c"] for r in rows),
                   "cooldown_mean_s": statistics.mean(r["cooldown_s"] for r in rows), "trials": rows})
        print(f"cooldown {c}: E {cs[-1]['energy_mean_j']:.5f} J (std {cs[-1]['energy_std_j']:.5f}) "
              f"T0 {cs[-1]['temp_start_mean_c']:.1f} C", flush=True)
    means = [r["energy_mean_j"] for r in cs]
    std2 = next((r["energy_std_j"] for r in ws if r["window_s"] == 2.0), stds[-1])
    out["cooldown_sweep"] = {"rows": cs, "energy_mean": means, "target_c": target_c,
                             "max_abs_dev_vs_target_j": max(abs(m - means[-1]) for m in means),
                             "window2_std_j": std2}
    out["cooldown_sweep"]["plateau_within_spread"] = abs(means[-2] - means[-1]) <= 2 * std2 / (a.cool_trials ** 0.5) * 2
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps({"window_sweep_passed": out["window_sweep"]["passed"], "stds": stds, "cool_means": means}))
    eng.close()
    comm.close()


if __name__ == "__main__":
    main()
