"""The reference optimizer on hardware, every partition of a layer (north_star).

For each partition of the BASELINE workload, the UNMODIFIED reference `schedfront.mbo.run_mbo`
(mbo.py:269-340, baseline/_ref) drives real executions through `Engine.measure` (installed over
`schedfront.mbo.measure`, engine.install) with the validated profiling protocol.  Its search space
is the reference's own `enumerate_space` over the engine's frequency grid (the frequencies this GPU
can honour: profiles/r2_clock_probe.json) x `SmGrid.default_for_group(8)` x launch timings.

Per partition this writes a profile table (profiler.ProfileTable; replayed bit-exactly through the
reference optimizer afterwards) and the MBO frontier.  Frontier points are then re-measured
`--repeat` times for their spread.  From the per-partition frontiers three iteration-level
schedule sets are selected -- min-time, min-energy, and iso-time (per partition the lowest-energy
frontier point no slower than the default schedule) -- and executed as WHOLE iterations next to the
default nanobatching schedule (f_max, default comm CTAs, overlap(0,n)) and the sequential (Megatron)
schedule: `--trials` interleaved rounds of >= `--iter-window` s each, device time + NVML energy.

python tools/mbo_hardware.py --config 1 --window 1.0 --out profiles/r2_mbo_config1.json"""
import argparse
import json
import math
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
REF = os.path.join(ROOT, "baseline", "_ref")
if REF not in sys.path:
    sys.path.append(REF)


def ci95(xs):
    if len(xs) < 2:
        return 0.0
    return 1.96 * statistics.stdev(xs) / math.sqrt(len(xs))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--tokens", type=int, default=None)
    ap.add_argument("--warmup", type=float, default=0.3)
    ap.add_argument("--window", type=float, default=1.0)
    ap.add_argument("--cooldown", type=float, default=0.0)
    ap.add_argument("--cooldown-target", type=float, default=None, help="also wait until the GPU is below this C")
    ap.add_argument("--partitions", default="")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--repeat", type=int, default=3, help="re-measurements of every frontier point")
    ap.add_argument("--trials", type=int, default=5, help="interleaved whole-iteration rounds per schedule set")
    ap.add_argument("--iter-window", type=float, default=2.0)
    ap.add_argument("--table-dir", default="profiles/tables")
    ap.add_argument("--tag", default="r2")
    ap.add_argument("--out", default="gpurun_out/mbo_hardware.json")
    ap.add_argument("--resume", action="store_true", help="reuse rows of existing tables in --table-dir")
    a = ap.parse_args()

    import torch
    import schedfront
    from schedfront import mbo
    from schedfront.domain import FrequencyGrid, SmGrid
    from schedfront.simgpu import ProfilingProtocol, ThermalModel, ThermalState

    from paper_2601_17654_b200.comm import Communicator
    from paper_2601_17654_b200.compat import patch_reference
    from paper_2601_17654_b200.device import b200_model_measured as b200_model
    from paper_2601_17654_b200.domain import LaunchTiming, ScheduleConfig
    from paper_2601_17654_b200.engine import Engine, install
    from paper_2601_17654_b200.layer import PartitionedLayer, sym_bytes_for
    from paper_2601_17654_b200.model import baseline_workload
    from paper_2601_17654_b200.profiler import ProfileTable, gpu_header, observation_dict
    from paper_2601_17654_b200.runner import LayerRunner, default_schedule, sequential_schedule

    dev = torch.device("cuda", 0)
    wl = baseline_workload(a.config, tokens=a.tokens)
    comm = Communicator.loopback_group(wl.world, sym_bytes_for(wl), device=dev)
    layer = PartitionedLayer(wl, comm)
    gpu = b200_model()
    eng = Engine.for_layer(layer, gpu, clock_control=True, cooldown_target_c=a.cooldown_target)
    restore = install(eng, schedfront)
    Meas = schedfront.domain.Measurement
    fgrid = FrequencyGrid(tuple(sorted(eng.frequencies(gpu))))
    sgrid = SmGrid.default_for_group(wl.world)
    proto = ProfilingProtocol(warmup_s=a.warmup, window_s=a.window, cooldown_s=a.cooldown)
    thermal = ThermalModel()
    names = a.partitions.split(",") if a.partitions else list(layer.order)
    out = {"workload": wl.tag, "protocol": {"warmup_s": a.warmup, "window_s": a.window, "cooldown_s": a.cooldown,
                                            "cooldown_target_c": a.cooldown_target},
           "freq_grid": list(fgrid.values), "sm_grid": list(sgrid.values), "clock_control": eng.freq.reason,
           "optimizer": "schedfront.mbo.run_mbo (reference, unmodified; baseline/_ref)", "partitions": {}}
    os.makedirs(a.table_dir, exist_ok=True)
    t_all = time.perf_counter()
    frontiers = {}
    for name in names:
        part = layer.programs[name].spec()
        hyper = mbo.MboHyperparams.for_partition(part, seed=a.seed)
        table = ProfileTable(name, {"gpu": gpu_header(gpu), "workload": wl.tag, "freq_grid": list(fgrid.values),
                                    "sm_grid": list(sgrid.values), "protocol": out["protocol"], "seed": a.seed,
                                    "hyper": {"n_init": hyper.n_init, "b_max": hyper.b_max, "batch_k": hyper.batch_k}})
        orig = eng.measure
        path = os.path.join(a.table_dir, f"{a.tag}_{wl.tag}_{name}.jsonl")
        prior = None
        if a.resume and os.path.exists(path):
            # a table from an interrupted run: its rows answer the optimizer's requests (the replay is
            # bit-exact, so the run continues exactly where the measurements left off); only
            # configurations missing from it are measured
            prior = ProfileTable.read(path)
            prior_eval = prior.evaluator(Meas)

        def recording(partition, config, gpu_, thermal_, protocol_, state_, table=table, prior=prior):
            if prior is not None and config in prior:
                table.add(config, prior_eval(partition, config), prior.lookup(config).obs)
                return prior_eval(partition, config)
            m = orig(partition, config, gpu_, thermal_, protocol_, state_)
            table.add(config, m, observation_dict(eng.last))
            return m

        mbo.measure = recording
        t0 = time.perf_counter()
        state = ThermalState.new(thermal, proto)
        res = mbo.run_mbo(part, gpu, thermal, proto, hyper, fgrid, sgrid)
        wall = time.perf_counter() - t0
        mbo.measure = orig
        space = mbo.enumerate_space(part, gpu, fgrid, sgrid)
        table.write(path)
        # replay: the table alone reproduces the optimizer's records bit-exactly
        ev = ProfileTable.read(path).evaluator(Meas)
        r2 = patch_reference(measure=lambda p, c, *x: ev(p, c), schedfront_module=schedfront)
        try:
            res2 = mbo.run_mbo(part, gpu, thermal, proto, hyper, fgrid, sgrid)
        finally:
            r2()
        install(eng, schedfront)
        replay_ok = [(r.config, r.measurement) for r in res.records] == [(r.config, r.measurement) for r in res2.records]
        # frontier points re-measured for their spread
        fr = []
        pts, seen_cfg = [], set()
        # the optimizer's (time, dynamic energy) frontier plus its (time, total energy) view
        for pt in list(res.frontier) + list(res.total_energy_frontier()):
            if pt.payload not in seen_cfg:
                seen_cfg.add(pt.payload)
                pts.append(pt.payload)
        for cfg in pts:
            ts, es = [], []
            for _ in range(a.repeat):
                m = eng.measure(part, cfg, gpu, thermal, proto, None)
                ts.append(m.time_ms)
                es.append(m.total_energy_j)
            row = table.lookup(cfg)
            fr.append({"config": f"{cfg.timing.encode()}@{cfg.sm_alloc}@{cfg.frequency_mhz:g}",
                       "time_ms": row.time_ms, "total_j": row.total_energy_j, "dyn_j": row.dyn_energy_j,
                       "repeat_time_ms": [statistics.mean(ts), ci95(ts)], "repeat_total_j": [statistics.mean(es), ci95(es)],
                       "flags": row.obs.get("flags", [])})
        frontiers[name] = [(ScheduleConfig(float(f["config"].split("@")[2]), int(f["config"].split("@")[1]),
                                           LaunchTiming.decode(f["config"].split("@")[0])), f) for f in fr]
        passes = mbo.frontier_pass_attribution(res)
        dyn_same_work = [r.dyn_energy_j for r in table.rows]
        out["partitions"][name] = {"space": len(space), "evals": len(res.records), "wall_s": round(wall, 1),
                                   "table": os.path.relpath(path, ROOT), "replay_bitexact": replay_ok,
                                   "frontier": fr, "frontier_pass_attribution": passes,
                                   "batches_run": res.batches_run, "stopped_early": res.stopped_early,
                                   "hv_history": [round(h, 6) for h in getattr(res, "hv_history", [])],
                                   "dyn_j_median_all": statistics.median(dyn_same_work),
                                   "dyn_j_spread_all": [min(dyn_same_work), max(dyn_same_work)],
                                   "flagged_rows": sum(1 for r in table.rows
                                                       if [f for f in r.obs.get("flags", []) if f != "power_capped"])}
        print(f"{name}: space {len(space)} evals {len(res.records)} frontier {len(fr)} {wall:.0f}s "
              f"replay {replay_ok}", flush=True)
        json.dump(out, open(a.out, "w"), indent=1)
    restore()
    out["mbo_wall_s"] = round(time.perf_counter() - t_all, 1)

    # ---------------------------------------------------------------- iteration-level schedule sets
    if set(names) == set(layer.order):
        dflt = default_schedule(layer, gpu)
        dflt_meas = {}
        for n_ in layer.order:
            m = eng.measure(layer.programs[n_].spec(), dflt[n_], gpu, thermal, proto, None)
            dflt_meas[n_] = (m.time_ms, m.total_energy_j)
        sets = {"nanobatching_default": dflt, "sequential_megatron": sequential_schedule(layer, gpu)}
        pick = {"mbo_min_time": lambda pts, n_: min(pts, key=lambda p: p[1]["repeat_time_ms"][0]),
                "mbo_min_energy": lambda pts, n_: min(pts, key=lambda p: p[1]["repeat_total_j"][0]),
                "mbo_iso_time": lambda pts, n_: min(
                    [p for p in pts if p[1]["repeat_time_ms"][0] <= dflt_meas[n_][0]] or
                    [min(pts, key=lambda p: p[1]["repeat_time_ms"][0])], key=lambda p: p[1]["repeat_total_j"][0])}
        for label, fn in pick.items():
            sets[label] = {n_: fn(frontiers[n_], n_)[0] for n_ in layer.order}
        # the reference's pruning can leave the default schedule out of a partition's space (TP8 forward
        # attention: the space is the single sequential candidate, 75% slower than the default overlap);
        # this set adds the measured default to every partition's candidates before the iso-time pick
        with_dflt = {n_: list(frontiers[n_]) + [(dflt[n_], {"repeat_time_ms": [dflt_meas[n_][0]],
                                                           "repeat_total_j": [dflt_meas[n_][1]]})]
                     for n_ in layer.order}
        sets["mbo_iso_time_with_default"] = {n_: pick["mbo_iso_time"](with_dflt[n_], n_)[0] for n_ in layer.order}
        out["default_partition_measurements"] = {n_: {"time_ms": v[0], "total_j": v[1]} for n_, v in dflt_meas.items()}
        out["sets"] = {k: {n_: f"{c.timing.encode()}@{c.sm_alloc}@{c.frequency_mhz:g}" for n_, c in s.items()}
                       for k, s in sets.items()}
        runners = {k: LayerRunner(layer, eng, schedule=s) for k, s in sets.items()}
        for r in runners.values():
            r.warm()
        # per-iteration estimate for the window length
        r0 = runners["nanobatching_default"]
        for _ in range(3):
            r0.step()
        torch.cuda.synchronize()
        q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        q0.record(eng.exec.compute)
        for _ in range(10):
            r0.step()
        q1.record(eng.exec.compute)
        q1.synchronize()
        it_ms = q0.elapsed_time(q1) / 10
        n_it = max(20, int(math.ceil(a.iter_window / (it_ms / 1e3))))
        res_it = {k: {"s_per_iter": [], "j_per_iter": [], "sm_mhz": [], "flags": []} for k in sets}
        for trial in range(a.trials):
            for k, r in runners.items():
                for _ in range(3):
                    r.step()
                torch.cuda.synchronize()
                w0 = time.perf_counter()
                q0.record(eng.exec.compute)
                for _ in range(n_it):
                    r.step()
                q1.record(eng.exec.compute)
                q1.synchronize()
                w1 = time.perf_counter()
                t_it = q0.elapsed_time(q1) / n_it / 1e3
                e_it = (eng.sampler.window_j(w0, w1) - max(0.0, (w1 - w0) - t_it * n_it) * gpu.p_static_w) / n_it
                clk = eng.sampler.clocks_summary(w0, w1)
                res_it[k]["s_per_iter"].append(t_it)
                res_it[k]["j_per_iter"].append(e_it)
                res_it[k]["sm_mhz"].append(clk.get("sm_mhz"))
                res_it[k]["flags"].append(clk.get("reasons", []))
                if a.cooldown > 0:
                    time.sleep(a.cooldown)
        summ = {}
        for k, v in res_it.items():
            summ[k] = {"s_per_iter": statistics.mean(v["s_per_iter"]), "s_ci95": ci95(v["s_per_iter"]),
                       "j_per_iter": statistics.mean(v["j_per_iter"]), "j_ci95": ci95(v["j_per_iter"]),
                       "trials": v, "iterations_per_trial": n_it}
        d = summ["nanobatching_default"]
        for k, v in summ.items():
            v["time_vs_default"] = v["s_per_iter"] / d["s_per_iter"] - 1
            v["energy_vs_default"] = v["j_per_iter"] / d["j_per_iter"] - 1
        out["executed"] = summ
        for k, v in summ.items():
            print(f"{k:22s} {v['s_per_iter']*1e3:8.4f} ms +- {v['s_ci95']*1e3:.4f}  {v['j_per_iter']:8.4f} J "
                  f"+- {v['j_ci95']:.4f}  dt {v['time_vs_default']*100:+.2f}% dE {v['energy_vs_default']*100:+.2f}%")
    json.dump(out, open(a.out, "w"), indent=1)
    eng.close()
    comm.close()


if __name__ == "__main__":
    main()
