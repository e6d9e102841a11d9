#!/usr/bin/env python
"""bench.py — partitioned-overlap layer iteration on B200 (driver contract, one JSON line on rank 0).

Workload (BASELINE.json configs[1]): one Llama-3.2-3B transformer layer under FSDP, forward +
backward, 2 nanobatches x 4096 tokens per rank, executed as the 8 partitions of the Kareus
partitioned-overlap model (each: hand-written sm_100a compute kernels on the compute stream, an
SM-budgeted P2P collective on the comm stream).  A *step* = one such layer iteration under the
baseline nanobatching schedule (f_max, default comm CTAs, overlap(0, n)).

  N = 1: the 8-rank FSDP group runs in loopback (virtual peers' shards in local HBM; the kernels,
         CTA budget and barriers are the real ones, the link is HBM).
  N > 1: one process per GPU (torchrun), CUDA-IPC peer mapping, FSDP over N ranks; time = max over
         ranks, energy = sum over ranks, value = whole-job iteration time.

`--impl reference` times the reference-side CPU path (the oracle's fp32 execution of the same
layer iteration, oracle/layer_ref.py) on the host cores; see DESIGN.md §Measurement.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

UT_ITERS = 10  # iterations of per-unit in-step timing (graph replay with events around every unit)
METRIC = "iteration time (s) & energy (J/iter) Pareto frontier, 1-8 B200; comm bus GB/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="kpo", choices=["kpo", "reference"])
    ap.add_argument("--config", type=int, default=1, help="BASELINE.json configs index (1..3)")
    ap.add_argument("--tokens", type=int, default=None, help="tokens per nanobatch (default: the config's own, 4096 for configs 1-3)")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-iters", type=int, default=3, help="full CPU oracle iterations for cpu_baseline")
    ap.add_argument("--sweep-window", type=float, default=2.0, help="seconds per executed schedule-set trial")
    ap.add_argument("--sweep-trials", type=int, default=2)
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def iteration_flops(wl) -> float:
    """Algorithmic FLOPs of one layer iteration (fwd + bwd, all nanobatches) for one rank."""
    T, h, d, hq, hkv, f = wl.tokens, wl.h, wl.d, wl.hq, wl.hkv, wl.ffn
    gemm_fwd = 2.0 * T * h * (wl.qkv_dim + hq * d + 2 * f + f)
    attn_fwd = 2.0 * T * T * hq * d
    per_nb = 3 * gemm_fwd + attn_fwd * 3.5
    return per_nb * wl.nanobatches


# ---------------------------------------------------------------------------- CPU baseline
def host_facts() -> dict:
    """CPU facts BASELINE.md §3 asks for: lscpu model, os.cpu_count(), torch threads."""
    import subprocess

    import torch

    model = ""
    try:
        txt = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        model = next((ln.split(":", 1)[1].strip() for ln in txt.splitlines() if ln.startswith("Model name")), "")
    except Exception:
        pass
    return {"cpu_model": model, "cpu_count": os.cpu_count(), "torch_threads": torch.get_num_threads()}


def cpu_layer_setup(wl, nanobatches: int):
    """The oracle's inputs for `nanobatches` full nanobatches of the workload (fp32, seeded)."""
    import torch

    m = wl.model
    g = torch.Generator().manual_seed(0)
    W = {
        "wqkv": torch.randn((m.n_heads + 2 * m.n_kv_heads) * m.head_dim, m.hidden, generator=g) * 0.02,
        "wo": torch.randn(m.hidden, m.n_heads * m.head_dim, generator=g) * 0.02,
        "wgu": torch.randn(2 * m.ffn, m.hidden, generator=g) * 0.02,
        "wd": torch.randn(m.hidden, m.ffn, generator=g) * 0.02,
        "g1": torch.ones(m.hidden), "g2": torch.ones(m.hidden),
    }
    xs = [torch.randn(wl.tokens, m.hidden, generator=g) for _ in range(nanobatches)]
    dys = [torch.randn(wl.tokens, m.hidden, generator=g) for _ in range(nanobatches)]
    return W, xs, dys


def cpu_iteration(wl, threads: int, setup=None) -> float:
    """Seconds for the oracle's fp32 forward + backward of ONE FULL layer iteration of the workload
    (wl.nanobatches x wl.tokens tokens, the same shapes the GPU step runs; no scaling), all host
    threads."""
    import torch

    from oracle import layer_ref

    torch.set_num_threads(threads)
    W, xs, dys = setup or cpu_layer_setup(wl, wl.nanobatches)
    t0 = time.perf_counter()
    layer_ref.layer_fwd_bwd(xs, dys, W, wl.model)
    return time.perf_counter() - t0


def workload_config(wl, world: int, group_world: int) -> dict:
    """The `config` object both arms print (identical keys and values for the same workload)."""
    return {
        "workload": f"{wl.model.name} layer iteration: fwd+bwd, {wl.nanobatches} nanobatches x {wl.tokens} "
                    f"tokens per rank, 8 partitions",
        "model": wl.model.name, "global_batch": wl.tokens * wl.nanobatches * world, "seq_len": wl.tokens,
        "parallelism": (f"{wl.parallel}{group_world}-loopback" if world == 1 else f"{wl.parallel}{world}"),
        "schedule": "nanobatching default: f_max, default comm CTAs, overlap(0,n)",
        "l2": "no flush: per-step working set (layer weights + activations) > 126 MB L2",
    }


def reference_cpu_path(wl, with_mbo: bool = True) -> dict | None:
    """The reference's own CPU cost for the path this engine replaces, from the
    unmodified reference package in baseline/_ref, single-threaded as the reference runs it:
      (i)  simgpu.simulate_schedule and simgpu.measure over the full schedule space of every partition
           of this workload (projected to reference KernelSpecs, reference GpuModel defaults), per call;
      (ii) mbo.run_mbo replaying a profile table for one partition, per partition (sklearn surrogate)."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(ref) and ref not in sys.path:
        sys.path.append(ref)
    try:
        import schedfront
        from schedfront import domain, mbo, simgpu, workloads
    except ImportError:
        return None
    from paper_2601_17654_b200 import specs

    def to_ref(p):
        return domain.PartitionSpec(tuple(domain.KernelSpec(k.name, k.flops, k.bytes, k.comm_bytes)
                                          for k in p.comp_kernels),
                                    domain.KernelSpec(p.comm_kernel.name, comm_bytes=p.comm_kernel.comm_bytes),
                                    p.comm_group_size, p.name)

    gpu, thermal = workloads.default_gpu(), workloads.default_thermal()
    proto = simgpu.ProfilingProtocol(2.0, 5.0, 5.0, 0.02, 6.0, 1234)
    fg, sg = domain.FrequencyGrid.default(), domain.SmGrid.default_for_group(8)
    parts = [to_ref(p) for p in specs.partition_specs(wl)]
    n = 0
    t_sim = t_meas = 0.0
    tables = {}
    for part in parts:
        space = mbo.enumerate_space(part, gpu, fg, sg)
        state = simgpu.ThermalState.new(thermal, proto)
        t0 = time.perf_counter()
        for c in space:
            simgpu.simulate_schedule(part, c, gpu)
        t1 = time.perf_counter()
        table = {c: simgpu.measure(part, c, gpu, thermal, proto, state) for c in space}
        t2 = time.perf_counter()
        t_sim += t1 - t0
        t_meas += t2 - t1
        n += len(space)
        tables[part.name] = table
    out = {"simulate_schedule_us": round(t_sim / n * 1e6, 2), "measure_us": round(t_meas / n * 1e6, 2),
           "candidates": n, "partitions": len(parts), "cores": 1,
           "source": f"baseline/_ref schedfront {getattr(schedfront, '__version__', '')} (unmodified)".strip()}
    if with_mbo:
        part = parts[0]
        table = tables[part.name]
        orig = mbo.measure
        mbo.measure = lambda p, c, *a: table[c]
        try:
            t0 = time.perf_counter()
            r = mbo.run_mbo(part, gpu, thermal, proto, mbo.MboHyperparams.for_partition(part, 0), fg, sg)
            out["run_mbo_replay_s"] = round(time.perf_counter() - t0, 3)
            out["run_mbo_partition"] = part.name
            out["run_mbo_evals"] = len(r.records)
        finally:
            mbo.measure = orig
    return out


def run_reference(args):
    """The reference-side CPU path of this workload: the oracle's fp32 execution of the same layer
    iteration (every step = one full iteration, 2 nanobatches x 4096 tokens, nothing scaled), on all
    host threads of rank 0."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2601_17654_b200.model import baseline_workload

    wl = baseline_workload(args.config, world=8, tokens=args.tokens)
    group_world = wl.world if world == 1 else world
    threads = os.cpu_count() or 1
    setup = cpu_layer_setup(wl, wl.nanobatches)
    vals = []
    t_start = time.perf_counter()
    for i in range(args.warmup + args.steps):
        v = cpu_iteration(wl, threads, setup)
        if i >= args.warmup:
            vals.append(v)
    total = time.perf_counter() - t_start
    v = statistics.mean(vals)
    facts = host_facts()
    sample = (f"oracle/layer_ref.py fp32 fwd+bwd of one full layer iteration per step ({wl.nanobatches} x "
              f"{wl.tokens} tokens, unscaled), {threads} threads on {facts['cpu_model'] or 'host CPU'}")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "s/iter", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(wl, world, group_world),
        "cpu_baseline": {"value": v, "unit": "s/iter", "cores": threads, "kind": "port", "sample": sample,
                         **facts, "timed_region_s": round(sum(vals), 2), "run_s": round(total, 2)},
        "e2e": {"value": v, "unit": "s/iter", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------- microbatch composition
def run_microbatch(args, wl, eng, gpu, layer, per_part, hbm, tf_sust, torch):
    from paper_2601_17654_b200.device import ProfilingProtocol
    from paper_2601_17654_b200.nonpartition import NonPartitionWork, measure_costs, unit_times

    work = NonPartitionWork(wl, eng.device)
    proto = ProfilingProtocol(warmup_s=0.2, window_s=args.sweep_window, cooldown_s=0.0)
    costs = {n: measure_costs(eng, work.programs[n], [gpu.f_max_mhz], proto) for n in ("np_fwd", "np_bwd")}
    ut = unit_times(work)
    units = {}
    for name in ("np_fwd", "np_bwd"):
        for u in work.programs[name].units:
            ms = ut[u.name]
            if u.kind == "gemm":
                units[u.name] = {"ms": round(ms, 4), "tflops": round(u.spec.flops / ms / 1e9, 1),
                                 "frac": round(u.spec.flops / ms / 1e9 / tf_sust, 4)}
            else:
                units[u.name] = {"ms": round(ms, 4), "gbs": round(u.spec.bytes / ms / 1e6, 1),
                                 "frac": round(u.spec.bytes / ms / 1e6 / hbm, 4)}
    out = {"non_partition_costs": {n: {str(f): [round(t, 4), round(e, 4)] for f, (t, e) in c.items()}
                                   for n, c in costs.items()},
           "non_partition_units": units, "n_layers": wl.model.n_layers, "vocab": wl.model.vocab}
    del work
    torch.cuda.empty_cache()
    try:
        ref = os.path.join(ROOT, "baseline", "_ref")
        if os.path.isdir(ref) and ref not in sys.path:
            sys.path.append(ref)
        from schedfront.compose import MicrobatchSpec, build_per_frequency_frontiers, microbatch_frontier
    except ImportError:
        out["composition"] = "skipped: reference package (baseline/_ref) not importable on this box"
        return out
    per_freq = build_per_frequency_frontiers({n: [(c, m) for c, m in rows] for n, rows in per_part.items()})
    L = wl.model.n_layers
    comp = {}
    for mb, blocks, npn in (("fwd", ("fwd_attn", "fwd_mlp"), "np_fwd"), ("bwd", ("bwd_mlp", "bwd_attn"), "np_bwd")):
        seq = [f"{blk}{b}" for blk in blocks for b in range(wl.nanobatches)] * L
        spec = MicrobatchSpec(f"{wl.model.name}-{mb}", tuple(seq), costs[npn])
        front = microbatch_frontier(spec, per_freq, gpu.p_static_w)
        comp[mb] = [{"time_ms": round(p.time_ms, 3), "energy_j": round(p.energy_j, 3),
                     "choices": {t: c.timing.encode() + f"@{c.sm_alloc}" for t, c in p.payload.choices}}
                    for p in front.points]
    out["composition"] = {"api": "schedfront.compose.microbatch_frontier (reference, unmodified)",
                          "microbatch": f"{L} layers x partitions + measured non-partition work, 1 pipeline stage",
                          "frontiers": comp}
    return out


# ---------------------------------------------------------------------------- GPU arm
def dominant_solo(unit, ncta: int, dev, torch, peak: float, bound: str, sampler=None, trials: int = 3,
                  window_ms: float = 50.0, idle_s: float = 1.0) -> dict:
    """The dominant launch unit timed alone: on all SMs, and with `ncta` whole SMs held by
    `kpo_sm_blocker` (2-CTA clusters, like the collectives) for the whole timed region. Median of
    `trials` windows of back-to-back launches (>= `window_ms` each), CUDA events on the launching stream,
    after `idle_s` of idle GPU so the power-capped clock of the preceding steps has recovered; the SM
    clock the sampler saw over the windows is reported next to the times."""
    from paper_2601_17654_b200 import _lib

    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    compute = torch.cuda.Stream(dev)
    side = torch.cuda.Stream(dev, priority=-1)
    launched = torch.cuda.Event()
    launched.record(side)

    def window(c: int, est_ms: float) -> float:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        if c:
            spin_ns = int((est_ms * reps * 3 * sms / max(1, sms - c) + 0.5) * 1e6)
            _lib.call("kpo_sm_blocker", c, spin_ns, launched.cuda_event, side.cuda_stream)
            compute.wait_event(launched)
        e0.record(compute)
        for _ in range(reps):
            unit.fn(compute)
        e1.record(compute)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1) / reps

    reps = 2
    window(0, 1.0)
    est = window(0, 1.0)
    reps = max(10, int(math.ceil(window_ms / max(est, 1e-3))))
    time.sleep(idle_s)
    work = unit.spec.flops / 1e12 if bound == "tensor" else unit.spec.bytes / 1e9
    out = {"method": "unit alone after %.1f s idle, median of %d windows x %d launches; 'blocked' holds the default "
                     "collective's %d whole SMs with kpo_sm_blocker" % (idle_s, trials, reps, ncta)}
    for key, c in (("all_sms", 0), ("blocked", ncta)):
        t0 = time.perf_counter()
        t = statistics.median(window(c, est) for _ in range(trials))
        clk = sampler.clocks_summary(t0, time.perf_counter()) if sampler is not None else {}
        out[key] = {"sms": sms - c, "avg_launch_ms": round(t, 4), "achieved": round(work / (t / 1e3), 1),
                    "frac": round(work / (t / 1e3) / peak, 4), "sm_mhz": clk.get("sm_mhz")}
    return out


def run_kpo(args):
    import torch
    import torch.distributed as dist

    from paper_2601_17654_b200.comm import Communicator
    from paper_2601_17654_b200.device import b200_model_measured, load_measured_peaks
    from paper_2601_17654_b200.domain import LaunchTiming, Measurement, ScheduleConfig
    from paper_2601_17654_b200.engine import Engine
    from paper_2601_17654_b200.layer import PartitionedLayer, sym_bytes_for
    from paper_2601_17654_b200.model import baseline_workload
    from paper_2601_17654_b200.runner import LayerRunner, sequential_schedule

    rank, world, local = dist_env()
    # KPO_SAME_DEVICE=1 (test only): every rank on cuda:0, gloo plumbing — exercises the N>1 path
    # (IPC peer mapping, cross-rank barriers, max/sum reductions) on a single-GPU box.
    same_dev = os.environ.get("KPO_SAME_DEVICE") == "1"
    if same_dev:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if same_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    red_dev = torch.device("cpu") if same_dev else dev
    group_world = world if world > 1 else 8
    wl = baseline_workload(args.config, world=group_world, tokens=args.tokens)
    if world == 1 and wl.world != group_world:  # config 0 (the reference's CPU case) is a 1-rank layer
        group_world = wl.world
    peaks = load_measured_peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    tf_burst = peaks.get("bf16_tflops", 1590.0)
    tf_sust = peaks.get("bf16_tflops_sustained", 1400.0)
    peak_src = "measured" if peaks else "fallback"
    gpu = b200_model_measured()  # committed descriptor (profiles/r2_descriptor.json), else nominal

    # symmetric heap: FSDP shards + two layer-parity gradient buffers; TP partial sums + stage
    sym = sym_bytes_for(wl)
    comm = (Communicator.loopback_group(group_world, sym, device=dev) if world == 1
            else Communicator.from_process_group(sym, device=dev))
    layer = PartitionedLayer(wl, comm)
    # the bench runs at the unlocked default clock (f_max); the frequency axis is the profiler's
    eng = Engine.for_layer(layer, gpu, clock_control=False)
    eng.sampler.aux_period_s = 0.01  # clock / power / throttle samples every 10 ms (a K-step region is ~0.1 s)
    run = LayerRunner(layer, eng)
    run.warm()

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t)

    def sum_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t)

    if world > 1:
        eng.agree_ms = max_over_ranks  # identical repetition counts on every rank (measure paths)

    for _ in range(max(3, args.warmup)):
        run.step()
    torch.cuda.synchronize(dev)
    # ------------------------------------------------ dominant kernel: per-unit times inside the step
    # (right before the timed steps, after the warm-up: the SM clock is then where the timed region
    # starts, so the per-unit fractions and `value` share a clock state; measured after the timed region
    # the power controller had already pulled the clock down by 200-500 MHz and the fractions moved with it)
    ut_t0 = time.perf_counter()
    try:
        ut = run.unit_times_graph(iters=UT_ITERS)
        ut_mode = "graph replay"
    except Exception as ex:  # capture unsupported: eager issue with the same events
        ut = run.unit_times(iters=UT_ITERS)
        ut_mode = "eager (" + type(ex).__name__ + ")"
    ut_clock = eng.sampler.clocks_summary(ut_t0, time.perf_counter())
    for _ in range(2):  # back on the step's own graphs before the timed region
        run.step()
    torch.cuda.synchronize(dev)
    # ------------------------------------------------ timed region (device time, max over ranks)
    barrier()
    torch.cuda.synchronize(dev)
    st = eng.exec.compute
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(st)
    for _ in range(args.steps):
        run.step()
    e1.record(st)
    torch.cuda.synchronize(dev)
    t1 = time.perf_counter()
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    clocks = eng.sampler.clocks_summary(t0, t1)

    # ------------------------------------------------ end to end through the host-buffer entry point
    pin = lambda t: torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    xs = [pin(a["x"]).copy_(a["x"].cpu()) for a in layer.nb]
    dys = [pin(a["dy"]).copy_(a["dy"].cpu()) for a in layer.nb]
    dxs = [pin(a["dx"]) for a in layer.nb]
    run.step_host(xs, dys, dxs)
    n_e2e = max(3, args.steps // 3)
    barrier()
    h0 = time.perf_counter()
    for _ in range(n_e2e):
        run.step_host(xs, dys, dxs)
    h1 = time.perf_counter()
    e2e_sync_s = max_over_ranks((h1 - h0) / n_e2e)
    # pipelined: H2D of step k+1 and D2H of step k-1 overlap step k on copy-engine streams; every
    # step's copies are still inside the timed region (first H2D .. last D2H)
    for _ in range(2):
        run.step_host_async(xs, dys, dxs)
    run.drain()
    n_pipe = max(100, args.steps)  # a training loop amortises the pipeline fill (first H2D) and drain (last D2H)
    barrier()
    h0 = time.perf_counter()
    for _ in range(n_pipe):
        run.step_host_async(xs, dys, dxs)
    run.drain()
    h1 = time.perf_counter()
    e2e_s = max_over_ranks((h1 - h0) / n_pipe)
    h2d = sum(t.numel() * t.element_size() for t in xs + dys)
    d2h = sum(t.numel() * t.element_size() for t in dxs)

    per_unit = {}
    for name in layer.order:
        for u in layer.programs[name].units:
            per_unit.setdefault(u.name, (u, []))
    totals = {k: sum(v) / UT_ITERS for k, v in ut.items()}
    step_ms_instr = sum(totals.values())
    dom = max(totals, key=lambda k: totals[k])  # dominant launch unit by share of the step
    kernels = []
    for k in sorted(totals, key=lambda k: -totals[k]):
        u = per_unit[k][0]
        avg = statistics.mean(ut[k])
        if u.kind in ("gemm", "attention"):
            ach = u.spec.flops / (avg / 1e3) / 1e12
            kernels.append({"unit": k, "bound": "tensor", "achieved": round(ach, 1), "unit_of": "TFLOP/s",
                            "frac": round(ach / tf_sust, 4), "avg_launch_ms": round(avg, 4),
                            "share": round(totals[k] / step_ms_instr, 4)})
        else:
            ach = u.spec.bytes / (avg / 1e3) / 1e9
            kernels.append({"unit": k, "bound": "hbm", "achieved": round(ach, 1), "unit_of": "GB/s",
                            "frac": round(ach / hbm, 4), "avg_launch_ms": round(avg, 4),
                            "share": round(totals[k] / step_ms_instr, 4)})
    dom_row = next(r for r in kernels if r["unit"] == dom)
    dom_unit = per_unit[dom][0]
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "dram_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(dom)
        except Exception:
            traffic = None

    # ------------------------------------------------ the dominant unit alone (explains the in-step frac)
    # timed alone on an idle GPU, and alone with the default collective's CTA count of whole SMs held by
    # kpo_sm_blocker (the SM budget an overlapped collective takes from it inside the step;
    # tools/unit_sm_sweep.py does this for every unit and SM count)
    solo = None
    try:
        solo = dominant_solo(dom_unit, eng.default_ncta(), dev, torch,
                             tf_sust if dom_row["bound"] == "tensor" else hbm, dom_row["bound"], eng.sampler)
    except Exception as ex:  # reported, never fatal
        solo = f"failed: {type(ex).__name__}: {ex}"

    # ------------------------------------------------ energy over a >= 2 s window of back-to-back steps
    n_energy = max(args.steps, int(math.ceil(2.0 / max(ms / 1e3, 1e-4))))
    barrier()
    torch.cuda.synchronize(dev)
    w0 = time.perf_counter()
    ew0, ew1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ew0.record(st)
    for _ in range(n_energy):
        run.step()
    ew1.record(st)
    torch.cuda.synchronize(dev)
    w1 = time.perf_counter()
    # the same steps over the >= 2 s window: the clock the power controller settles at under sw_power_cap
    # (the K-step timed region may end before the controller has pulled the SM clock down)
    ms_sustained = max_over_ranks(ew0.elapsed_time(ew1) / n_energy)
    energy_iter = sum_over_ranks(eng.sampler.window_j(w0, w1) / n_energy)
    eclocks = eng.sampler.clocks_summary(w0, w1)

    # ------------------------------------------------ collective bus bandwidth (comm unit alone)
    comm_rows = []
    cs = eng.exec.comm_stream
    for name in layer.order:
        cu = layer.programs[name].comm
        for nc in (eng.default_ncta(),):
            cu.fn(cs, nc)
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record(cs)
            for _ in range(5):
                cu.fn(cs, nc)
            c1.record(cs)
            c1.synchronize()
            cms = c0.elapsed_time(c1) / 5
            comm_rows.append({"unit": cu.name, "ncta": nc, "ms": round(cms, 4),
                              "busbw_gbps": round(cu.algo_bytes / (cms / 1e3) / 1e9, 1)})
    barrier()

    # ------------------------------------------------ MBO-selected schedule sets, executed as iterations
    # The per-partition frontiers come from the reference optimizer run on this hardware
    # (tools/mbo_hardware.py -> profiles/r2_mbo_config<N>.json + profile tables); here the selected
    # iteration-level sets run as whole iterations next to the default and sequential schedules,
    # interleaved trials of >= --sweep-window s each (device time max over ranks, NVML energy summed).
    frontier = None
    per_part = None
    # the 2 s-window run (frontier rows within 0.9% median of their re-measurement), else the first run
    # (config 1: the same tables replayed with the final kernels and the set that keeps the default among
    # each partition's candidates, r2x)
    mbo_path = os.path.join(ROOT, "profiles", f"r2x_mbo_config{args.config}.json")
    if not os.path.exists(mbo_path):
        mbo_path = os.path.join(ROOT, "profiles", f"r2w2_mbo_config{args.config}.json")
    if not os.path.exists(mbo_path):
        mbo_path = os.path.join(ROOT, "profiles", f"r2_mbo_config{args.config}.json")
    if args.no_sweep:
        pass
    elif not os.path.exists(mbo_path):
        frontier = {"skipped": f"no MBO result for config {args.config} ({os.path.relpath(mbo_path, ROOT)})"}
    else:
        mb = json.load(open(mbo_path))
        if mb.get("workload", "").split("-T")[-1] != wl.tag.split("-T")[-1]:
            frontier = {"skipped": f"MBO result is for {mb.get('workload')}, not {wl.tag}"}
        else:
            def decode(enc):
                t, sm, f = enc.split("@")
                return ScheduleConfig(float(f), int(sm), LaunchTiming.decode(t))

            sets = {"nanobatching_default": run.schedule, "sequential_megatron": sequential_schedule(layer, gpu)}
            for k, sel in mb.get("sets", {}).items():
                if k.startswith("mbo_"):
                    sets[k] = {n: decode(sel[n]) for n in layer.order}
            runners = {k: LayerRunner(layer, eng, schedule=sch) for k, sch in sets.items()}
            for r2 in runners.values():
                r2.warm()
            n_it = max(args.steps, int(math.ceil(args.sweep_window / max(ms / 1e3, 1e-4))))
            acc = {k: {"s": [], "j": []} for k in sets}
            q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for _trial in range(args.sweep_trials):
                for k, r2 in runners.items():
                    for _ in range(3):
                        r2.step()
                    barrier()
                    torch.cuda.synchronize(dev)
                    w0 = time.perf_counter()
                    q0.record(eng.exec.compute)
                    for _ in range(n_it):
                        r2.step()
                    q1.record(eng.exec.compute)
                    torch.cuda.synchronize(dev)
                    w1 = time.perf_counter()
                    t_it = q0.elapsed_time(q1) / n_it / 1e3
                    e_win = eng.sampler.window_j(w0, w1) - max(0.0, (w1 - w0) - t_it * n_it) * gpu.p_static_w
                    acc[k]["s"].append(max_over_ranks(t_it))
                    acc[k]["j"].append(sum_over_ranks(e_win / n_it))
            ex_rows = {}
            for k, v in acc.items():
                sd = lambda xs: statistics.stdev(xs) if len(xs) > 1 else 0.0
                ex_rows[k] = {"s_per_iter": round(statistics.mean(v["s"]), 7), "s_std": round(sd(v["s"]), 7),
                              "j_per_iter": round(statistics.mean(v["j"]), 4), "j_std": round(sd(v["j"]), 4)}
            d0 = ex_rows["nanobatching_default"]
            for k, v in ex_rows.items():
                v["time_vs_default"] = round(v["s_per_iter"] / d0["s_per_iter"] - 1, 5)
                v["energy_vs_default"] = round(v["j_per_iter"] / d0["j_per_iter"] - 1, 5)
            # the same per-unit in-step timing as `kernels`, under the MBO min-time schedule set (its
            # collectives launch later and on fewer SMs, so fewer units share their SMs with one)
            kernels_mbo = None
            if "mbo_min_time" in runners:
                try:
                    ut2 = runners["mbo_min_time"].unit_times_graph(iters=UT_ITERS)
                    kernels_mbo = {}
                    for k2, v2 in ut2.items():
                        u2 = next(u for nm in layer.order for u in layer.programs[nm].units if u.name == k2)
                        avg2 = statistics.mean(v2)
                        if u2.kind in ("gemm", "attention"):
                            kernels_mbo[k2] = {"avg_launch_ms": round(avg2, 4),
                                               "frac": round(u2.spec.flops / (avg2 / 1e3) / 1e12 / tf_sust, 4)}
                        else:
                            kernels_mbo[k2] = {"avg_launch_ms": round(avg2, 4),
                                               "frac": round(u2.spec.bytes / (avg2 / 1e3) / 1e9 / hbm, 4)}
                except Exception as ex:  # reported, never fatal
                    kernels_mbo = f"failed: {type(ex).__name__}: {ex}"
            frontier = {"source": os.path.relpath(mbo_path, ROOT), "optimizer": mb.get("optimizer"),
                        "protocol": mb.get("protocol"), "sets": mb.get("sets"), "executed": ex_rows,
                        "trials": args.sweep_trials, "iterations_per_trial": n_it,
                        "kernels_mbo_min_time": kernels_mbo,
                        "note": "frequency axis fixed at f_max: every NVML clock knob is refused on this pool "
                                "(profiles/r2_clock_probe.json)"}
            # the measured profile tables feed the reference's microbatch composition below
            per_part = {}
            from paper_2601_17654_b200.profiler import ProfileTable
            for n in layer.order:
                tp = os.path.join(ROOT, mb["partitions"][n]["table"]) if n in mb.get("partitions", {}) else None
                if tp is None or not os.path.exists(tp):
                    per_part = None
                    break
                t = ProfileTable.read(tp)
                per_part[n] = [(r.config(), Measurement(r.time_ms, r.dyn_energy_j, r.static_energy_j,
                                                        r.total_energy_j)) for r in t.rows]

    # ------------------------------------------------ non-partition work + microbatch composition
    # (SURVEY §8f item 1): embedding / final norm / LM head / loss measured on the hardware, and
    # the reference's own microbatch_frontier composing the measured partition candidates with it
    microbatch = None
    if not args.no_sweep and per_part is not None:
        microbatch = run_microbatch(args, wl, eng, gpu, layer, per_part, hbm, tf_sust, torch)

    # ------------------------------------------------ CPU baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        setup = cpu_layer_setup(wl, wl.nanobatches)
        cpu_iteration(wl, threads, setup)  # first call pays allocator / thread-pool warm-up
        ts = [cpu_iteration(wl, threads, setup) for _ in range(args.cpu_iters)]
        facts = host_facts()
        cpu = {"value": statistics.mean(ts), "unit": "s/iter", "cores": threads, "kind": "port",
               "sample": f"oracle/layer_ref.py fp32 fwd+bwd of {args.cpu_iters} full layer iterations "
                         f"({wl.nanobatches} x {wl.tokens} tokens each, unscaled; {sum(ts):.1f} s of CPU work)",
               **facts}
        try:
            cpu["reference_path"] = reference_cpu_path(wl)
        except Exception as ex:  # reported, never fatal: the reference package is an optional guest here
            cpu["reference_path"] = f"failed: {type(ex).__name__}: {ex}"

    # iteration-level roofline: T_lb = max(F_tc / P_tc, B_hbm / BW_hbm, B_link / BW_link)
    specs_all = [u.spec for name in layer.order for u in layer.programs[name].units]
    f_tc = sum(sp.flops for sp in specs_all if sp.kind == "compute-bound")
    b_hbm = sum(sp.bytes for sp in specs_all if sp.kind == "memory-bound")
    b_link = sum(layer.programs[name].comm.algo_bytes for name in layer.order)
    link_bw = (hbm if world == 1 else 770.0) * 1e9  # loopback moves the "link" bytes through HBM
    t_lb = max(f_tc / (tf_sust * 1e12), b_hbm / (hbm * 1e9), b_link / link_bw)
    iter_roofline = {"t_lb_ms": round(t_lb * 1e3, 4), "t_meas_ms": round(ms, 4), "frac": round(t_lb * 1e3 / ms, 4),
                     "tensor_flops": f_tc, "hbm_bytes": b_hbm, "link_bytes": b_link,
                     "bounds_ms": {"tensor": round(f_tc / (tf_sust * 1e12) * 1e3, 4),
                                   "hbm": round(b_hbm / (hbm * 1e9) * 1e3, 4),
                                   "link": round(b_link / link_bw * 1e3, 4)},
                     "peaks": f"{peak_src}: {tf_sust} TF/s sustained bf16, {hbm} GB/s HBM, "
                              f"{'HBM (loopback)' if world == 1 else '770 GB/s NVLink per direction'}"}

    if rank == 0:
        launches = run.kernels_per_step() * args.steps
        line = {
            "metric": METRIC, "value": ms / 1e3, "unit": "s/iter", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (weights N(0,0.02) seed 0, activations N(0,1) seed 1000+rank)",
            "config": workload_config(wl, world, group_world),
            "default_comm_ctas": eng.default_ncta(),
            "graphs": {"captured": len(eng.exec.graphs), "failures": len(eng.exec.graph_failures),
                       "launch_gate": eng.exec.gate_status},
            "energy_j_per_iter": energy_iter, "energy_window_steps": n_energy,
            "sustained": {"ms_per_step": round(ms_sustained, 4), "steps": n_energy,
                          "sm_mhz": eclocks.get("sm_mhz"), "clock_samples": eclocks.get("samples"),
                          "reasons": eclocks.get("reasons"),
                          "note": "the same step back to back over the >= 2 s energy window (CUDA events, max "
                                  "over ranks); value / ms_per_step are the K-step timed region"},
            "avg_power_w": energy_iter / (ms / 1e3) if ms > 0 else None,
            "tflops_per_gpu": iteration_flops(wl) / (ms / 1e3) / 1e12,
            "roofline": {"bound": dom_row["bound"], "kernel": dom, "achieved": dom_row["achieved"],
                         "peak": tf_sust if dom_row["bound"] == "tensor" else hbm, "unit": dom_row["unit_of"],
                         "frac": dom_row["frac"], "traffic": traffic,
                         "peak_kind": (f"{peak_src} sustained bf16 (kernel timed inside the step)"
                                       if dom_row["bound"] == "tensor" else f"{peak_src} HBM copy"),
                         "share_of_step": dom_row["share"],
                         "algorithmic_per_launch": dom_unit.spec.flops if dom_row["bound"] == "tensor"
                         else dom_unit.spec.bytes, "avg_launch_ms": dom_row["avg_launch_ms"],
                         "solo": solo},
            "kernels": kernels,
            "kernels_timing": "CUDA events around each launch unit on the compute stream, " + ut_mode + f", {UT_ITERS} iterations",
            "kernels_sm_mhz": ut_clock.get("sm_mhz"),
            "iteration_roofline": iter_roofline,
            "comm": {"mode": "loopback (HBM)" if world == 1 else "cuda-ipc p2p (NVLink)", "units": comm_rows},
            "frontier": frontier,
            "microbatch": microbatch,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_s, "unit": "s/iter", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": "LayerRunner.step_host_async x K + drain(): pinned host x/dy in, dx out, copies "
                           "pipelined on copy-engine streams (wall clock, max over ranks)",
                    "unpipelined_value": e2e_sync_s},
            "gpu_launches": launches,
            "clocks": {"sm_mhz": clocks.get("sm_mhz") or eclocks.get("sm_mhz"), "sm_max_mhz": eng.nvml.max_sm_clock_mhz(),
                       "samples": clocks.get("samples", 0), "energy_window_sm_mhz": eclocks.get("sm_mhz"),
                       "reasons": sorted(set(clocks.get("reasons", [])) | set(eclocks.get("reasons", []))),
                       "power_w_max": eclocks.get("power_w_max")},
        }
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_kpo(args)


if __name__ == "__main__":
    sys.exit(main())
