"""Solo launch-unit times per available SM count ("measured solo-kernel times per
(f, SMs)"; reference kernel_duration(k, f, sms), simgpu.py:144-168).  The frequency axis is fixed at
f_max on this pool (profiles/r2_clock_probe.json); the SM axis is realised the way the executor
realises it in an overlapped partition: `kpo_sm_blocker` holds `c` SMs (whole-SM CTAs, 2-CTA clusters
like the collectives) for the duration of the measurement, and the unit runs on the other 148 - c.

For every launch unit of the BASELINE config-1 layer and c in --ctas: median of --trials windows of
--reps back-to-back launches (CUDA events on the compute stream, after the blocker's launch-completion
event).  Reported next to the reference model's assumption, t(c) = t(0) * 148 / (148 - c) for
compute-bound kernels (flop_rate proportional to SMs) and an SM-independent HBM rate otherwise.

python tools/unit_sm_sweep.py [--ctas 0,6,12,24,36,48,74] --out gpurun_out/unit_sm_sweep.json"""
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
    ap.add_argument("--ctas", default="0,6,12,24,36,48,74")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--trials", type=int, default=3)
    ap.add_argument("--out", default="gpurun_out/unit_sm_sweep.json")
    a = ap.parse_args()

    import torch

    from paper_2601_17654_b200 import _lib
    from paper_2601_17654_b200.comm import Communicator
    from paper_2601_17654_b200.layer import PartitionedLayer, sym_bytes_for
    from paper_2601_17654_b200.model import baseline_workload

    dev = torch.device("cuda", 0)
    wl = baseline_workload(a.config)
    comm = Communicator.loopback_group(wl.world, sym_bytes_for(wl), device=dev)
    layer = PartitionedLayer(wl, comm)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    compute = torch.cuda.Stream(dev)
    side = torch.cuda.Stream(dev, priority=-1)
    launched = torch.cuda.Event()
    launched.record(side)  # materialise the CUDA event
    units = {}
    for name in layer.order:
        for u in layer.programs[name].units:
            units.setdefault(u.name, u)
    ctas = [int(x) for x in a.ctas.split(",")]

    def timed(u, c, reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        if c:
            spin = int((est.get(u.name, 1.0) * reps * 3 * (sms / max(1, sms - c)) + 0.5) * 1e6)
            _lib.call("kpo_sm_blocker", c, spin, launched.cuda_event, side.cuda_stream)
            compute.wait_event(launched)
        e0.record(compute)
        for _ in range(reps):
            u.fn(compute)
        e1.record(compute)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1) / reps

    est = {}
    for nm, u in units.items():  # warm-up and full-SM estimate
        timed(u, 0, 2)
        est[nm] = timed(u, 0, a.reps)
    rows = {}
    for nm, u in units.items():
        sp = u.spec
        row = {"kind": sp.kind, "flops": sp.flops, "bytes": sp.bytes, "ms": {}}
        for c in ctas:
            row["ms"][str(c)] = statistics.median(timed(u, c, a.reps) for _ in range(a.trials))
        t0 = row["ms"][str(ctas[0])]
        row["slowdown"] = {str(c): round(row["ms"][str(c)] / t0, 4) for c in ctas}
        row["linear_model"] = {str(c): round(sms / (sms - c), 4) if sp.kind == "compute-bound" else 1.0 for c in ctas}
        rows[nm] = row
        print(nm, {c: round(v, 4) for c, v in row["ms"].items()}, flush=True)
    out = {"workload": wl.tag, "num_sms": sms, "ctas_blocked": ctas, "reps": a.reps, "trials": a.trials,
           "method": "kpo_sm_blocker holds c whole SMs (2-CTA clusters) during the unit's timed launches",
           "units": rows}
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)
    comm.close()


if __name__ == "__main__":
    main()
