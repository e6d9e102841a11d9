"""Where the end-to-end (host-buffer) iteration time goes beyond the device step: the pipelined
step_host_async loop vs the same loop without the PCIe copies, without the staging D2D copies, and the
bare step.  Measurement only.  python tools/e2e_probe.py [--config 1]"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_17654_b200.comm import Communicator
from paper_2601_17654_b200.device import b200_model_measured as b200_model
from paper_2601_17654_b200.engine import Engine
from paper_2601_17654_b200.layer import PartitionedLayer
from paper_2601_17654_b200.model import baseline_workload
from paper_2601_17654_b200.runner import LayerRunner

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--n", type=int, default=60)
a = ap.parse_args()
wl = baseline_workload(a.config, world=8, tokens=4096)
n = wl.weight_numels()
from paper_2601_17654_b200.layer import sym_bytes_for
sym = sym_bytes_for(wl)
layer = PartitionedLayer(wl, Communicator.loopback_group(8, sym))
eng = Engine.for_layer(layer, b200_model())
run = LayerRunner(layer, eng)
run.warm()
pin = lambda t: torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
xs = [pin(x["x"]).copy_(x["x"].cpu()) for x in layer.nb]
dys = [pin(x["dy"]).copy_(x["dy"].cpu()) for x in layer.nb]
dxs = [pin(x["dx"]) for x in layer.nb]


clk = {}


def wall(fn, key=None):
    for _ in range(3):
        fn()
    run.drain()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(a.n):
        fn()
    run.drain()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    if key:  # median SM clock and power over the window (NVML, engine sampler)
        c = eng.sampler.clocks_summary(t0, t1)
        clk.setdefault(key, []).append((c.get("sm_mhz"), c.get("power_w_max")))
    return (t1 - t0) / a.n * 1e3


comp = eng.exec.compute
stg = [torch.empty_like(x["x"]) for x in layer.nb]
h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()


def with_h2d():  # the step with the pipelined loop's H2D volume (x and dy) running beside it
    with torch.cuda.stream(h2d):
        for x, dy, s in zip(xs, dys, stg):
            s.copy_(x, non_blocking=True)
            s.copy_(dy, non_blocking=True)
    run.step()


def with_d2h():  # the step with the loop's D2H volume (dx) running beside it
    with torch.cuda.stream(d2h):
        for x, dx in zip(layer.nb, dxs):
            dx.copy_(x["dx"], non_blocking=True)
    run.step()


variants = {"step_only_ms": run.step, "pipelined_e2e_ms": lambda: run.step_host_async(xs, dys, dxs),
            "step_with_concurrent_h2d_ms": with_h2d, "step_with_concurrent_d2h_ms": with_d2h}
res = {k: [] for k in variants}
for _ in range(3):  # interleaved rounds: the box's power / thermal drift hits every variant alike
    for k, fn in variants.items():
        res[k].append(wall(fn, k))
        if k != "pipelined_e2e_ms":
            h2d.synchronize()
            d2h.synchronize()
print(json.dumps({"ms": {k: [round(x, 4) for x in v] for k, v in res.items()}, "sm_mhz_power_w": clk}))
