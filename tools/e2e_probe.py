"""Where the end-to-end (host-buffer) iteration time goes beyond the device step: the pipelined
step_host_async loop vs the same loop without the PCIe copies, without the staging D2D copies, and the
bare step.  Measurement only.  python tools/e2e_probe.py [--config 1]"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_17654_b200.comm import Communicator
from paper_2601_17654_b200.device import b200_model
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


def wall(fn):
    for _ in range(3):
        fn()
    run.drain()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(a.n):
        fn()
    run.drain()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / a.n * 1e3


res = {"step_only_ms": wall(run.step)}
res["pipelined_e2e_ms"] = wall(lambda: run.step_host_async(xs, dys, dxs))
comp = eng.exec.compute


def d2d_only():
    with torch.cuda.stream(comp):
        for x in layer.nb:
            x["x"].copy_(x["x"], non_blocking=True)
            x["dy"].copy_(x["dy"], non_blocking=True)
    run.step()
    with torch.cuda.stream(comp):
        for x in layer.nb:
            x["dx"].copy_(x["dx"], non_blocking=True)


stg = [torch.empty_like(x["x"]) for x in layer.nb]


def d2d_copies():
    with torch.cuda.stream(comp):
        for x, s in zip(layer.nb, stg):
            s.copy_(x["x"], non_blocking=True)
            x["x"].copy_(s, non_blocking=True)
            s.copy_(x["dy"], non_blocking=True)
            x["dy"].copy_(s, non_blocking=True)
    run.step()


res["step_plus_4_d2d_ms"] = wall(d2d_copies)
h2d = torch.cuda.Stream()


def pcie_only():
    with torch.cuda.stream(h2d):
        for x, s in zip(xs, stg):
            s.copy_(x, non_blocking=True)
    run.step()


res["step_with_concurrent_h2d_ms"] = wall(pcie_only)
print(json.dumps({k: round(v, 4) for k, v in res.items()}))
