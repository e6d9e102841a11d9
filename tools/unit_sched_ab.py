"""Per-launch-unit in-step durations under the default (comm overlapped from kernel 0) and the
sequential schedule, to separate comm interference from kernel speed.  Measurement only.
python tools/unit_sched_ab.py [--config 2]"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_17654_b200.comm import Communicator
from paper_2601_17654_b200.device import b200_model
from paper_2601_17654_b200.engine import Engine
from paper_2601_17654_b200.layer import PartitionedLayer
from paper_2601_17654_b200.model import baseline_workload
from paper_2601_17654_b200.runner import LayerRunner, sequential_schedule

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
a = ap.parse_args()
wl = baseline_workload(a.config, world=8, tokens=4096)
n = wl.weight_numels()
from paper_2601_17654_b200.layer import sym_bytes_for
sym = sym_bytes_for(wl)
comm = Communicator.loopback_group(8, sym)
layer = PartitionedLayer(wl, comm)
eng = Engine.for_layer(layer, b200_model())
out = {}
for tag, sched in (("default", None), ("sequential", sequential_schedule(layer, eng.gpu))):
    r = LayerRunner(layer, eng, schedule=sched)
    r.warm()
    t = r.unit_times_graph(iters=5)
    out[tag] = {k: round(sorted(v)[len(v) // 2], 4) for k, v in t.items()}
print(json.dumps(out))

# whole-step time (same process) for comparison with the sum of unit times
r = LayerRunner(layer, eng)
r.warm()
for _ in range(5):
    r.step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(eng.exec.compute)
for _ in range(20):
    r.step()
e1.record(eng.exec.compute)
torch.cuda.synchronize()
print(json.dumps({"step_ms": e0.elapsed_time(e1) / 20,
                  "unit_sum_default_ms": sum(out["default"].values()),
                  "n_units": len(out["default"])}))

# the same launch units, collectives replaced by no-ops, per-partition graphs: the compute-only step
import dataclasses
from paper_2601_17654_b200.runner import sequential_schedule as _seq
progs = {}
for name in layer.order:
    p = layer.programs[name]
    nocomm = dataclasses.replace(p.comm, fn=lambda st, ncta: None)
    progs[name] = type(p)(p.name, p.units, nocomm, p.comm_group_size)
saved = dict(layer.programs)
layer.programs.update(progs)
eng.exec.graphs.clear()
r3 = LayerRunner(layer, eng, schedule=_seq(layer, eng.gpu))
r3.warm()
for _ in range(5):
    r3.step()
torch.cuda.synchronize()
e0.record(eng.exec.compute)
for _ in range(20):
    r3.step()
e1.record(eng.exec.compute)
torch.cuda.synchronize()
print(json.dumps({"compute_only_ms": e0.elapsed_time(e1) / 20}))
layer.programs.update(saved)
