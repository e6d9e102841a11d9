"""Candidate profiler on hardware: measure a partition's enumerated schedule space with the
thermally-stable protocol, write the profile table (JSONL) and replay it through the UNMODIFIED
reference optimizer (baseline/_ref) to select the Pareto schedule set.

python tools/profile_partition.py --config 1 --partition fwd_mlp0 --window 0.3 --cooldown 0.1 \
       --out gpurun_out/table_fwd_mlp0.jsonl
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
import torch

from paper_2601_17654_b200 import FrequencyGrid, SmGrid, b200_model
from paper_2601_17654_b200.comm import Communicator
from paper_2601_17654_b200.compat import patch_reference
from paper_2601_17654_b200.device import ProfilingProtocol, ThermalModel, ThermalState
from paper_2601_17654_b200.engine import Engine
from paper_2601_17654_b200.layer import PartitionedLayer
from paper_2601_17654_b200.model import baseline_workload
from paper_2601_17654_b200.profiler import ProfileTable, Profiler, gpu_header

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--partition", default="fwd_mlp0")
ap.add_argument("--warmup", type=float, default=0.1)
ap.add_argument("--window", type=float, default=0.3)
ap.add_argument("--cooldown", type=float, default=0.1)
ap.add_argument("--max-configs", type=int, default=0)
ap.add_argument("--out", default="gpurun_out/profile_table.jsonl")
a = ap.parse_args()

wl = baseline_workload(a.config, world=8)
n = wl.weight_numels()
from paper_2601_17654_b200.layer import sym_bytes_for
sym = sym_bytes_for(wl)
comm = Communicator.loopback_group(8, sym)
layer = PartitionedLayer(wl, comm)
eng = Engine.for_layer(layer, b200_model())
gpu = eng.gpu
part = layer.programs[a.partition].spec()

import schedfront
from schedfront import mbo

# the B200 schedule space: NVML clocks cannot be locked on this pool -> frequency fixed at f_max
freqs = FrequencyGrid((gpu.f_max_mhz,))
sms = SmGrid.b200()
space = mbo.enumerate_space(part, gpu, freqs, sms, max_overlap_span=9)
if a.max_configs:
    space = space[: a.max_configs]
proto = ProfilingProtocol(warmup_s=a.warmup, window_s=a.window, cooldown_s=a.cooldown)
state = ThermalState.new(ThermalModel(), proto)
t0 = time.time()
table = Profiler(eng, gpu, proto, ThermalModel(), state).collect(
    part, space, header={"gpu": gpu_header(gpu), "freq_grid": list(freqs.values), "sm_grid": list(sms.values),
                         "max_overlap_span": 9, "workload": wl.tag, "protocol": vars(proto) if hasattr(proto, "__dict__") else {},
                         "clock_control": eng.freq.reason})
dt = time.time() - t0
table.write(a.out)

# replay through the reference optimizer (bit-exact with the measured rows)
ev = ProfileTable.read(a.out).evaluator(schedfront.domain.Measurement)
restore = patch_reference(measure=lambda p, c, *x: ev(p, c), schedfront_module=schedfront)
try:
    res = mbo.run_mbo(part, gpu, ThermalModel(), proto, mbo.MboHyperparams.for_partition(part, seed=0), freqs, sms)
finally:
    restore()
default = next(r for r in table.rows if r.timing == f"ov0x{len(part.comp_kernels)}" and r.sm_alloc == 16)
seq = next(r for r in table.rows if r.timing == "seq")
summary = {
    "partition": a.partition, "workload": wl.tag, "configs_measured": len(table), "profiling_s": round(dt, 1),
    "s_per_candidate": round(dt / max(1, len(table)), 3),
    "mbo_evals": len(res.records), "frontier": [(round(p.time_ms, 4), round(p.energy_j, 4), p.payload.timing.encode(),
                                                  p.payload.sm_alloc) for p in res.frontier],
    "default_nanobatching": {"time_ms": default.time_ms, "total_j": default.total_energy_j},
    "sequential": {"time_ms": seq.time_ms, "total_j": seq.total_energy_j},
    "best_time_measured": min((r.time_ms, r.timing, r.sm_alloc) for r in table.rows),
    "best_energy_measured": min((r.total_energy_j, r.timing, r.sm_alloc) for r in table.rows),
}
print(json.dumps(summary))
json.dump(summary, open(a.out.replace(".jsonl", "_summary.json"), "w"), indent=1)
eng.close()
