"""Profile one steady-state layer iteration of the bench workload (for ncu --profile-from-start off).

python tools/profile_step.py [--config 1] [--tokens 4096] [--eager]
Builds the bench layer, warms the per-partition graphs, then brackets exactly ONE iteration with
cudaProfilerStart/Stop so the ncu launch list is the step's kernels and nothing else."""
import argparse
import os
import sys

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
ap.add_argument("--tokens", type=int, default=4096)
ap.add_argument("--eager", action="store_true")
a = ap.parse_args()
wl = baseline_workload(a.config, world=8, tokens=a.tokens)
n = wl.weight_numels()
from paper_2601_17654_b200.layer import sym_bytes_for
sym = sym_bytes_for(wl)
comm = Communicator.loopback_group(8, sym)
layer = PartitionedLayer(wl, comm)
eng = Engine.for_layer(layer, b200_model(), use_graphs=not a.eager)
run = LayerRunner(layer, eng)
run.warm()
for _ in range(2):
    run.step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
run.step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
eng.close()
print("profiled one step:", run.kernels_per_step(), "kernels")
