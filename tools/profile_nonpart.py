"""Profile one execution of the non-partition programs (embedding, final norm, LM head GEMMs, fused
cross-entropy, embedding backward) of the bench workload; for ncu --profile-from-start off."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2601_17654_b200.model import baseline_workload
from paper_2601_17654_b200.nonpartition import NonPartitionWork

wl = baseline_workload(1, world=8)
w = NonPartitionWork(wl, torch.device("cuda", 0))
w.run()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
w.run()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
