"""Attention-backward ablation timing (measurement only): KPO_ATTN_BWD_ABLATE bits switch off parts of
the kernel (1 dQ reduce-add, 2 dQ drain, 4 exponentials, 8 dQ^T MMA) to find which part bounds it.
python tools/attn_ablate.py [--T 4096 --hq 24 --hkv 8]"""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2601_17654_b200 import ops


def timeit(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


ap = argparse.ArgumentParser()
ap.add_argument("--T", type=int, default=4096)
ap.add_argument("--hq", type=int, default=24)
ap.add_argument("--hkv", type=int, default=8)
ap.add_argument("--modes", default="0,1,3,4,8,11,15")
a = ap.parse_args()
T, hq, hkv, d = a.T, a.hq, a.hkv, 128
dev = torch.device("cuda")
qkv = torch.randn(T, (hq + 2 * hkv) * d, device=dev).bfloat16()
q, k, v = qkv[:, :hq * d], qkv[:, hq * d:(hq + hkv) * d], qkv[:, (hq + hkv) * d:]
o = torch.empty(T, hq * d, device=dev, dtype=torch.bfloat16)
lse = torch.empty(hq, T, device=dev)
scale = 1 / math.sqrt(d)
ops.attn_fwd(q, k, v, o, lse, T, hq, hkv, d, scale)
fl = 2.5 * 2.0 * T * T * hq * d / 2 * 2  # causal fwd 2*T^2*hq*d (x2 GEMMs / 2 causal), bwd = 2.5x
dout = torch.randn_like(o)
dqkv = torch.empty_like(qkv)
ws = ops.attn_bwd_workspace(T, hq, hkv, d, dev)
res = {}
for m in [int(x) for x in a.modes.split(",")]:
    os.environ["KPO_ATTN_BWD_ABLATE"] = str(m)
    t = timeit(lambda: ops.attn_bwd(q, k, v, o, dout, lse, dqkv[:, :hq * d], dqkv[:, hq * d:(hq + hkv) * d],
                                    dqkv[:, (hq + hkv) * d:], T, hq, hkv, d, scale, ws), reps=10)
    res[m] = {"ms": round(t, 4), "tflops": round(fl / t / 1e9, 1)}
os.environ["KPO_ATTN_BWD_ABLATE"] = "0"
print(json.dumps(res))
