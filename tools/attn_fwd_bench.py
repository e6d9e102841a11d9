"""Attention forward timing at config-1 shapes (T 4096, 24 q / 8 kv heads, d 128, causal), CUDA events over
back-to-back calls; env knobs (KPO_ATTN_FWD, KPO_ATTN_FWD_POLY, KPO_ATTN_PINGPONG) select variants.
Measurement only.  python tools/attn_fwd_bench.py [--T 4096 --hq 24 --hkv 8]"""
import argparse, json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_17654_b200 import ops

ap = argparse.ArgumentParser()
ap.add_argument("--T", type=int, default=4096)
ap.add_argument("--hq", type=int, default=24)
ap.add_argument("--hkv", type=int, default=8)
a = ap.parse_args()
T, hq, hkv, d = a.T, a.hq, a.hkv, 128
qkv = torch.randn(T, (hq + 2 * hkv) * d, device="cuda").bfloat16()
q, k, v = qkv[:, :hq * d], qkv[:, hq * d:(hq + hkv) * d], qkv[:, (hq + hkv) * d:]
o = torch.empty(T, hq * d, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(hq, T, device="cuda")
fn = lambda: ops.attn_fwd(q, k, v, o, lse, T, hq, hkv, d, 1 / math.sqrt(d))
for _ in range(3):
    fn()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    fn()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(json.dumps({"ms": round(ms, 4), "tflops": round(2.0 * T * T * hq * d / ms / 1e9, 1),
                  "poly": os.environ.get("KPO_ATTN_FWD_POLY", "0")}))
