"""Run the attention backward once (config-2 shapes) between cudaProfilerStart/Stop for ncu."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_17654_b200 import ops
T, hq, hkv, d = 4096, 24, 8, 128
qkv = torch.randn(T, (hq + 2 * hkv) * d, device="cuda").bfloat16()
q, k, v = qkv[:, :hq * d], qkv[:, hq * d:(hq + hkv) * d], qkv[:, (hq + hkv) * d:]
o = torch.empty(T, hq * d, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(hq, T, device="cuda")
ops.attn_fwd(q, k, v, o, lse, T, hq, hkv, d, 1 / math.sqrt(d))
dout = torch.randn_like(o)
dqkv = torch.empty_like(qkv)
ws = ops.attn_bwd_workspace(T, hq, hkv, d, "cuda")
args = (q, k, v, o, dout, lse, dqkv[:, :hq * d], dqkv[:, hq * d:(hq + hkv) * d], dqkv[:, (hq + hkv) * d:], T, hq, hkv, d,
        1 / math.sqrt(d), ws)
ops.attn_bwd(*args)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
ops.attn_fwd(q, k, v, o, lse, T, hq, hkv, d, 1 / math.sqrt(d))
ops.attn_bwd(*args)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
