"""Microbench of the hot kernels at BASELINE config-2 shapes (CUDA events, warm, inputs > L2 not needed:
kernels are compute-bound).  python tools/kernel_bench.py [--T 4096]"""
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
ap.add_argument("--d", type=int, default=128)
a = ap.parse_args()
T, hq, hkv, d = a.T, a.hq, a.hkv, a.d
dev = torch.device("cuda")
qkv = torch.randn(T, (hq + 2 * hkv) * d, device=dev).bfloat16()
q, k, v = qkv[:, :hq * d], qkv[:, hq * d:(hq + hkv) * d], qkv[:, (hq + hkv) * d:]
o = torch.empty(T, hq * d, device=dev, dtype=torch.bfloat16)
lse = torch.empty(hq, T, device=dev)
scale = 1 / math.sqrt(d)
fl = 2.0 * T * T * hq * d
res = {}
t = timeit(lambda: ops.attn_fwd(q, k, v, o, lse, T, hq, hkv, d, scale))
res["attn_fwd_tcgen05"] = {"ms": t, "tflops": fl / t / 1e9}
o2 = torch.empty_like(o)
lse2 = torch.empty_like(lse)
t = timeit(lambda: ops.attn_fwd_mma(q, k, v, o2, lse2, T, hq, hkv, d, scale))
res["attn_fwd_mma"] = {"ms": t, "tflops": fl / t / 1e9}
res["fwd_max_abs_diff_vs_mma"] = (o.float() - o2.float()).abs().max().item()
res["lse_max_abs_diff_vs_mma"] = (lse - lse2).abs().max().item()
dout = torch.randn_like(o)
dqkv = torch.empty_like(qkv)
ws = ops.attn_bwd_workspace(T, hq, hkv, d, dev)
t = timeit(lambda: ops.attn_bwd(q, k, v, o, dout, lse, dqkv[:, :hq * d], dqkv[:, hq * d:(hq + hkv) * d],
                                dqkv[:, (hq + hkv) * d:], T, hq, hkv, d, scale, ws), reps=10)
res["attn_bwd"] = {"ms": t, "tflops": 2.5 * fl / t / 1e9}
x = torch.randn(T, 3072, device=dev).bfloat16()
w = torch.randn(16384, 3072, device=dev).bfloat16()
y = torch.empty(T, 16384, device=dev, dtype=torch.bfloat16)
t = timeit(lambda: ops.linear(x, w, y))
res["gemm_4096x16384x3072"] = {"ms": t, "tflops": 2 * T * 16384 * 3072 / t / 1e9}
t = timeit(lambda: torch.matmul(x, w.t(), out=y))
res["cublas_4096x16384x3072"] = {"ms": t, "tflops": 2 * T * 16384 * 3072 / t / 1e9}
print(json.dumps(res, indent=1))

# ---- memory-bound kernels standalone (config-2 shapes), GB/s of algorithmic bytes
h, f = 3072, 8192
x = torch.randn(T, h, device="cuda").bfloat16(); w = torch.ones(h, device="cuda").bfloat16()
y = torch.empty_like(x); rstd = torch.empty(T, device="cuda"); dy = torch.randn_like(x); dres = torch.randn_like(x)
dx = torch.empty_like(x); parts = torch.empty(ops.rmsnorm_partials(T, h), h, device="cuda")
mem = {}
t = timeit(lambda: ops.rmsnorm_fwd(x, w, y, rstd)); mem["rmsnorm_fwd"] = (t, 2 * T * h * 2)
t = timeit(lambda: ops.rmsnorm_bwd(dy, x, w, rstd, dx, parts, dres=dres)); mem["rmsnorm_bwd"] = (t, 4 * T * h * 2)
gu = torch.randn(T, 2 * f, device="cuda").bfloat16(); act = torch.empty(T, f, device="cuda", dtype=torch.bfloat16)
t = timeit(lambda: ops.swiglu_fwd(gu, act)); mem["swiglu_fwd"] = (t, 3 * T * f * 2)
dgu = torch.empty_like(gu)
t = timeit(lambda: ops.swiglu_bwd(act, gu, dgu)); mem["swiglu_bwd"] = (t, 5 * T * f * 2)
qkr = torch.empty(T, (hq + hkv) * d, device="cuda", dtype=torch.bfloat16)
t = timeit(lambda: ops.rope(qkv, qkr, hq + hkv, d, 500000.0)); mem["rope"] = (t, 2 * T * (hq + hkv) * d * 2)
print(json.dumps({k: {"ms": round(v[0], 4), "GB/s": round(v[1] / v[0] / 1e6, 1)} for k, v in mem.items()}, indent=1))
