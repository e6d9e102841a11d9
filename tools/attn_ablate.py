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

# ---------------------------------------------------------------- peer points on the same box (library kernels)
peers = {}
qh = q.reshape(T, hq, d).transpose(0, 1).unsqueeze(0).contiguous().requires_grad_()
kh = k.reshape(T, hkv, d).transpose(0, 1).unsqueeze(0).contiguous().requires_grad_()
vh = v.reshape(T, hkv, d).transpose(0, 1).unsqueeze(0).contiguous().requires_grad_()
go = dout.reshape(T, hq, d).transpose(0, 1).unsqueeze(0).contiguous()
from torch.nn.attention import SDPBackend, sdpa_kernel
for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION),
                 ("efficient", SDPBackend.EFFICIENT_ATTENTION)):
    try:
        with sdpa_kernel([be]):
            out = torch.nn.functional.scaled_dot_product_attention(qh, kh, vh, is_causal=True, enable_gqa=True)
            tf = timeit(lambda: torch.nn.functional.scaled_dot_product_attention(qh, kh, vh, is_causal=True,
                                                                                 enable_gqa=True), reps=10)
            tb = timeit(lambda: torch.autograd.grad(out, (qh, kh, vh), go, retain_graph=True), reps=10)
        peers[name] = {"fwd_ms": round(tf, 4), "fwd_tflops": round(fl / 2.5 / tf / 1e9, 1), "bwd_ms": round(tb, 4),
                       "bwd_tflops": round(fl / tb / 1e9, 1)}
    except Exception as ex:  # backend unavailable for this shape / GPU
        peers[name] = f"unavailable: {type(ex).__name__}: {str(ex)[:120]}"
try:
    from flash_attn import flash_attn_func
    qf, kf, vf = (t.reshape(T, -1, d).unsqueeze(0).contiguous().requires_grad_() for t in (q, k, v))
    of = flash_attn_func(qf, kf, vf, causal=True)
    gof = dout.reshape(1, T, hq, d)
    tf = timeit(lambda: flash_attn_func(qf, kf, vf, causal=True), reps=10)
    tb = timeit(lambda: torch.autograd.grad(of, (qf, kf, vf), gof, retain_graph=True), reps=10)
    peers["flash_attn_pkg"] = {"fwd_ms": round(tf, 4), "fwd_tflops": round(fl / 2.5 / tf / 1e9, 1),
                               "bwd_ms": round(tb, 4), "bwd_tflops": round(fl / tb / 1e9, 1)}
except Exception as ex:
    peers["flash_attn_pkg"] = f"unavailable: {type(ex).__name__}: {str(ex)[:120]}"
try:  # FlashAttention-4 (CuTe DSL, tcgen05; vllm's vendored copy): the sm100-native peer
    from vllm.vllm_flash_attn.cute.interface import flash_attn_func as fa4
    qf, kf, vf = (t.reshape(T, -1, d).unsqueeze(0).contiguous().requires_grad_() for t in (q, k, v))
    of = fa4(qf, kf, vf, causal=True)
    of = of[0] if isinstance(of, tuple) else of
    gof = dout.reshape(1, T, hq, d)
    tf = timeit(lambda: fa4(qf, kf, vf, causal=True), reps=10)
    tb = timeit(lambda: torch.autograd.grad(of, (qf, kf, vf), gof, retain_graph=True), reps=10)
    peers["fa4_cute_sm100"] = {"fwd_ms": round(tf, 4), "fwd_tflops": round(fl / 2.5 / tf / 1e9, 1),
                               "bwd_ms": round(tb, 4), "bwd_tflops": round(fl / tb / 1e9, 1)}
except Exception as ex:
    peers["fa4_cute_sm100"] = f"unavailable: {type(ex).__name__}: {str(ex)[:160]}"
res["peers"] = peers
print(json.dumps(res))
