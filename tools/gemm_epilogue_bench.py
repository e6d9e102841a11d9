"""GEMM epilogue cost: the layer's residual / accumulate GEMM shapes with and without the fused C
input (kpo tcgen05 kernels, CUDA events).  python tools/gemm_epilogue_bench.py"""
import json
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


T, h, f = 4096, 3072, 8192
out = {}
for name, M, N, K in (("linear_proj", T, h, h), ("linear_down", T, h, f)):
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = torch.randn(N, K, device="cuda").bfloat16()
    r = torch.randn(M, N, device="cuda").bfloat16()
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    a = timeit(lambda: ops.linear(x, w, y))
    b = timeit(lambda: ops.linear(x, w, y, residual=r))
    out[name] = {"plain_ms": round(a, 4), "residual_ms": round(b, 4)}
for name, N, K in (("o_wgrad", h, h), ("down_wgrad", h, f)):
    dy = torch.randn(T, N, device="cuda").bfloat16()
    xx = torch.randn(T, K, device="cuda").bfloat16()
    dw = torch.empty(N, K, device="cuda", dtype=torch.bfloat16)
    acc = torch.randn(N, K, device="cuda").bfloat16()
    a = timeit(lambda: ops.linear_wgrad(dy, xx, dw))
    b = timeit(lambda: ops.linear_wgrad(dy, xx, dw, accumulate=acc))
    out[name] = {"plain_ms": round(a, 4), "accumulate_ms": round(b, 4)}
print(json.dumps(out))
