"""All layer GEMM shapes (config 2, T=4096) standalone: kpo tcgen05 vs cuBLAS (torch.matmul)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_17654_b200 import ops

def timeit(fn, reps=20, warm=3):
    for _ in range(warm): fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

import argparse
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
args = ap.parse_args()
T = 4096
if args.config == 1:
    h, f, qkv, hd = 3072, 8192, 5120, 3072
elif args.config == 2:  # Llama-3-8B TP8, per rank
    h, f, qkv, hd = 4096, 1792, 768, 512
else:  # Llama-3-70B FSDP8
    h, f, qkv, hd = 8192, 28672, 10240, 8192
shapes = [  # name, M, N, K, a_mn, b_mn
    ("linear_qkv", T, qkv, h, 0, 0), ("linear_proj", T, h, hd, 0, 0), ("linear_up", T, 2 * f, h, 0, 0),
    ("linear_down", T, h, f, 0, 0), ("down_dgrad", T, f, h, 0, 1), ("down_wgrad", h, f, T, 1, 1),
    ("gu_dgrad", T, h, 2 * f, 0, 1), ("gu_wgrad", 2 * f, h, T, 1, 1), ("o_dgrad", T, hd, h, 0, 1),
    ("o_wgrad", h, hd, T, 1, 1), ("qkv_dgrad", T, h, qkv, 0, 1), ("qkv_wgrad", qkv, h, T, 1, 1)]
out = {}
tot_k = tot_c = 0.0
for name, M, N, K, amn, bmn in shapes:
    A = torch.randn((K, M) if amn else (M, K), device="cuda").bfloat16()
    B = torch.randn((K, N) if bmn else (N, K), device="cuda").bfloat16()
    D = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    tk = timeit(lambda: ops.gemm_raw(A, B, D, M, N, K, bool(amn), bool(bmn)))
    At = A.t() if amn else A
    Bt = B if bmn else B.t()
    tc = timeit(lambda: torch.matmul(At, Bt, out=D))
    fl = 2.0 * M * N * K
    out[name] = {"kpo_ms": round(tk, 4), "kpo_tflops": round(fl / tk / 1e9, 1), "cublas_ms": round(tc, 4),
                 "cublas_tflops": round(fl / tc / 1e9, 1), "ratio": round(tc / tk, 3)}
    tot_k += tk; tot_c += tc
out["total"] = {"kpo_ms": round(tot_k, 4), "cublas_ms": round(tot_c, 4), "ratio": round(tot_c / tot_k, 3)}
print(json.dumps(out, indent=1))
