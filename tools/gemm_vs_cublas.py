"""One GEMM shape, kpo tcgen05 kernel then cuBLAS (torch.matmul), for side-by-side ncu captures.
python tools/gemm_vs_cublas.py [M N K]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2601_17654_b200 import ops

M, N, K = (int(x) for x in (sys.argv[1:4] if len(sys.argv) >= 4 else (4096, 5120, 3072)))
A = torch.randn(M, K, device="cuda").bfloat16()
B = torch.randn(N, K, device="cuda").bfloat16()
D = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    ops.gemm_raw(A, B, D, M, N, K, False, False)
    torch.matmul(A, B.t(), out=D)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
ops.gemm_raw(A, B, D, M, N, K, False, False)
torch.matmul(A, B.t(), out=D)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
