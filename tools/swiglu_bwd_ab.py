"""Down-projection dgrad with and without the fused SwiGLU backward epilogue at config-1 shapes
(T 4096, h 3072, ffn 8192), CUDA events over back-to-back calls.  Measurement only."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_17654_b200 import ops
T, h, f = 4096, 3072, 8192
bf = dict(dtype=torch.bfloat16, device="cuda")
dy = torch.randn(T, h, **bf); wd = torch.randn(h, f, **bf) * 0.02; gu = torch.randn(T, 2 * f, **bf)
dgu = torch.empty_like(gu); dact = torch.empty(T, f, **bf)


def t(fn, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps * 1e3, 1)


print(json.dumps({"dgrad_us": t(lambda: ops.linear_dgrad(dy, wd, dact)),
                  "swiglu_bwd_us": t(lambda: ops.swiglu_bwd(dact, gu, dgu, block=128)),
                  "fused_us": t(lambda: ops.linear_dgrad_swiglu_bwd(dy, wd, gu, dgu))}))
