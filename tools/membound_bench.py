"""HBM-bound launch units at the layer's shapes (config 1: T 4096, h 3072, ffn 8192), each call timed
alone with CUDA events after writing a 512 MB buffer (inputs come from HBM, as in the step).
Measurement only.  python tools/membound_bench.py [--T 4096 --h 3072 --f 8192]"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_17654_b200 import ops

ap = argparse.ArgumentParser()
ap.add_argument("--T", type=int, default=4096)
ap.add_argument("--h", type=int, default=3072)
ap.add_argument("--f", type=int, default=8192)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
T, h, f = a.T, a.h, a.f
dev = "cuda"
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
bf = dict(dtype=torch.bfloat16, device=dev)


def timed(fn):
    """(flush + fn) x reps minus flush x reps, one event pair each: below the ~2 us event granularity."""
    def run(with_fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(a.reps):
            flush.fill_(i & 0xFF)
            if with_fn:
                fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)
    fn(); run(True); run(False)
    return (run(True) - run(False)) / a.reps


x = torch.randn(T, h, **bf); w = torch.randn(h, **bf); y = torch.empty_like(x)
rstd = torch.empty(T, dtype=torch.float32, device=dev)
dy = torch.randn(T, h, **bf); dres = torch.randn(T, h, **bf); dx = torch.empty_like(x)
parts = torch.empty(ops.rmsnorm_partials(T, h), h, device=dev)
gu = torch.randn(T, 2 * f, **bf); act = torch.empty(T, f, **bf); dact = torch.randn(T, f, **bf)
dgu = torch.empty_like(gu)
res = {}
ops.rmsnorm_fwd(x, w, y, rstd)
for name, fn, nbytes in (
        ("rmsnorm_fwd", lambda: ops.rmsnorm_fwd(x, w, y, rstd), 2 * T * h * 2),
        ("rmsnorm_bwd", lambda: ops.rmsnorm_bwd(dy, x, w, rstd, dx, parts, dres=dres), 4 * T * h * 2),
        ("swiglu_fwd", lambda: ops.swiglu_fwd(gu, act), 3 * T * f * 2),
        ("swiglu_bwd", lambda: ops.swiglu_bwd(dact, gu, dgu), 5 * T * f * 2)):
    ms = timed(fn)
    res[name] = {"us": round(ms * 1e3, 2), "GB/s": round(nbytes / ms / 1e6, 0)}
print(json.dumps(res))
