"""A/B of the attention-backward kernels (KPO_ATTN_BWD=2: 64-query steps, 3: 128-query steps) in
separate processes (the variant switch is read once per process), each checked against a torch fp32
reference of the same causal GQA attention.
python tools/attn_bwd_ab.py [--variants 2,3] [--shapes T:hq:hkv[:d],...]"""
import argparse
import json
import math
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(T, hq, hkv, reps, d=128):
    sys.path.insert(0, ROOT)
    import torch

    from paper_2601_17654_b200 import ops

    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(0)
    qkv = torch.randn(T, (hq + 2 * hkv) * d, device=dev, generator=g).bfloat16()
    q, k, v = qkv[:, :hq * d], qkv[:, hq * d:(hq + hkv) * d], qkv[:, (hq + hkv) * d:]
    o = torch.empty(T, hq * d, device=dev, dtype=torch.bfloat16)
    lse = torch.empty(hq, T, device=dev)
    scale = 1 / math.sqrt(d)
    ops.attn_fwd(q, k, v, o, lse, T, hq, hkv, d, scale)
    for _ in range(3):
        ops.attn_fwd(q, k, v, o, lse, T, hq, hkv, d, scale)
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    for _ in range(reps):
        ops.attn_fwd(q, k, v, o, lse, T, hq, hkv, d, scale)
    f1.record()
    torch.cuda.synchronize()
    fwd_ms = f0.elapsed_time(f1) / reps
    dout = torch.randn(T, hq * d, device=dev, generator=g).bfloat16()
    dqkv = torch.empty_like(qkv)
    ws = ops.attn_bwd_workspace(T, hq, hkv, d, dev)
    run = lambda: ops.attn_bwd(q, k, v, o, dout, lse, dqkv[:, :hq * d], dqkv[:, hq * d:(hq + hkv) * d],
                               dqkv[:, (hq + hkv) * d:], T, hq, hkv, d, scale, ws)
    for _ in range(3):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    fl = 2.5 * 2.0 * T * T * hq * d  # causal: 2 GEMMs x 2*T^2*hq*d / 2, backward 2.5x
    # torch fp32 reference
    qh = q.float().reshape(T, hq, d).transpose(0, 1).requires_grad_()
    kh = k.float().reshape(T, hkv, d).transpose(0, 1).requires_grad_()
    vh = v.float().reshape(T, hkv, d).transpose(0, 1).requires_grad_()
    rep = hq // hkv
    s = (qh @ kh.repeat_interleave(rep, 0).transpose(1, 2)) * scale
    s = s.masked_fill(torch.ones(T, T, device=dev, dtype=torch.bool).triu(1), float("-inf"))
    out = torch.softmax(s, -1) @ vh.repeat_interleave(rep, 0)
    out.backward(dout.float().reshape(T, hq, d).transpose(0, 1))
    rel = lambda a, b: float((a.float() - b).norm() / b.norm())
    errs = {"dq": rel(dqkv[:, :hq * d], qh.grad.transpose(0, 1).reshape(T, -1)),
            "dk": rel(dqkv[:, hq * d:(hq + hkv) * d], kh.grad.transpose(0, 1).reshape(T, -1)),
            "dv": rel(dqkv[:, (hq + hkv) * d:], vh.grad.transpose(0, 1).reshape(T, -1))}
    import hashlib
    run()  # one more call on the same inputs: a deterministic backward reproduces its bits
    digest = hashlib.sha256(dqkv.contiguous().view(torch.int16).cpu().numpy().tobytes()).hexdigest()[:16]
    print(json.dumps({"ms": round(ms, 4), "tflops": round(fl / ms / 1e9, 1), "fwd_ms": round(fwd_ms, 4),
                      "fwd_tflops": round(fl / 2.5 / fwd_ms / 1e9, 1),
                      "rel": {k: round(x, 5) for k, x in errs.items()}, "sha": digest}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variants", default="2,3")
    ap.add_argument("--shapes", default="4096:24:8,4096:4:1,4096:64:8,1000:8:2")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--child", default=None)
    a = ap.parse_args()
    if a.child:
        child(*[int(x) for x in a.child.split(":")[:3]], a.reps, *[int(x) for x in a.child.split(":")[3:]])
        return
    res = {}
    for shape in a.shapes.split(","):
        for var in a.variants.split(","):
            # "3+dv": variant 3 with the dV-before-dP MMA order (KPO_ATTN_BWD3_DVFIRST=1)
            # "2@base": variant 2 of the library at tools/ab/libkpo_base.so (an older build, same-box A/B)
            # "2+f2": also KPO_ATTN_FWD=2 (the forward variant the child times)
            var_b, *opts = var.split("+")
            v, _, lib = var_b.partition("@")
            env = dict(os.environ, KPO_ATTN_BWD=v)
            for o in opts:
                if o.startswith("f"):
                    env["KPO_ATTN_FWD"] = o[1:]
            if lib:
                env["KPO_LIB_PATH"] = os.path.join(ROOT, "tools", "ab", f"libkpo_{lib}.so")
            r = subprocess.run([sys.executable, __file__, "--child", shape, "--reps", str(a.reps)], env=env,
                               capture_output=True, text=True, timeout=240)
            try:
                res[f"{shape}/v{var}"] = json.loads(r.stdout.strip().splitlines()[-1])
            except Exception:
                res[f"{shape}/v{var}"] = {"error": (r.stderr or r.stdout)[-600:]}
            print(shape, var, res[f"{shape}/v{var}"], flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
