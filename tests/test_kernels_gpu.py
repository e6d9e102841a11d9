"""Numerics of the hand-written sm_100a kernels against plain PyTorch fp32 references."""
import math
import os

import pytest
import torch

pytestmark = pytest.mark.gpu


def rel_err(a, b):
    a = a.float()
    b = b.float()
    return ((a - b).norm() / b.norm().clamp_min(1e-12)).item()


@pytest.mark.parametrize("M,N,K", [(256, 256, 64), (128, 128, 128), (4096, 3072, 3072), (1000, 776, 520), (4096, 5120, 512), (3072, 8192, 256),
                                   (4096, 768, 4096), (384, 16384, 256),
                                   # Llama-3-70B layer GEMMs at T=4096 (config 3): gate|up, qkv, down / o,
                                   # and the gate|up weight-gradient shape
                                   (4096, 57344, 8192), (4096, 10240, 8192), (4096, 8192, 28672),
                                   (57344, 8192, 4096)])
@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, False), (True, True)])
def test_gemm_all_majors(cuda, M, N, K, a_mn, b_mn):
    from paper_2601_17654_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K)
    A = torch.randn((K, M) if a_mn else (M, K), device=cuda, generator=g).bfloat16()
    B = torch.randn((K, N) if b_mn else (N, K), device=cuda, generator=g).bfloat16()
    D = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    ops.gemm_raw(A, B, D, M, N, K, a_mn, b_mn)
    torch.cuda.synchronize()
    Af = A.float().t() if a_mn else A.float()
    Bf = B.float() if b_mn else B.float().t()
    ref = Af @ Bf
    assert rel_err(D, ref) < 8e-3


def test_gemm_residual_and_cap(cuda):
    from paper_2601_17654_b200 import ops
    M, N, K = 512, 1024, 512
    x = torch.randn(M, K, device=cuda).bfloat16()
    w = torch.randn(N, K, device=cuda).bfloat16()
    r = torch.randn(M, N, device=cuda).bfloat16()
    out = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    for cap in (0, 1, 7, 148):
        ops.linear(x, w, out, residual=r, max_ctas=cap)
        torch.cuda.synchronize()
        ref = x.float() @ w.float().t() + r.float()
        assert rel_err(out, ref) < 8e-3


def test_gemm_replay_resets_scheduler(cuda):
    from paper_2601_17654_b200 import ops
    M, N, K = 1024, 1024, 256
    x = torch.randn(M, K, device=cuda).bfloat16()
    w = torch.randn(N, K, device=cuda).bfloat16()
    out = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    ref = (x.float() @ w.float().t())
    for _ in range(20):
        out.zero_()
        ops.linear(x, w, out)
    torch.cuda.synchronize()
    assert rel_err(out, ref) < 8e-3
    assert int(ops._default_sched[0].buf.abs().sum()) == 0


@pytest.mark.parametrize("rows,cols", [(4096, 3072), (100, 1024), (33, 8192), (7, 520), (8192, 2048), (5, 3072), (1001, 3072)])
def test_rmsnorm(cuda, rows, cols):
    from paper_2601_17654_b200 import ops
    x = torch.randn(rows, cols, device=cuda).bfloat16()
    w = (1 + 0.1 * torch.randn(cols, device=cuda)).bfloat16()
    y = torch.empty_like(x)
    rstd = torch.empty(rows, device=cuda)
    ops.rmsnorm_fwd(x, w, y, rstd, eps=1e-5)
    xf = x.float().requires_grad_()
    wf = w.float().requires_grad_()
    ref = xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + 1e-5) * wf
    assert rel_err(y, ref) < 5e-3
    dy = torch.randn_like(x)
    dres = torch.randn_like(x)
    dx = torch.empty_like(x)
    parts = torch.empty(ops.rmsnorm_partials(rows, cols), cols, device=cuda)
    ops.rmsnorm_bwd(dy, x, w, rstd, dx, parts, dres=dres)
    dw = torch.empty(cols, device=cuda, dtype=torch.bfloat16)
    ops.colsum(parts, dw)
    ref.backward(dy.float())
    assert rel_err(dx, xf.grad + dres.float()) < 1e-2
    assert rel_err(dw, wf.grad) < 1e-2


def _rope_ref(x, heads, d, theta, inverse=False):
    T = x.shape[0]
    half = d // 2
    inv = theta ** (-(torch.arange(half, dtype=torch.float64, device=x.device) * 2 / d))
    ang = torch.arange(T, dtype=torch.float64, device=x.device)[:, None] * inv[None]
    c, s = ang.cos().float(), ang.sin().float()
    if inverse:
        s = -s
    xv = x.float().view(T, heads, d)
    a, b = xv[..., :half], xv[..., half:]
    out = torch.cat([a * c[:, None] - b * s[:, None], b * c[:, None] + a * s[:, None]], -1)
    return out.view(T, heads * d)


def test_rope_strided(cuda):
    from paper_2601_17654_b200 import ops
    T, hq, hkv, d = 300, 6, 2, 128
    qkv = torch.randn(T, (hq + 2 * hkv) * d, device=cuda).bfloat16()
    out = torch.empty(T, (hq + hkv) * d, device=cuda, dtype=torch.bfloat16)
    ops.rope(qkv, out, hq + hkv, d, 500000.0)
    ref = _rope_ref(qkv[:, : (hq + hkv) * d], hq + hkv, d, 500000.0)
    assert rel_err(out, ref) < 5e-3
    back = torch.empty_like(out)
    ops.rope(out, back, hq + hkv, d, 500000.0, inverse=True)
    assert rel_err(back, qkv[:, : (hq + hkv) * d]) < 1e-2


def test_swiglu(cuda):
    from paper_2601_17654_b200 import ops
    rows, ffn = 513, 1024
    gu = torch.randn(rows, 2 * ffn, device=cuda).bfloat16()
    act = torch.empty(rows, ffn, device=cuda, dtype=torch.bfloat16)
    ops.swiglu_fwd(gu, act)
    guf = gu.float().requires_grad_()
    ref = torch.nn.functional.silu(guf[:, :ffn]) * guf[:, ffn:]
    assert rel_err(act, ref) < 5e-3
    dact = torch.randn_like(act)
    dgu = torch.empty_like(gu)
    ops.swiglu_bwd(dact, gu, dgu)
    ref.backward(dact.float())
    assert rel_err(dgu, guf.grad) < 1e-2


def _attn_ref(q, k, v, hq, hkv, d, causal=True):
    T = q.shape[0]
    qf = q.float().view(T, hq, d).transpose(0, 1)
    kf = k.float().view(T, hkv, d).transpose(0, 1).repeat_interleave(hq // hkv, 0)
    vf = v.float().view(T, hkv, d).transpose(0, 1).repeat_interleave(hq // hkv, 0)
    return torch.nn.functional.scaled_dot_product_attention(qf, kf, vf, is_causal=causal)


@pytest.mark.parametrize("T,hq,hkv,d", [(256, 4, 1, 128), (1000, 6, 2, 128), (512, 8, 8, 64), (4096, 3, 1, 128),
                                      (2048, 16, 16, 64),    # GPT layer, config 0 (head_dim 64)
                                      (4096, 24, 8, 128),
                                      (4096, 4, 1, 128),     # Llama-3-8B TP8 per-rank heads (config 2)
                                      (4096, 64, 8, 128)])   # Llama-3-70B (config 3)
def test_attention_fwd_bwd(cuda, T, hq, hkv, d):
    from paper_2601_17654_b200 import ops
    torch.manual_seed(T + hq)
    qkv = torch.randn(T, (hq + 2 * hkv) * d, device=cuda).bfloat16()
    q = qkv[:, : hq * d]
    k = qkv[:, hq * d:(hq + hkv) * d]
    v = qkv[:, (hq + hkv) * d:]
    o = torch.empty(T, hq * d, device=cuda, dtype=torch.bfloat16)
    lse = torch.empty(hq, T, device=cuda)
    scale = 1.0 / math.sqrt(d)
    ops.attn_fwd(q, k, v, o, lse, T, hq, hkv, d, scale)
    qf, kf, vf = (t.float().requires_grad_() for t in (q, k, v))
    ref = _attn_ref(qf, kf, vf, hq, hkv, d)  # [hq, T, d]
    assert rel_err(o.view(T, hq, d).transpose(0, 1), ref) < 1e-2
    dout = torch.randn(T, hq * d, device=cuda).bfloat16()
    dqkv = torch.empty_like(qkv)
    dq, dk, dv = dqkv[:, : hq * d], dqkv[:, hq * d:(hq + hkv) * d], dqkv[:, (hq + hkv) * d:]
    ws = ops.attn_bwd_workspace(T, hq, hkv, d, cuda)
    ops.attn_bwd(q, k, v, o, dout, lse, dq, dk, dv, T, hq, hkv, d, scale, ws)
    ref.backward(dout.float().view(T, hq, d).transpose(0, 1))
    assert rel_err(dq, qf.grad) < 2e-2
    assert rel_err(dk, kf.grad) < 2e-2
    assert rel_err(dv, vf.grad) < 2e-2


@pytest.mark.parametrize("T,hq,hkv", [(1024, 4, 1), (2048, 8, 2)])
def test_attention_fwd_lazy_rescale_divergent_rows(cuda, T, hq, hkv):
    """Scores whose row maxima jump by > 2^8 on later key tiles for SOME rows only: exercises the
    forward's lazy O-rescale path with warp-divergent decisions (regression: a per-lane predicate
    around warp-collective tcgen05.ld/st hung the kernel on real layer data)."""
    from paper_2601_17654_b200 import ops
    d = 128
    torch.manual_seed(7)
    qkv = torch.randn(T, (hq + 2 * hkv) * d, device=cuda)
    ramp = (1.0 + torch.arange(T, device=cuda, dtype=torch.float32) / 128.0)[:, None]
    qkv[:, hq * d:(hq + hkv) * d] *= ramp                       # keys grow with position
    qkv[:, :hq * d] *= torch.rand(T, 1, device=cuda) * 4.0       # per-row query scale: some rows jump, some not
    qkv = qkv.bfloat16()
    q, k, v = qkv[:, :hq * d], qkv[:, hq * d:(hq + hkv) * d], qkv[:, (hq + hkv) * d:]
    o = torch.empty(T, hq * d, device=cuda, dtype=torch.bfloat16)
    lse = torch.empty(hq, T, device=cuda)
    ops.attn_fwd(q, k, v, o, lse, T, hq, hkv, d, 1.0 / math.sqrt(d))
    torch.cuda.synchronize()
    ref = _attn_ref(q.float(), k.float(), v.float(), hq, hkv, d)
    assert rel_err(o.view(T, hq, d).transpose(0, 1), ref) < 1e-2


@pytest.mark.parametrize("M,N,rope_cols", [(4096, 5120, 4096), (1000, 768, 512), (300, 384, 384)])
def test_gemm_rope_epilogue(cuda, M, N, rope_cols):
    """Fused rotary epilogue of the QKV projection vs fp32 GEMM + rotate-half of the q / k heads."""
    from paper_2601_17654_b200 import ops
    K, d, theta = 512, 128, 500000.0
    g = torch.Generator(device="cuda").manual_seed(M + N)
    x = torch.randn(M, K, device=cuda, generator=g).bfloat16()
    w = torch.randn(N, K, device=cuda, generator=g).bfloat16()
    out = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    table = ops.rope_table(M, d, theta, cuda)
    ops.linear_rope(x, w, out, table, rope_cols, d)
    torch.cuda.synchronize()
    ref = x.float() @ w.float().t()
    half = d // 2
    inv = theta ** (-(torch.arange(half, dtype=torch.float64, device=cuda) * 2 / d))
    ang = torch.arange(M, dtype=torch.float64, device=cuda)[:, None] * inv[None]
    c, s_ = ang.cos().float(), ang.sin().float()
    qk = ref[:, :rope_cols].view(M, rope_cols // d, d)
    a, b = qk[..., :half], qk[..., half:]
    rot = torch.cat([a * c[:, None] - b * s_[:, None], b * c[:, None] + a * s_[:, None]], -1).view(M, rope_cols)
    ref = torch.cat([rot, ref[:, rope_cols:]], 1)
    assert rel_err(out, ref) < 8e-3
    # table entries: fp32 angle arithmetic like the separate rope kernel (angle rounding ~ pos * 2^-24)
    assert torch.allclose(table[:, :, 0], c, atol=1e-3) and torch.allclose(table[:, :, 1], s_, atol=1e-3)


@pytest.mark.parametrize("M,ffn,K", [(256, 128, 256), (1000, 1024, 512), (4096, 1792, 4096)])
def test_gemm_swiglu_epilogue(cuda, M, ffn, K):
    """Fused SwiGLU epilogue of the gate|up projection: gu (blocked layout) equals the plain GEMM over the
    blocked weights bit-exactly, and act equals the separate swiglu kernel on that gu bit-exactly
    (both compute bf16 g * sigmoid(bf16 g) * bf16 u in fp32); act vs the fp32 reference within bf16
    tolerance."""
    from paper_2601_17654_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(M + ffn)
    x = torch.randn(M, K, device=cuda, generator=g).bfloat16()
    w = (torch.randn(2 * ffn, K, device=cuda, generator=g) * 0.05).bfloat16()
    wb = ops.interleave_gate_up(w)
    assert torch.equal(ops.deinterleave_gate_up(wb), w)
    gu = torch.empty(M, 2 * ffn, device=cuda, dtype=torch.bfloat16)
    act = torch.empty(M, ffn, device=cuda, dtype=torch.bfloat16)
    ops.linear_swiglu(x, wb, gu, act)
    gu_plain = torch.empty_like(gu)
    ops.linear(x, wb, gu_plain)
    act_sep = torch.empty_like(act)
    ops.swiglu_fwd(gu_plain, act_sep, block=ops.SWIGLU_BLOCK)
    torch.cuda.synchronize()
    assert torch.equal(gu, gu_plain)
    assert torch.equal(act, act_sep)
    ref_gu = x.float() @ w.float().t()
    ref = torch.nn.functional.silu(ref_gu[:, :ffn]) * ref_gu[:, ffn:]
    assert rel_err(act, ref) < 1e-2
    assert rel_err(ops.deinterleave_gate_up(gu.t()).t(), ref_gu) < 8e-3


@pytest.mark.parametrize("M,ffn,K", [(256, 256, 256), (1000, 1024, 512), (4096, 1792, 4096)])
def test_gemm_swiglu_bwd_epilogue(cuda, M, ffn, K):
    """Fused SwiGLU backward in the down dgrad: dgu equals linear_dgrad followed by the blocked swiglu_bwd
    kernel bit-exactly (dact rounded to bf16 first, same expressions); and vs autograd in fp32."""
    from paper_2601_17654_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(M + ffn + K)
    dy = torch.randn(M, K, device=cuda, generator=g).bfloat16()
    wd = (torch.randn(K, ffn, device=cuda, generator=g) * 0.05).bfloat16()
    gu = torch.randn(M, 2 * ffn, device=cuda, generator=g).bfloat16()
    dgu = torch.full((M, 2 * ffn), float("nan"), device=cuda, dtype=torch.bfloat16)
    ops.linear_dgrad_swiglu_bwd(dy, wd, gu, dgu)
    dact = torch.empty(M, ffn, device=cuda, dtype=torch.bfloat16)
    ops.linear_dgrad(dy, wd, dact)
    dgu_sep = torch.empty_like(gu)
    ops.swiglu_bwd(dact, gu, dgu_sep, block=ops.SWIGLU_BLOCK)
    torch.cuda.synchronize()
    assert torch.equal(dgu, dgu_sep)
    guh = ops.deinterleave_gate_up(gu.t()).t().float().requires_grad_()
    act = torch.nn.functional.silu(guh[:, :ffn]) * guh[:, ffn:]
    act.backward(dy.float() @ wd.float())
    assert rel_err(ops.deinterleave_gate_up(dgu.t()).t(), guh.grad) < 1e-2


def test_swiglu_blocked_layout(cuda):
    """The blocked gate|up layout (block 128) gives the same act / dgu as the halves layout, permuted."""
    from paper_2601_17654_b200 import ops
    rows, ffn = 300, 768
    gu = torch.randn(rows, 2 * ffn, device=cuda).bfloat16()
    gub = ops.interleave_gate_up(gu.t()).t().contiguous()
    act, actb = (torch.empty(rows, ffn, device=cuda, dtype=torch.bfloat16) for _ in range(2))
    ops.swiglu_fwd(gu, act)
    ops.swiglu_fwd(gub, actb, block=128)
    dact = torch.randn_like(act)
    dgu, dgub = torch.empty_like(gu), torch.empty_like(gu)
    ops.swiglu_bwd(dact, gu, dgu)
    ops.swiglu_bwd(dact, gub, dgub, block=128)
    torch.cuda.synchronize()
    assert torch.equal(act, actb)
    assert torch.equal(ops.deinterleave_gate_up(dgub.t()).t(), dgu)


@pytest.mark.parametrize("T,hq,hkv", [(1024, 8, 2), (512, 4, 1)])
def test_attention_bwd_rope_fused(cuda, T, hq, hkv):
    """attn_bwd with the fused inverse rotary (q / k rotated by the QKV epilogue) equals attn_bwd followed
    by the separate inverse rope kernel on dq / dk (both split-group and grouped dK paths)."""
    from paper_2601_17654_b200 import ops
    d, theta = 128, 500000.0
    g = torch.Generator(device="cuda").manual_seed(T + hq)
    qkv = torch.randn(T, (hq + 2 * hkv) * d, device=cuda, generator=g).bfloat16()
    qd = (hq + hkv) * d
    q, k, v = qkv[:, :hq * d], qkv[:, hq * d:qd], qkv[:, qd:]
    o = torch.empty(T, hq * d, device=cuda, dtype=torch.bfloat16)
    lse = torch.empty(hq, T, device=cuda)
    scale = 1 / math.sqrt(d)
    ops.attn_fwd(q, k, v, o, lse, T, hq, hkv, d, scale)
    dout = torch.randn_like(o)
    ws = ops.attn_bwd_workspace(T, hq, hkv, d, cuda)
    table = ops.rope_table(T, d, theta, cuda)
    d1 = torch.empty_like(qkv)
    ops.attn_bwd(q, k, v, o, dout, lse, d1[:, :hq * d], d1[:, hq * d:qd], d1[:, qd:], T, hq, hkv, d, scale, ws,
                 rope_table=table)
    d0 = torch.empty_like(qkv)
    ops.attn_bwd(q, k, v, o, dout, lse, d0[:, :hq * d], d0[:, hq * d:qd], d0[:, qd:], T, hq, hkv, d, scale, ws)
    ref = torch.empty_like(qkv)
    ref[:, qd:] = d0[:, qd:]
    ops.rope(d0, ref, hq + hkv, d, theta, inverse=True)
    torch.cuda.synchronize()
    assert rel_err(d1[:, :qd], ref[:, :qd]) < 1e-2
    assert rel_err(d1[:, qd:], ref[:, qd:]) < 1e-2


@pytest.mark.parametrize("shape", ["1024:6:2", "2048:4:1", "512:8:8:64"])
def test_attention_bwd_variants_match_reference(cuda, shape):
    """Every attention-backward implementation (selected per process by KPO_ATTN_BWD: 2 = the 64-query
    single kernel, 3 = the 128-query single kernel, 4 = the dQ + dK/dV two-kernel default) against the
    same torch fp32 reference (tools/attn_bwd_ab.py runs each in its own process)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    variants = "3,4" if shape.endswith(":64") else "2,3,4"
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "attn_bwd_ab.py"), "--variants", variants,
                        "--shapes", shape, "--reps", "2"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for key, v in res.items():
        assert "rel" in v, (key, v)
        assert all(e < 2e-2 for e in v["rel"].values()), (key, v)


def test_attention_bwd_two_kernel_path_is_deterministic(cuda):
    """KPO_ATTN_BWD=4 (dQ kernel + dK/dV kernel) reduces nothing across CTAs in grouped mode, so two
    processes on the same seeded inputs produce bit-identical dq / dk / dv."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, KPO_ATTN_BWD="4", KPO_ATTN_BWD_SPLIT="0")  # grouped mode: no dK / dV atomics
    shas = []
    for _ in range(2):
        r = subprocess.run([sys.executable, os.path.join(root, "tools", "attn_bwd_ab.py"), "--child", "2048:8:2",
                            "--reps", "2"], capture_output=True, text=True, timeout=600, env=env)
        assert r.returncode == 0, r.stderr[-2000:]
        line = json.loads(r.stdout.strip().splitlines()[-1])
        assert all(e < 2e-2 for e in line["rel"].values()), line
        shas.append(line["sha"])
    assert shas[0] == shas[1], shas

