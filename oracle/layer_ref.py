"""CPU fp32 restatement of the partitioned transformer layer (TEST INFRASTRUCTURE ONLY).

PARITY UNPINNED: the reference ships no layer math — its kernels are abstract KernelSpecs
(reference workloads.py:38-93) — so this oracle restates the public Llama block the partitions
stand for (SURVEY.md §8c "Layer numerics"): RMSNorm -> QKV -> RoPE (rotate-half, theta) -> causal
GQA attention -> O (+residual) -> RMSNorm -> gate|up -> SwiGLU -> down (+residual), with autograd
for the gradients.  Collectives are emulated by the full (unsharded) computation: a TP rank's
all-reduced output equals the full layer output, and its weight gradients are slices of the full
gradients; FSDP ranks compute the full layer on their own tokens.

Used by tests/ (GPU parity at small sizes), smoke(), and bench.py's CPU baseline / --impl
reference leg (timed on the host cores with all threads).
"""

from __future__ import annotations

import math

import torch


def rmsnorm(x, w, eps):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w


def rope(x, heads, d, theta, pos0=0):
    T = x.shape[0]
    half = d // 2
    inv = theta ** (-(torch.arange(half, dtype=torch.float64) * 2.0 / d))
    ang = (torch.arange(T, dtype=torch.float64)[:, None] + pos0) * inv[None]
    c, s = ang.cos().to(x.dtype), ang.sin().to(x.dtype)
    xv = x.reshape(T, heads, d)
    a, b = xv[..., :half], xv[..., half:]
    return torch.cat([a * c[:, None] - b * s[:, None], b * c[:, None] + a * s[:, None]], -1).reshape(T, heads * d)


def attention(q, k, v, hq, hkv, d):
    T = q.shape[0]
    qh = q.reshape(T, hq, d).transpose(0, 1)
    kh = k.reshape(T, hkv, d).transpose(0, 1).repeat_interleave(hq // hkv, 0)
    vh = v.reshape(T, hkv, d).transpose(0, 1).repeat_interleave(hq // hkv, 0)
    s = (qh @ kh.transpose(1, 2)) / math.sqrt(d)
    mask = torch.ones(T, T, dtype=torch.bool).triu(1)
    s = s.masked_fill(mask, float("-inf"))
    p = torch.softmax(s, -1)
    return (p @ vh).transpose(0, 1).reshape(T, hq * d)


def layer_forward(x, W, cfg):
    """cfg: ModelConfig-like (hidden, ffn, n_heads, n_kv_heads, head_dim, rope_theta, norm_eps)."""
    hq, hkv, d, f = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.ffn
    xn1 = rmsnorm(x, W["g1"], cfg.norm_eps)
    qkv = xn1 @ W["wqkv"].t()
    qk = rope(qkv[:, :(hq + hkv) * d], hq + hkv, d, cfg.rope_theta)
    ao = attention(qk[:, :hq * d], qk[:, hq * d:], qkv[:, (hq + hkv) * d:], hq, hkv, d)
    h = x + ao @ W["wo"].t()
    xn2 = rmsnorm(h, W["g2"], cfg.norm_eps)
    gu = xn2 @ W["wgu"].t()
    act = torch.nn.functional.silu(gu[:, :f]) * gu[:, f:]
    return h + act @ W["wd"].t(), h


def layer_fwd_bwd(xs, dys, weights, cfg):
    """Forward + backward over the nanobatches `xs` (list of [T, h]) with upstream grads `dys`.
    Returns per-nanobatch outputs y, h, dx and the weight gradients summed over nanobatches."""
    W = {k: v.detach().float().clone().requires_grad_(True) for k, v in weights.items()}
    out = {"y": [], "h": [], "dx": []}
    for x, dy in zip(xs, dys):
        xr = x.detach().float().clone().requires_grad_(True)
        y, h = layer_forward(xr, W, cfg)
        y.backward(dy.float())
        out["y"].append(y.detach())
        out["h"].append(h.detach())
        out["dx"].append(xr.grad.detach())
    out["grads"] = {k: v.grad.detach() for k, v in W.items()}
    return out
