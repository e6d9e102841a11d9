"""Thin torch-tensor front end over libkpo.so.

PyTorch only owns memory and streams here; every op below is one or more hand-written sm_100a
kernels reached through the C ABI (include/kpo.h).  There is no eager/PyTorch fallback: a CPU
tensor or a missing library raises.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib

BF16 = torch.bfloat16


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _need_cuda(*ts: torch.Tensor | None) -> None:
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("kpo ops take CUDA tensors only (no CPU fallback)")


# ------------------------------------------------------------------ RMSNorm
def rmsnorm_fwd(x: torch.Tensor, w: torch.Tensor, y: torch.Tensor, rstd: torch.Tensor, eps: float = 1e-5,
                stream=None) -> None:
    _need_cuda(x, w, y, rstd)
    rows, cols = x.shape
    _lib.call("kpo_rmsnorm_fwd", _ptr(x), _ptr(w), _ptr(y), _ptr(rstd), rows, cols, ctypes.c_float(eps),
              _stream(stream))


def rmsnorm_partials(rows: int, cols: int) -> int:
    n = ctypes.c_int64(0)
    _lib.call("kpo_rmsnorm_bwd_partial_rows", rows, cols, ctypes.byref(n))
    return n.value


def rmsnorm_bwd(dy, x, w, rstd, dx, dw_partial, dres=None, stream=None) -> None:
    _need_cuda(dy, x, w, rstd, dx, dw_partial, dres)
    rows, cols = x.shape
    _lib.call("kpo_rmsnorm_bwd", _ptr(dy), _ptr(x), _ptr(w), _ptr(rstd), _ptr(dres), _ptr(dx), _ptr(dw_partial),
              rows, cols, _stream(stream))


def colsum(partial: torch.Tensor, out: torch.Tensor, stream=None) -> None:
    _need_cuda(partial, out)
    rows, cols = partial.shape
    _lib.call("kpo_colsum_f32_to_bf16", _ptr(partial), _ptr(out), rows, cols, _stream(stream))


# ------------------------------------------------------------------ RoPE / SwiGLU
def rope(inp: torch.Tensor, out: torch.Tensor, heads: int, head_dim: int, theta: float, pos0: int = 0,
         inverse: bool = False, stream=None) -> None:
    """inp/out: 2-D views [tokens, >= heads*head_dim] (row strides may differ)."""
    _need_cuda(inp, out)
    tokens = inp.shape[0]
    _lib.call("kpo_rope", _ptr(inp), inp.stride(0), _ptr(out), out.stride(0), tokens, heads, head_dim,
              ctypes.c_float(theta), pos0, int(inverse), _stream(stream))


def swiglu_fwd(gu: torch.Tensor, act: torch.Tensor, stream=None, block: int = 0) -> None:
    _need_cuda(gu, act)
    rows, ffn = act.shape
    _lib.call("kpo_swiglu_fwd_blocked", _ptr(gu), _ptr(act), rows, ffn, block, _stream(stream))


def swiglu_bwd(dact: torch.Tensor, gu: torch.Tensor, dgu: torch.Tensor, stream=None, block: int = 0) -> None:
    """block = 0: gu = [gate | up] halves; block > 0: the blocked layout of linear_swiglu."""
    _need_cuda(dact, gu, dgu)
    rows, ffn = dact.shape
    _lib.call("kpo_swiglu_bwd_blocked", _ptr(dact), _ptr(gu), _ptr(dgu), rows, ffn, block, _stream(stream))


# gate / up block of the fused gate|up projection's weight order (kpo_gemm_swiglu)
SWIGLU_BLOCK = 128


def interleave_gate_up(w: torch.Tensor, block: int = SWIGLU_BLOCK) -> torch.Tensor:
    """[gate (f rows); up (f rows)] -> 128-row blocks g0, u0, g1, u1, ... (rows of any trailing shape)."""
    f = w.shape[0] // 2
    tail = w.shape[1:]
    return w.reshape(2, f // block, block, *tail).transpose(0, 1).reshape(2 * f, *tail).contiguous()


def deinterleave_gate_up(w: torch.Tensor, block: int = SWIGLU_BLOCK) -> torch.Tensor:
    f = w.shape[0] // 2
    tail = w.shape[1:]
    return w.reshape(f // block, 2, block, *tail).transpose(0, 1).reshape(2 * f, *tail).contiguous()


def linear_swiglu(x: torch.Tensor, w_blocked: torch.Tensor, gu: torch.Tensor, act: torch.Tensor,
                  max_ctas: int = 0, sched: int | None = None, stream=None) -> None:
    """gu = x @ w_blocked^T and act = silu(gate) * up in one GEMM (w_blocked = interleave_gate_up(w))."""
    _need_cuda(x, w_blocked, gu, act)
    M, K = x.shape
    N = w_blocked.shape[0]
    if sched is None:
        sched = default_sched(x.device)
    _lib.call("kpo_gemm_swiglu", _ptr(x), _ptr(w_blocked), _ptr(gu), _ptr(act), M, N, K, x.stride(0),
              w_blocked.stride(0), gu.stride(0), act.stride(0), max_ctas, sched, _stream(stream))


# ------------------------------------------------------------------ GEMM
class GemmScheduler:
    """Device-resident tile-scheduler words (int32[2] per concurrently running GEMM)."""

    def __init__(self, device, slots: int = 64):
        self.buf = torch.zeros(slots * 2, dtype=torch.int32, device=device)
        self.slots = slots
        self._next = 0

    def slot(self) -> int:
        i = self._next % self.slots
        self._next += 1
        return self.buf.data_ptr() + 8 * i


_default_sched: dict[int, GemmScheduler] = {}


def default_sched(device) -> int:
    idx = torch.device(device).index or 0
    if idx not in _default_sched:
        _default_sched[idx] = GemmScheduler(torch.device("cuda", idx), slots=1)
    return _default_sched[idx].buf.data_ptr()


def gemm_raw(A: torch.Tensor, B: torch.Tensor, D: torch.Tensor, M: int, N: int, K: int, a_mn: bool, b_mn: bool,
             C: torch.Tensor | None = None, max_ctas: int = 0, sched: int | None = None, stream=None) -> None:
    _need_cuda(A, B, D, C)
    lda, ldb, ldd = A.stride(0), B.stride(0), D.stride(0)
    if sched is None:
        sched = default_sched(A.device)
    _lib.call("kpo_gemm", _ptr(A), _ptr(B), _ptr(D), _ptr(C), M, N, K, int(a_mn), int(b_mn), lda, ldb, ldd,
              max_ctas, sched, _stream(stream))


def linear(x: torch.Tensor, w: torch.Tensor, out: torch.Tensor, residual: torch.Tensor | None = None,
           **kw) -> None:
    """out[M,N] = x[M,K] @ w[N,K]^T (+ residual) — forward (TN)."""
    M, K = x.shape
    N = w.shape[0]
    gemm_raw(x, w, out, M, N, K, False, False, C=residual, **kw)


def rope_table(tokens: int, head_dim: int, theta: float, device, pos0: int = 0, stream=None) -> torch.Tensor:
    """fp32 [tokens, head_dim/2, 2] (cos, sin) table for linear_rope."""
    t = torch.empty(tokens, head_dim // 2, 2, dtype=torch.float32, device=device)
    _lib.call("kpo_rope_table", tokens, head_dim, ctypes.c_float(theta), pos0, _ptr(t), _stream(stream))
    return t


def linear_rope(x: torch.Tensor, w: torch.Tensor, out: torch.Tensor, table: torch.Tensor, rope_cols: int,
                head_dim: int = 128, max_ctas: int = 0, sched: int | None = None, stream=None) -> None:
    """out = x @ w^T with the rotary embedding applied to output columns [0, rope_cols) in the epilogue."""
    _need_cuda(x, w, out, table)
    M, K = x.shape
    N = w.shape[0]
    if sched is None:
        sched = default_sched(x.device)
    _lib.call("kpo_gemm_rope", _ptr(x), _ptr(w), _ptr(out), M, N, K, x.stride(0), w.stride(0), out.stride(0),
              max_ctas, sched, _ptr(table), rope_cols, head_dim, _stream(stream))


def linear_dgrad_swiglu_bwd(dy: torch.Tensor, w: torch.Tensor, gu: torch.Tensor, dgu: torch.Tensor,
                            max_ctas: int = 0, sched: int | None = None, stream=None) -> None:
    """dgu = swiglu_bwd(dy @ w, gu) in one GEMM (gu / dgu in the blocked order of linear_swiglu;
    w = the down weight [hidden, ffn])."""
    _need_cuda(dy, w, gu, dgu)
    M, K = dy.shape
    N = w.shape[1]
    if sched is None:
        sched = default_sched(dy.device)
    _lib.call("kpo_gemm_swiglu_bwd", _ptr(dy), _ptr(w), _ptr(gu), _ptr(dgu), M, N, K, dy.stride(0), w.stride(0),
              gu.stride(0), dgu.stride(0), max_ctas, sched, _stream(stream))


def linear_dgrad(dy: torch.Tensor, w: torch.Tensor, dx: torch.Tensor, accumulate: torch.Tensor | None = None,
                 **kw) -> None:
    """dx[M,K] = dy[M,N] @ w[N,K]  (B is MN-major: w rows are the reduction dim)."""
    M, N = dy.shape
    K = w.shape[1]
    gemm_raw(dy, w, dx, M, K, N, False, True, C=accumulate, **kw)


def linear_wgrad(dy: torch.Tensor, x: torch.Tensor, dw: torch.Tensor, accumulate: torch.Tensor | None = None,
                 **kw) -> None:
    """dw[N,K] = dy[M,N]^T @ x[M,K]  (both operands MN-major: reduction over tokens)."""
    M, N = dy.shape
    K = x.shape[1]
    gemm_raw(dy, x, dw, N, K, M, True, True, C=accumulate, **kw)


# ------------------------------------------------------------------ attention
def attn_fwd(q, k, v, o, lse, T: int, hq: int, hkv: int, d: int, scale: float, causal: bool = True,
             stream=None) -> None:
    """q/k/v/o: 2-D token-major views ([T, >=heads*d], any row stride); lse: fp32 [hq, T]."""
    _need_cuda(q, k, v, o, lse)
    _lib.call("kpo_attn_fwd", _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), T, hq, hkv, d, q.stride(0),
              k.stride(0), v.stride(0), o.stride(0), ctypes.c_float(scale), int(causal), _stream(stream))


def attn_fwd_mma(q, k, v, o, lse, T: int, hq: int, hkv: int, d: int, scale: float, causal: bool = True,
                 stream=None) -> None:
    """Round-1 warp-level (mma.sync) forward: A/B baseline and cross-check only."""
    _need_cuda(q, k, v, o, lse)
    _lib.call("kpo_attn_fwd_mma", _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), T, hq, hkv, d, q.stride(0),
              k.stride(0), v.stride(0), o.stride(0), ctypes.c_float(scale), int(causal), _stream(stream))


def attn_bwd_workspace(T: int, hq: int, hkv: int, d: int, device) -> torch.Tensor:
    n = _lib.lib().kpo_attn_bwd_workspace_bytes(T, hq, hkv, d)
    return torch.empty(n, dtype=torch.uint8, device=device)


def attn_bwd(q, k, v, o, dout, lse, dq, dk, dv, T, hq, hkv, d, scale, workspace, causal=True, stream=None,
             rope_table=None):
    """rope_table (from rope_table()): q / k were rotated by linear_rope, so dq / dk are returned
    inverse-rotated (the fused backward of the rotary embedding)."""
    _need_cuda(q, k, v, o, dout, lse, dq, dk, dv, workspace, rope_table)
    if dout.stride(0) != o.stride(0):
        raise ValueError("attn_bwd: dout must share o's token stride")
    args = (_ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(dout), _ptr(lse), _ptr(dq), _ptr(dk), _ptr(dv), T, hq, hkv, d,
            q.stride(0), k.stride(0), v.stride(0), o.stride(0), dq.stride(0), dk.stride(0), dv.stride(0),
            ctypes.c_float(scale), int(causal), _ptr(workspace))
    if rope_table is None:
        _lib.call("kpo_attn_bwd", *args, _stream(stream))
    else:
        _lib.call("kpo_attn_bwd_rope", *args, _ptr(rope_table), _stream(stream))


# ------------------------------------------------------------------ non-partition work (nonpart.cu)
def embedding_fwd(ids: torch.Tensor, table: torch.Tensor, out: torch.Tensor, bad_flag: torch.Tensor,
                  stream=None) -> None:
    """out[t] = table[ids[t]]; ids int32 [T], table bf16 [V, h]; bad_flag int32 [1] set on bad ids."""
    _need_cuda(ids, table, out, bad_flag)
    if ids.dtype != torch.int32 or bad_flag.dtype != torch.int32:
        raise ValueError("embedding ids / bad_flag must be int32")
    _lib.call("kpo_embedding_fwd", _ptr(ids), _ptr(table), _ptr(out), ids.numel(), table.shape[1], table.shape[0],
              _ptr(bad_flag), _stream(stream))


def embedding_bwd(ids: torch.Tensor, dy: torch.Tensor, dtable: torch.Tensor, stream=None) -> None:
    """dtable[ids[t]] += dy[t] (fp32 gradient table [V, h])."""
    _need_cuda(ids, dy, dtable)
    if ids.dtype != torch.int32 or dtable.dtype != torch.float32:
        raise ValueError("embedding_bwd: ids int32, dtable fp32")
    _lib.call("kpo_embedding_bwd", _ptr(ids), _ptr(dy), _ptr(dtable), ids.numel(), dtable.shape[1],
              dtable.shape[0], _stream(stream))


def cross_entropy(logits: torch.Tensor, labels: torch.Tensor, loss: torch.Tensor, dlogits: torch.Tensor,
                  grad_scale: float = 1.0, ignore_index: int = -100, stream=None) -> None:
    """Fused softmax cross-entropy: loss[t] (fp32) and dlogits = (softmax - onehot) * grad_scale (bf16,
    may be `logits` itself)."""
    _need_cuda(logits, labels, loss, dlogits)
    if labels.dtype != torch.int32:
        raise ValueError("labels must be int32")
    T, V = logits.shape
    _lib.call("kpo_cross_entropy", _ptr(logits), _ptr(dlogits), _ptr(labels), _ptr(loss), T, V, logits.stride(0),
              ctypes.c_float(grad_scale), ignore_index, _stream(stream))
