"""CPU fp32 restatement of the non-partition work (TEST INFRASTRUCTURE ONLY).

PARITY UNPINNED (like oracle/layer_ref.py): the reference has no embedding / LM-head / loss math;
its non-partition work is abstract `non_partition_kernels` costed analytically (reference
cli.py:171-175, 227-241).  This restates the public Llama head the engine executes
(paper_2601_17654_b200/nonpartition.py): embedding gather, final RMSNorm, LM head, softmax
cross-entropy (mean over tokens, ignore_index rows excluded from nothing but their own gradient),
with autograd for dlogits / dx / dW_lm and the embedding-table gradient.
"""

from __future__ import annotations

import torch


def cross_entropy(logits, labels, grad_scale=1.0, ignore_index=-100):
    """Per-row loss (fp32) and dlogits = (softmax - onehot) * grad_scale; ignored rows are zero."""
    x = logits.float()
    lse = torch.logsumexp(x, -1)
    valid = (labels != ignore_index) & (labels >= 0) & (labels < x.shape[1])
    lab = labels.clamp(0, x.shape[1] - 1).long()
    loss = torch.where(valid, lse - x.gather(1, lab[:, None])[:, 0], torch.zeros_like(lse))
    p = torch.softmax(x, -1)
    p[torch.arange(x.shape[0]), lab] -= 1.0
    d = p * grad_scale * valid[:, None].float()
    return loss, d


def head_fwd_bwd(x_last, w_lm, g_final, labels, eps, grad_scale):
    """final RMSNorm -> LM head -> cross-entropy; returns loss rows, dlogits, dx_last, dW_lm."""
    x = x_last.float().clone().requires_grad_(True)
    w = w_lm.float().clone().requires_grad_(True)
    xn = x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * g_final.float()
    logits = xn @ w.t()
    loss, d = cross_entropy(logits.detach(), labels, grad_scale)
    logits.backward(d)
    return {"loss": loss, "dlogits": d, "dx": x.grad, "dw": w.grad, "logits": logits.detach()}


def embedding_bwd(ids, dy, vocab):
    out = torch.zeros(vocab, dy.shape[1], dtype=torch.float32)
    out.index_add_(0, ids.long(), dy.float())
    return out
