"""Shape-only description of a Workload's partitions (no GPU needed).

Each launch unit projects to a reference `KernelSpec` (domain.py:165-198) with its algorithmic
work: GEMMs 2MNK flops and read+write bytes; causal attention 2*T^2*hq*d forward flops (x2.5 for
backward); memory-bound units their HBM read+write bytes.  Communication units carry the bytes
each rank moves over the link (all-reduce 2(W-1)/W * S, all-gather / reduce-scatter (W-1)/W * S),
which is what the reference's `comm_bytes / comm_rate` cost model consumes (simgpu.py:162-163).
`PartitionedLayer` builds its launch units from these same specs.
"""

from __future__ import annotations

import os

from .domain import KernelSpec, PartitionSpec
from .model import Workload

FWD_ATTN = ["norm1", "linear_qkv", "rope", "attention_core", "linear_proj"]
FWD_MLP = ["norm2", "linear_up", "swiglu", "linear_down"]
BWD_MLP = ["norm1_bwd", "down_dgrad", "down_wgrad", "swiglu_bwd", "gu_dgrad", "gu_wgrad"]
BWD_ATTN = ["norm2_bwd", "o_dgrad", "o_wgrad", "attention_bwd", "rope_bwd", "qkv_dgrad", "qkv_wgrad"]
BLOCKS = [("fwd_attn", FWD_ATTN), ("fwd_mlp", FWD_MLP), ("bwd_mlp", BWD_MLP), ("bwd_attn", BWD_ATTN)]


def fused_rope(wl: Workload) -> bool:
    """head_dim 128: the rotary embedding runs in the QKV GEMM's epilogue (kpo_gemm_rope), so the
    forward attention partition has no separate "rope" launch unit."""
    return wl.d == 128 and os.environ.get("KPO_FUSED_ROPE", "1") != "0"


def fused_swiglu(wl: Workload) -> bool:
    """The SwiGLU runs in the gate|up GEMM's epilogue (kpo_gemm_swiglu: CTA-pair 256x256 tiles over
    128-row gate / up weight blocks), so the forward MLP partition has no separate "swiglu" unit."""
    return (wl.ffn % 128 == 0 and wl.tokens >= 256
            and os.environ.get("KPO_FUSED_SWIGLU", "1") != "0")


def fused_swiglu_bwd(wl: Workload) -> bool:
    """The SwiGLU backward runs in the down-projection dgrad's epilogue (kpo_gemm_swiglu_bwd), so the
    backward MLP partition has no separate "swiglu_bwd" unit (needs ffn % 256 == 0)."""
    return (fused_swiglu(wl) and wl.ffn % 256 == 0
            and os.environ.get("KPO_FUSED_SWIGLU_BWD", "1") != "0")


def blocks(wl: Workload) -> list[tuple[str, list[str]]]:
    drop = set()
    if fused_rope(wl):
        drop |= {"rope", "rope_bwd"}  # dq / dk leave attention backward inverse-rotated
    if fused_swiglu(wl):
        drop.add("swiglu")
    if fused_swiglu_bwd(wl):
        drop.add("swiglu_bwd")
    return [(blk, [k for k in units if k not in drop]) for blk, units in BLOCKS]


def block_units(wl: Workload, blk: str, b: int) -> list[str]:
    """Launch units of partition (blk, b): the block's units, plus the dγ column sums
    ("norm_grads") at the end of the iteration's last backward partition."""
    units = list(dict(blocks(wl))[blk])
    if blk == "bwd_attn" and b == wl.nanobatches - 1:
        units.append("norm_grads")
    return units


# FSDP comm units per partition: ('ag', t) all-gathers the next layer's weight t, ('rs', t)
# reduce-scatters the previous layer's gradient of t (fused into one comm unit, compose.py:32-45).
FSDP_COMMS = {
    ("fwd_attn", 0): [("ag", "wqkv")], ("fwd_attn", 1): [("ag", "wo")],
    ("fwd_mlp", 0): [("ag", "wgu")], ("fwd_mlp", 1): [("ag", "wd")],
    ("bwd_mlp", 0): [("rs", "wd"), ("ag", "wd")], ("bwd_mlp", 1): [("rs", "wgu"), ("ag", "wgu")],
    ("bwd_attn", 0): [("rs", "wo"), ("ag", "wo")],
    # the last one also reduce-scatters the previous layer's RMSNorm gradients [dγ1; dγ2] ("gn")
    ("bwd_attn", 1): [("rs", "wqkv"), ("ag", "wqkv"), ("rs", "gn")],
}
# TP: partition i all-reduces the partial produced by partition i-1 (the other nanobatch).
TP_PRODUCED = {"fwd_attn": "hp", "fwd_mlp": "yp", "bwd_mlp": "dxn2p", "bwd_attn": "dxn1p"}
GEMM_UNITS = {"linear_qkv", "linear_proj", "linear_up", "linear_down", "down_dgrad", "down_wgrad", "gu_dgrad",
              "gu_wgrad", "o_dgrad", "o_wgrad", "qkv_dgrad", "qkv_wgrad"}


def fsdp_numel(wl: Workload, tensor: str) -> int:
    """Elements of one FSDP flat tensor: the weights, or "gn" = [dγ1; dγ2] padded to 8*world."""
    if tensor == "gn":
        q = 8 * wl.world
        return (2 * wl.h + q - 1) // q * q
    return wl.weight_numels()[tensor]


def _gemm(name, M, N, K):
    return KernelSpec(name, flops=2.0 * M * N * K, bytes=2.0 * (M * K + N * K + M * N))


def _mem(name, nbytes, flops=0.0):
    return KernelSpec(name, flops=float(flops), bytes=float(nbytes))


def unit_specs(wl: Workload) -> dict[str, KernelSpec]:
    T, h, d, hq, hkv, f = wl.tokens, wl.h, wl.d, wl.hq, wl.hkv, wl.ffn
    qd = (hq + hkv) * d
    attn = 2.0 * T * T * hq * d  # causal: 4*T^2*hq*d / 2
    return {
        "norm1": _mem("norm1", 4 * T * h + 2 * h + 4 * T, 3 * T * h),
        "linear_qkv": _gemm("linear_qkv", T, wl.qkv_dim, h),
        "rope": _mem("rope", 4 * T * qd, 6 * T * qd),
        "attention_core": KernelSpec("attention_core", flops=attn, bytes=2.0 * T * (2 * hq + 2 * hkv) * d),
        "linear_proj": _gemm("linear_proj", T, h, hq * d),
        "norm2": _mem("norm2", 4 * T * h + 2 * h + 4 * T, 3 * T * h),
        "linear_up": _gemm("linear_up", T, 2 * f, h),
        "swiglu": _mem("swiglu", 2 * T * 3 * f, 4 * T * f),
        "linear_down": _gemm("linear_down", T, h, f),
        "norm1_bwd": _mem("norm1_bwd", 2 * 5 * T * h, 8 * T * h),
        "down_dgrad": _gemm("down_dgrad", T, f, h),
        "down_wgrad": _gemm("down_wgrad", h, f, T),
        "swiglu_bwd": _mem("swiglu_bwd", 2 * T * 5 * f, 10 * T * f),
        "gu_dgrad": _gemm("gu_dgrad", T, h, 2 * f),
        "gu_wgrad": _gemm("gu_wgrad", 2 * f, h, T),
        "norm2_bwd": _mem("norm2_bwd", 2 * 5 * T * h, 8 * T * h),
        "o_dgrad": _gemm("o_dgrad", T, hq * d, h),
        "o_wgrad": _gemm("o_wgrad", h, hq * d, T),
        "attention_bwd": KernelSpec("attention_bwd", flops=2.5 * attn,
                                    bytes=2.0 * T * (4 * hq + 4 * hkv) * d + 8.0 * T * hq * d),
        "rope_bwd": _mem("rope_bwd", 4 * T * qd, 6 * T * qd),
        "qkv_dgrad": _gemm("qkv_dgrad", T, h, wl.qkv_dim),
        "qkv_wgrad": _gemm("qkv_wgrad", wl.qkv_dim, h, T),
        # column sums of nanobatches x per-CTA fp32 partials of dγ1 and dγ2 -> bf16
        "norm_grads": _mem("norm_grads", 2 * (wl.nanobatches * _norm_partials(T, h) * h * 4 + 2 * h),
                           2 * wl.nanobatches * _norm_partials(T, h) * h),
    }


def _norm_partials(T: int, h: int) -> int:
    """Rows of per-CTA dγ partials kpo_rmsnorm_bwd writes (mirrors kpo_rmsnorm_bwd_partial_rows,
    elementwise.cu), without needing the library."""
    try:
        from . import ops
        return ops.rmsnorm_partials(T, h)
    except Exception:
        return 2 * 148


def partition_order(wl: Workload) -> list[tuple[str, int]]:
    return [(blk, b) for blk, _ in BLOCKS for b in range(wl.nanobatches)]


def ar_spec(wl: Workload, src: tuple[str, int]) -> tuple[KernelSpec, float]:
    W = wl.world
    size = wl.tokens * wl.h * 2
    link = 2.0 * (W - 1) / W * size if W > 1 else float(size)  # world 1: the loopback copy of S bytes
    label = f"allreduce_{src[0]}{src[1]}"
    return KernelSpec(label, comm_bytes=max(link, 1.0)), link


def fsdp_spec(wl: Workload, tensors: list[tuple[str, str]]) -> tuple[KernelSpec, float]:
    W = wl.world
    link = sum((W - 1) / W * fsdp_numel(wl, t) * 2 for _, t in tensors)
    label = "+".join(f"{k}_{t}" for k, t in tensors)
    return KernelSpec(label, comm_bytes=max(link, 1.0)), link


def comm_plan(wl: Workload) -> dict[str, tuple]:
    """partition name -> ('ar', (produced, nb)) or ('fsdp', [(kind, tensor), ...])."""
    order = partition_order(wl)
    plan = {}
    for i, (blk, b) in enumerate(order):
        name = f"{blk}{b}"
        if wl.parallel == "tp":
            pblk, pb = order[i - 1]
            plan[name] = ("ar", (TP_PRODUCED[pblk], pb))
        else:
            plan[name] = ("fsdp", FSDP_COMMS[(blk, b)])
    return plan


def partition_specs(wl: Workload) -> list[PartitionSpec]:
    us = unit_specs(wl)
    plan = comm_plan(wl)
    out = []
    for blk, b in partition_order(wl):
        name = f"{blk}{b}"
        kind, arg = plan[name]
        cspec = ar_spec(wl, arg)[0] if kind == "ar" else fsdp_spec(wl, arg)[0]
        out.append(PartitionSpec(tuple(us[k] for k in block_units(wl, blk, b)), cspec, wl.world, name))
    return out
