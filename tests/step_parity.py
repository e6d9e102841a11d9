"""Helpers for the executed-schedule parity tests (test_step_parity_gpu.py, tools/ipc_step_parity.py).

What is checked is the thing bench.py times: `LayerRunner.step()` replaying the captured partition
graphs under a schedule assignment (collectives on their own SMs, launch gate, sync points), with
the layer-parity buffers alternating between iterations.  Inputs are the same every iteration, so
after two iterations the steady state equals one dependency-correct layer forward + backward,
which the CPU fp32 oracle (oracle/layer_ref.py) computes.

Before each schedule every buffer an iteration produces is poisoned with NaN (activations,
gradients, partial sums, the weight buffer the next iteration gathers into), so a stale value left
by an earlier schedule or a skipped launch cannot pass.

Tolerance (stated, north_star check 1): relative Frobenius error <= 3e-2 for y, h,
dx, every dW and dγ (bf16 storage of ~10 chained intermediates; measured ~2e-3 - 1e-2).  Collective
outputs are bit-exact against the numpy collective oracle.
"""
from __future__ import annotations

import numpy as np
import torch

TOL = 3e-2


def rel(a, b) -> float:
    a, b = a.float().cpu(), b.float().cpu()
    return ((a - b).norm() / b.norm().clamp_min(1e-12)).item()


def bits(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().cpu().view(torch.int16).numpy().view(np.uint16).reshape(-1)


def schedules(layer, gpu):
    """The default nanobatching schedule and two non-default ones."""
    from paper_2601_17654_b200.domain import LaunchTiming, ScheduleConfig
    from paper_2601_17654_b200.runner import default_schedule, sequential_schedule

    f = gpu.f_max_mhz
    ov12 = {n: ScheduleConfig(f, 8, LaunchTiming.overlap(min(1, len(layer.programs[n].units) - 1), 2))
            for n in layer.order}
    return {"default": default_schedule(layer, gpu), "ov1x2@8": ov12, "seq": sequential_schedule(layer, gpu)}


def poison(layer, next_parity: int) -> None:
    """NaN-fill every produced buffer; `next_parity` is the parity of the next iteration (its
    all-gathers write wbuf[1 - next_parity], which the iteration after it reads)."""
    nan = float("nan")
    for a in layer.nb:
        for k, t in a.items():
            if k not in ("x", "dy") and t.is_floating_point():
                t.fill_(nan)
    for t in layer.dwp_all:
        t.fill_(nan)
    if layer.wl.parallel == "fsdp":
        for par in range(2):
            for k, reg in layer.dw_sym[par].items():
                # "gn": only [dγ1; dγ2] is ever written, its padding stays zero
                (reg.local()[:2 * layer.wl.h] if k == "gn" else reg.local()).fill_(nan)
        for t in layer.dw_shard.values():
            t.fill_(nan)
        # the buffer the first poisoned iteration gathers into (the second one reads it)
        for t in layer.wbuf[1 - (next_parity & 1)].values():
            t.fill_(nan)
    else:
        for d in layer.partial:
            for reg in d.values():
                reg.local().fill_(nan)
        layer.stage.local().fill_(nan)
        layer.dg1.fill_(nan)
        layer.dg2.fill_(nan)
    torch.cuda.synchronize(layer.device)


def oracle_for(layer, xs=None, dys=None):
    from oracle import layer_ref

    W = {k: v.float().cpu() for k, v in layer._full_for_oracle.items()}
    xs = xs if xs is not None else [a["x"].cpu() for a in layer.nb]
    dys = dys if dys is not None else [a["dy"].cpu() for a in layer.nb]
    torch.set_num_threads(max(1, torch.get_num_threads()))
    return layer_ref.layer_fwd_bwd(xs, dys, W, layer.wl.model)


def check_outputs(layer, ref, tp_rank_slices=None) -> dict:
    """Relative errors of this rank's y, h, dx, dW, dγ against the oracle (TP: the rank's weight
    slices of the full gradients)."""
    errs = {}
    for b, a in enumerate(layer.nb):
        for k in ("h", "y", "dx"):
            errs[f"{k}{b}"] = rel(a[k], ref[k][b])
    for k in ("wqkv", "wo", "wgu", "wd"):
        g = ref["grads"][k]
        if tp_rank_slices is not None:
            g = tp_rank_slices(g, k)
        errs[f"d{k}"] = rel(layer.weight_grad(k), g)
    errs["dg1"] = rel(layer.dg1, ref["grads"]["g1"])
    errs["dg2"] = rel(layer.dg2, ref["grads"]["g2"])
    return errs


def check_fsdp_collectives_loopback(layer) -> dict:
    """After an iteration of parity p: (1) the all-gathers wrote the full weights into wbuf[1-p]
    (bit-exact), and wbuf[p] (gathered by the previous iteration) too; (2) the reduce-scatters
    reduced dw_sym[1-p] (the previous iteration's gradients) with the virtual peers' fixed
    gradients, bit-exact against the numpy collective oracle (fp32 rank-order sum)."""
    from oracle import collectives as oc

    out = {}
    p = layer.parity
    for k in layer.tensors:
        full = layer.full_weights[k]
        out[f"ag_{k}"] = bool(torch.equal(layer.wbuf[1 - p][k], full)) and bool(torch.equal(layer.wbuf[p][k], full))
    c = layer.comm
    for k in layer.tensors + ("gn",):
        reg = layer.dw_sym[1 - p][k]
        ins = [bits(reg.local()) if q == c.rank else bits(reg.peer(q)) for q in range(c.world)]
        exp = oc.reduce_scatter(ins, c.rank)
        out[f"rs_{k}"] = bool(np.array_equal(bits(layer.dw_shard[k]), exp))
    return out


def previous_grads_rel(layer, ref) -> dict:
    """The previous iteration's gradients (the reduce-scatter input) also match the oracle."""
    from paper_2601_17654_b200 import ops

    p = layer.parity
    out = {}
    for k in layer.tensors:
        g = layer.dw_sym[1 - p][k].local().view(layer.wbuf[0][k].shape)
        if k == "wgu" and layer.swiglu_fused:
            g = ops.deinterleave_gate_up(g)
        out[f"prev_d{k}"] = rel(g, ref["grads"][k])
    return out
