"""Partitioned transformer layer: real tensors, launch units and partition programs.

A *partition* (reference domain.py:201-229) is one communication unit overlapped with the
ordered computation kernels of the other nanobatch.  Here every abstract KernelSpec of the
reference's workloads (workloads.py:38-93: norm, linear_qkv, rope, attention_core, linear_proj,
linear_up, linear_down, allreduce) is a concrete *launch unit* that issues hand-written sm_100a
kernels on preallocated device buffers, and the comm kernel is an SM-budgeted P2P collective.

Per layer iteration (forward + backward, 2 nanobatches) there are 8 partitions:

  TP (Megatron-style, all-reduce; config 3):
    fwd   attn(b) = [norm1, qkv, rope, attention, o_proj(+residual on rank 0)]  || AR(prev block out)
          mlp(b)  = [norm2, gate_up, swiglu, down(+residual on rank 0)]        || AR(...)
    bwd   mlp(b)  = [norm1_bwd(upper layer), down_dgrad, down_wgrad, swiglu_bwd, gu_dgrad, gu_wgrad]
          attn(b) = [norm2_bwd(+dres), o_dgrad, o_wgrad, attention_bwd, rope_bwd, qkv_dgrad, qkv_wgrad]
    comm of partition i = all-reduce of the partial sum produced by partition i-1 (the other
    nanobatch), exactly the nanobatching overlap of the paper.
  FSDP (ZeRO-3, all-gather / reduce-scatter; configs 2 and 4):
    same compute units on full (gathered) weights; fwd comm = all-gather of the next layer's
    weight tensor (qkv, o, gate_up, down — one per partition); bwd comm = reduce-scatter of the
    previous layer's gradient of one tensor fused with the re-gather of the next layer's weight
    (reference compose.py:32-45 fuses consecutive comm kernels into one unit).

Weights are random-init N(0, 0.02) from one seed on every rank, then sharded; activations are
N(0, 1) (synthetic data).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable

import torch

from . import ops, specs
from .comm import Communicator
from .domain import KernelSpec, PartitionSpec
from .model import Workload

BF16 = torch.bfloat16


@dataclass
class LaunchUnit:
    name: str
    spec: KernelSpec
    fn: Callable[[torch.cuda.Stream], None]
    kind: str = "memory"  # "gemm" | "attention" | "memory"
    n_kernels: int = 1    # device kernels one call launches


@dataclass
class CommUnit:
    name: str
    spec: KernelSpec
    fn: Callable[[torch.cuda.Stream, int], None]
    algo_bytes: float = 0.0   # bytes each rank moves over the link (busbw numerator)
    n_kernels: int = 1


@dataclass
class PartitionProgram:
    name: str
    units: list[LaunchUnit]
    comm: CommUnit
    comm_group_size: int

    def spec(self) -> PartitionSpec:
        return PartitionSpec(tuple(u.spec for u in self.units), self.comm.spec, self.comm_group_size, self.name)


def sym_bytes_for(wl: Workload, slack: int = 64 << 20) -> int:
    """Symmetric-heap bytes one rank's PartitionedLayer allocates: FSDP flat shards plus two
    layer-parity gradient buffers per tensor (and the dγ buffer); TP four partial sums per
    nanobatch plus the all-reduce stage."""
    if wl.parallel == "fsdp":
        tot = 0
        for t in ("wqkv", "wo", "wgu", "wd", "gn"):
            n = specs.fsdp_numel(wl, t)
            tot += (0 if t == "gn" else (n // wl.world * 2 + 256)) + 2 * (n * 2 + 256)
        return tot + slack
    return (4 * wl.nanobatches + 1) * (wl.tokens * wl.h * 2 + 256) + slack


class PartitionedLayer:
    """One rank's partitioned layer (weights, activations, gradients) for a Workload."""

    def __init__(self, wl: Workload, comm: Communicator, device=None, seed: int = 0, data_seed: int | None = None,
                 fill_virtual_peers: bool = True):
        self.wl = wl
        self.comm = comm
        self.device = torch.device(device or comm.device)
        self.rank, self.world = comm.rank, comm.world
        if comm.world != wl.world:
            raise ValueError("communicator world size does not match the workload")
        self.sched = ops.GemmScheduler(self.device, slots=64)
        self._init_weights(seed)
        # data seed 1000 + rank; TP ranks share their input (replicated activations)
        if data_seed is None:
            data_seed = 1000 if wl.parallel == "tp" else 1000 + self.rank
        self._init_activations(data_seed)
        self.programs: dict[str, PartitionProgram] = {}
        self.order: list[str] = []
        self._build_units()
        self._build_programs()

    # ------------------------------------------------------------------ init
    def _full_weights(self, seed: int) -> dict[str, torch.Tensor]:
        m = self.wl.model
        g = torch.Generator(device=self.device).manual_seed(seed)
        qkv_full = (m.n_heads + 2 * m.n_kv_heads) * m.head_dim

        def randn(*shape, std=0.02):
            return (torch.randn(*shape, generator=g, device=self.device) * std).to(BF16)

        return {
            "wqkv": randn(qkv_full, m.hidden),
            "wo": randn(m.hidden, m.n_heads * m.head_dim),
            "wgu": randn(2 * m.ffn, m.hidden),
            "wd": randn(m.hidden, m.ffn),
            "g1": (1.0 + 0.1 * torch.randn(m.hidden, generator=g, device=self.device)).to(BF16),
            "g2": (1.0 + 0.1 * torch.randn(m.hidden, generator=g, device=self.device)).to(BF16),
        }

    def tp_shard(self, full: dict[str, torch.Tensor], r: int) -> dict[str, torch.Tensor]:
        """Rank r's TP shard of the full weights (Megatron column/row parallel layout)."""
        wl, m = self.wl, self.wl.model
        d, hq, hkv, f = wl.d, wl.hq, wl.hkv, wl.ffn
        kv0 = (r * m.n_kv_heads) // wl.world if m.n_kv_heads >= wl.world else (r * m.n_kv_heads) // wl.world
        q_rows = full["wqkv"][r * hq * d:(r + 1) * hq * d]
        k_base = m.n_heads * d
        v_base = (m.n_heads + m.n_kv_heads) * d
        k_rows = full["wqkv"][k_base + kv0 * d:k_base + (kv0 + hkv) * d]
        v_rows = full["wqkv"][v_base + kv0 * d:v_base + (kv0 + hkv) * d]
        return {
            "wqkv": torch.cat([q_rows, k_rows, v_rows]).contiguous(),
            "wo": full["wo"][:, r * hq * d:(r + 1) * hq * d].contiguous(),
            "wgu": torch.cat([full["wgu"][r * f:(r + 1) * f], full["wgu"][m.ffn + r * f:m.ffn + (r + 1) * f]]).contiguous(),
            "wd": full["wd"][:, r * f:(r + 1) * f].contiguous(),
            "g1": full["g1"].clone(),
            "g2": full["g2"].clone(),
        }

    def _init_weights(self, seed: int) -> None:
        wl = self.wl
        full = self._full_weights(seed)
        self._full_for_oracle = full  # reference layout (parity tests)
        # fused SwiGLU: the engine stores gate|up weights (and so gu / dgu / the wgu gradient) in
        # 128-row gate / up blocks (ops.interleave_gate_up); weight_grad() returns reference layout
        self.swiglu_fused = specs.fused_swiglu(wl)
        if self.swiglu_fused and wl.parallel != "tp":
            full = dict(full, wgu=ops.interleave_gate_up(full["wgu"]))
        self.full_weights = full if wl.world == 1 or wl.parallel == "fsdp" else None
        self.tensors = ("wqkv", "wo", "wgu", "wd")
        T, h = wl.tokens, wl.h
        dev = self.device
        c = self.comm
        # `self.w` / `self.dw` are the LIVE dicts the launch units read when they are issued; for FSDP
        # set_parity() repoints them at the layer-parity buffers (see there)
        self.parity = 0
        if wl.parallel == "tp":
            self.w = self.tp_shard(full, self.rank)
            if self.swiglu_fused:
                self.w["wgu"] = ops.interleave_gate_up(self.w["wgu"])
        else:
            self.w = {k: v for k, v in full.items()}
        if wl.parallel == "fsdp":
            # Layer-parity double buffering (steady state of a stack of identical layers): iteration k
            # computes with the gathered weights wbuf[k%2] and writes its weight gradients into
            # dw_sym[k%2]; its collectives all-gather the NEXT layer's weights into wbuf[1-k%2] and
            # reduce-scatter the PREVIOUS layer's gradients from dw_sym[1-k%2].  So every gathered
            # weight is consumed by the next iteration and every reduce-scatter reads real gradients.
            # wbuf[1] starts zeroed: iteration 1 is only correct if iteration 0's all-gathers were.
            self.shard = {}
            self.wbuf = [{}, {}]
            self.dw_sym = [{}, {}]  # gradient buffers (RS inputs) in the symmetric heap
            self.dw_shard = {}
            names = self.tensors + ("gn",)
            for name in names:
                n = specs.fsdp_numel(wl, name)
                if n % (8 * wl.world):
                    raise ValueError(f"{name} numel {n} not divisible by 8*world")
                per = n // wl.world
                if name != "gn":  # norm weights are replicated; only their gradients are reduced
                    reg = c.alloc(per * 2)
                    reg.local().copy_(full[name].view(-1)[self.rank * per:(self.rank + 1) * per])
                    if c.loopback:
                        for p in range(wl.world):
                            if p != self.rank:
                                reg.peer(p).copy_(full[name].view(-1)[p * per:(p + 1) * per])
                    self.shard[name] = reg
                    self.wbuf[0][name] = full[name].clone()  # full_weights stays the pristine copy
                    self.wbuf[1][name] = torch.zeros_like(full[name])
                for par in range(2):
                    reg = c.alloc(n * 2)
                    reg.local().zero_()
                    if c.loopback:
                        # virtual peers' gradients: a fixed seeded pattern (never rewritten), so the
                        # loopback reduce-scatter output is checkable against the numpy oracle
                        g = torch.Generator(device=dev).manual_seed(7919 * (par + 1) + len(name))
                        for p in range(wl.world):
                            if p != self.rank:
                                reg.peer(p).copy_((torch.randn(n, generator=g, device=dev) * 1e-2).to(BF16))
                    self.dw_sym[par][name] = reg
                self.dw_shard[name] = torch.empty(per, dtype=BF16, device=dev)
            self.dw = {}
            self.set_parity(0)
        else:
            self.dw = {k: torch.empty_like(self.w[k]) for k in self.tensors}
            self.partial = [{}, {}]
            for b in range(wl.nanobatches):
                for name in ("hp", "yp", "dxn2p", "dxn1p"):
                    self.partial[b % 2][(name, b)] = c.alloc(T * h * 2)
            self.stage = c.alloc(T * h * 2)
            self.dg1 = torch.empty(h, dtype=BF16, device=dev)
            self.dg2 = torch.empty(h, dtype=BF16, device=dev)

    @property
    def parity_period(self) -> int:
        """Number of distinct buffer sets consecutive iterations cycle through (graph variants)."""
        return 2 if self.wl.parallel == "fsdp" else 1

    def set_parity(self, p: int) -> None:
        """Point the live weight / gradient dicts at layer-parity p (FSDP; a no-op for TP).  Launch
        units and comm units resolve their buffers when they are issued, so a CUDA graph captured
        under parity p replays parity p."""
        p &= 1
        if self.wl.parallel != "fsdp":
            self.parity = 0
            return
        self.parity = p
        h = self.wl.h
        self.w.update(self.wbuf[p])
        for k in self.tensors:
            self.dw[k] = self.dw_sym[p][k].local().view(self.wbuf[p][k].shape)
        gn = self.dw_sym[p]["gn"].local()
        self.dg1, self.dg2 = gn[:h], gn[h:2 * h]

    @property
    def w_next(self) -> dict[str, torch.Tensor]:
        """The buffers this iteration's all-gathers write (the next iteration's weights)."""
        return self.wbuf[1 - self.parity]

    def dgn_shard(self) -> torch.Tensor:
        """This rank's reduce-scattered shard of [dg1; dg2] (FSDP)."""
        return self.dw_shard["gn"]

    def _init_activations(self, data_seed: int) -> None:
        wl = self.wl
        T, h, d = wl.tokens, wl.h, wl.d
        dev = self.device
        g = torch.Generator(device=dev).manual_seed(data_seed)
        E = lambda *s, dt=BF16: torch.zeros(*s, dtype=dt, device=dev)
        self.nb = []
        nparts = ops.rmsnorm_partials(T, h)
        # per-CTA fp32 partials of dγ for every nanobatch, contiguous so one column sum reduces them
        self.dwp_all = [E(wl.nanobatches * nparts, h, dt=torch.float32) for _ in range(2)]
        for b in range(wl.nanobatches):
            a = {
                "x": torch.randn(T, h, generator=g, device=dev).to(BF16),
                "dy": torch.randn(T, h, generator=g, device=dev).to(BF16),
                "xn1": E(T, h), "rstd1": E(T, dt=torch.float32), "qkv": E(T, wl.qkv_dim),
                "qkr": E(T, (wl.hq + wl.hkv) * d), "ao": E(T, wl.hq * d), "lse": E(wl.hq, T, dt=torch.float32),
                "h": E(T, h), "xn2": E(T, h), "rstd2": E(T, dt=torch.float32), "gu": E(T, 2 * wl.ffn),
                "act": E(T, wl.ffn), "y": E(T, h),
                "dact": E(T, wl.ffn), "dgu": E(T, 2 * wl.ffn), "dxn2": E(T, h), "dh": E(T, h),
                "dao": E(T, wl.hq * d), "dqkr": E(T, (wl.hq + wl.hkv) * d), "dqkv": E(T, wl.qkv_dim),
                "dxn1": E(T, h), "dx": E(T, h),
                "dwp1": self.dwp_all[0][b * nparts:(b + 1) * nparts],
                "dwp2": self.dwp_all[1][b * nparts:(b + 1) * nparts],
            }
            if wl.parallel == "fsdp":
                a["dxn2p"] = a["dxn2"]
                a["dxn1p"] = a["dxn1"]
            self.nb.append(a)
        self.attn_ws = ops.attn_bwd_workspace(T, wl.hq, wl.hkv, d, dev)

    # ------------------------------------------------------------------ launch units
    def _gemm(self, slot):
        def run(fn, *args, **kw):
            fn(*args, sched=slot, **kw)
        return run

    def _build_units(self) -> None:
        wl = self.wl
        T, h, d, hq, hkv = wl.tokens, wl.h, wl.d, wl.hq, wl.hkv
        qd = (hq + hkv) * d
        scale = 1.0 / math.sqrt(d)
        eps, theta = wl.model.norm_eps, wl.model.rope_theta
        tp = wl.parallel == "tp"
        rank0 = self.rank == 0
        W, dw = self.w, self.dw  # live dicts (set_parity repoints their entries)
        US = specs.unit_specs(wl)
        fused = specs.fused_rope(wl)
        qk_src = "qkv" if fused else "qkr"
        if fused:
            self.rope_cs = ops.rope_table(T, d, theta, self.device)
        self.units: dict[tuple[str, int], LaunchUnit] = {}
        kinds = {"attention_core": "attention", "attention_bwd": "attention"}

        for b in range(wl.nanobatches):
            a = self.nb[b]
            # partial-sum outputs of row-parallel GEMMs (TP) live in the symmetric buffer
            if tp:
                hp, yp, dxn2p, dxn1p = (self.partial[b % 2][(k, b)].local().view(T, h)
                                        for k in ("hp", "yp", "dxn2p", "dxn1p"))
            else:
                hp, yp, dxn2p, dxn1p = a["h"], a["y"], a["dxn2"], a["dxn1"]
            a["hp"], a["yp"] = hp, yp
            # residual inputs are looked up when the unit is issued (LayerRunner swaps a["x"] between
            # host-staging slots, each with its own captured graphs)
            res_attn = "x" if (not tp or rank0) else None
            res_mlp = "h" if (not tp or rank0) else None
            s = {k: self.sched.slot() for k in US if k in specs.GEMM_UNITS}
            acc = b > 0  # weight gradients accumulate over nanobatches (epilogue C input)
            fns = {
                # ---------------- forward
                "norm1": lambda st, a=a: ops.rmsnorm_fwd(a["x"], W["g1"], a["xn1"], a["rstd1"], eps, stream=st),
                "linear_qkv": (lambda st, a=a, s=s: ops.linear_rope(a["xn1"], W["wqkv"], a["qkv"], self.rope_cs, qd,
                                                                    d, sched=s["linear_qkv"], stream=st))
                if fused else (lambda st, a=a, s=s: ops.linear(a["xn1"], W["wqkv"], a["qkv"], sched=s["linear_qkv"],
                                                              stream=st)),
                "rope": lambda st, a=a: ops.rope(a["qkv"], a["qkr"], hq + hkv, d, theta, stream=st),
                # with the fused rotary epilogue q / k are rotated in place in qkv
                "attention_core": lambda st, a=a, qk=qk_src: ops.attn_fwd(a[qk][:, :hq * d], a[qk][:, hq * d:qd],
                                                                          a["qkv"][:, qd:], a["ao"], a["lse"], T, hq,
                                                                          hkv, d, scale, stream=st),
                "linear_proj": lambda st, a=a, s=s, hp=hp, r=res_attn: ops.linear(
                    a["ao"], W["wo"], hp, residual=a[r] if r else None, sched=s["linear_proj"], stream=st),
                "norm2": lambda st, a=a: ops.rmsnorm_fwd(a["h"], W["g2"], a["xn2"], a["rstd2"], eps, stream=st),
                "linear_up": (lambda st, a=a, s=s: ops.linear_swiglu(a["xn2"], W["wgu"], a["gu"], a["act"],
                                                                     sched=s["linear_up"], stream=st))
                if self.swiglu_fused else (lambda st, a=a, s=s: ops.linear(a["xn2"], W["wgu"], a["gu"],
                                                                          sched=s["linear_up"], stream=st)),
                "swiglu": lambda st, a=a, blk=ops.SWIGLU_BLOCK if self.swiglu_fused else 0: ops.swiglu_fwd(
                    a["gu"], a["act"], stream=st, block=blk),
                "linear_down": lambda st, a=a, s=s, yp=yp, r=res_mlp: ops.linear(
                    a["act"], W["wd"], yp, residual=a[r] if r else None, sched=s["linear_down"], stream=st),
                # ---------------- backward
                "norm1_bwd": lambda st, a=a: ops.rmsnorm_bwd(a["dxn1"], a["x"], W["g1"], a["rstd1"], a["dx"],
                                                             a["dwp1"], dres=a["dh"], stream=st),
                # fused: dgu straight from the dgrad's epilogue (dact never materialised)
                "down_dgrad": (lambda st, a=a, s=s: ops.linear_dgrad_swiglu_bwd(
                    a["dy"], W["wd"], a["gu"], a["dgu"], sched=s["down_dgrad"], stream=st))
                if specs.fused_swiglu_bwd(wl) else (lambda st, a=a, s=s: ops.linear_dgrad(
                    a["dy"], W["wd"], a["dact"], sched=s["down_dgrad"], stream=st)),
                "down_wgrad": lambda st, a=a, s=s, acc=acc: ops.linear_wgrad(
                    a["dy"], a["act"], dw["wd"], accumulate=dw["wd"] if acc else None, sched=s["down_wgrad"],
                    stream=st),
                "swiglu_bwd": lambda st, a=a, blk=ops.SWIGLU_BLOCK if self.swiglu_fused else 0: ops.swiglu_bwd(
                    a["dact"], a["gu"], a["dgu"], stream=st, block=blk),
                "gu_dgrad": lambda st, a=a, s=s, o=dxn2p: ops.linear_dgrad(a["dgu"], W["wgu"], o,
                                                                           sched=s["gu_dgrad"], stream=st),
                "gu_wgrad": lambda st, a=a, s=s, acc=acc: ops.linear_wgrad(
                    a["dgu"], a["xn2"], dw["wgu"], accumulate=dw["wgu"] if acc else None, sched=s["gu_wgrad"],
                    stream=st),
                "norm2_bwd": lambda st, a=a: ops.rmsnorm_bwd(a["dxn2"], a["h"], W["g2"], a["rstd2"], a["dh"],
                                                             a["dwp2"], dres=a["dy"], stream=st),
                "o_dgrad": lambda st, a=a, s=s: ops.linear_dgrad(a["dh"], W["wo"], a["dao"], sched=s["o_dgrad"],
                                                                 stream=st),
                "o_wgrad": lambda st, a=a, s=s, acc=acc: ops.linear_wgrad(
                    a["dh"], a["ao"], dw["wo"], accumulate=dw["wo"] if acc else None, sched=s["o_wgrad"], stream=st),
                "attention_bwd": (lambda st, a=a: ops.attn_bwd(
                    a["qkv"][:, :hq * d], a["qkv"][:, hq * d:qd], a["qkv"][:, qd:], a["ao"], a["dao"], a["lse"],
                    a["dqkv"][:, :hq * d], a["dqkv"][:, hq * d:qd], a["dqkv"][:, qd:], T, hq, hkv, d, scale,
                    self.attn_ws, stream=st, rope_table=self.rope_cs)) if fused else (lambda st, a=a: ops.attn_bwd(
                    a["qkr"][:, :hq * d], a["qkr"][:, hq * d:], a["qkv"][:, qd:], a["ao"], a["dao"], a["lse"],
                    a["dqkr"][:, :hq * d], a["dqkr"][:, hq * d:], a["dqkv"][:, qd:], T, hq, hkv, d, scale,
                    self.attn_ws, stream=st)),
                "rope_bwd": lambda st, a=a: ops.rope(a["dqkr"], a["dqkv"], hq + hkv, d, theta, inverse=True,
                                                     stream=st),
                "qkv_dgrad": lambda st, a=a, s=s, o=dxn1p: ops.linear_dgrad(a["dqkv"], W["wqkv"], o,
                                                                            sched=s["qkv_dgrad"], stream=st),
                "qkv_wgrad": lambda st, a=a, s=s, acc=acc: ops.linear_wgrad(
                    a["dqkv"], a["xn1"], dw["wqkv"], accumulate=dw["wqkv"] if acc else None, sched=s["qkv_wgrad"],
                    stream=st),
            }
            if b == wl.nanobatches - 1:
                # dγ1 / dγ2 of the iteration: column sums of both nanobatches' per-CTA partials (FSDP:
                # into the symmetric gradient buffer the next iteration reduce-scatters)
                fns["norm_grads"] = lambda st: (ops.colsum(self.dwp_all[0], self.dg1, stream=st),
                                                ops.colsum(self.dwp_all[1], self.dg2, stream=st))
            for name, fn in fns.items():
                kind = "gemm" if name in specs.GEMM_UNITS else kinds.get(name, "memory")
                nk = {"attention_bwd": 3, "norm_grads": 2}.get(name, 1)  # attn: pre-pass, main, dq conversion
                self.units[(name, b)] = LaunchUnit(name, US[name], fn, kind, nk)

    # ------------------------------------------------------------------ comm units
    def _ar_unit(self, src_key: tuple[str, int], out: torch.Tensor) -> CommUnit:
        name, b = src_key
        reg = self.partial[b % 2][src_key]
        spec, link = specs.ar_spec(self.wl, src_key)

        def fn(st, ncta, reg=reg, out=out):
            self.comm.all_reduce(reg, self.stage, out, ncta, stream=st)

        return CommUnit(spec.name, spec, fn, algo_bytes=link)

    def _fsdp_unit(self, tensors: list[tuple[str, str]]) -> CommUnit:
        spec, link = specs.fsdp_spec(self.wl, tensors)

        def fn(st, ncta):
            for kind, name in tensors:
                # buffers resolved at issue time: parity p gathers into wbuf[1-p], reduces dw_sym[1-p]
                if kind == "ag":
                    self.comm.all_gather(self.shard[name], self.wbuf[1 - self.parity][name], ncta, stream=st)
                else:
                    self.comm.reduce_scatter(self.dw_sym[1 - self.parity][name], self.dw_shard[name], ncta,
                                             stream=st)

        return CommUnit(spec.name, spec, fn, algo_bytes=link, n_kernels=len(tensors))

    def _build_programs(self) -> None:
        wl = self.wl
        if wl.nanobatches != 2:
            raise ValueError("partition programs are built for 2 nanobatches")
        out_of = {"hp": "h", "yp": "y", "dxn2p": "dxn2", "dxn1p": "dxn1"}
        plan = specs.comm_plan(wl)
        for blk, b in specs.partition_order(wl):
            name = f"{blk}{b}"
            kind, arg = plan[name]
            if kind == "ar":
                comm = self._ar_unit(arg, self.nb[arg[1]][out_of[arg[0]]])
            else:
                comm = self._fsdp_unit(arg)
            units = [self.units[(k, b)] for k in specs.block_units(self.wl, blk, b)]
            self.programs[name] = PartitionProgram(name, units, comm, wl.world)
            self.order.append(name)

    # ------------------------------------------------------------------ helpers
    def finalize_norm_grads(self, stream=None) -> None:
        """dg1/dg2 = column sums of the per-CTA partials of both nanobatches (the norm_grads unit)."""
        self.units[("norm_grads", self.wl.nanobatches - 1)].fn(stream or torch.cuda.current_stream())

    def partition_specs(self) -> list[PartitionSpec]:
        return [self.programs[n].spec() for n in self.order]

    def run_unrolled(self, stream=None, ncta: int = 16) -> None:
        """Dependency-correct single-layer forward+backward (for parity tests): every launch unit
        once per nanobatch, each collective right after the unit that produces its input."""
        st = stream or torch.cuda.current_stream()
        tp = self.wl.parallel == "tp"
        blk = dict(specs.blocks(self.wl))  # unit lists (no separate rope units when RoPE is fused)
        for b in range(self.wl.nanobatches):
            a = self.nb[b]
            for k in blk["fwd_attn"]:
                self.units[(k, b)].fn(st)
            if tp:
                self.comm.all_reduce(self.partial[b % 2][("hp", b)], self.stage, a["h"], ncta, stream=st)
            for k in blk["fwd_mlp"]:
                self.units[(k, b)].fn(st)
            if tp:
                self.comm.all_reduce(self.partial[b % 2][("yp", b)], self.stage, a["y"], ncta, stream=st)
        for b in range(self.wl.nanobatches):
            a = self.nb[b]
            for k in [u for u in blk["bwd_mlp"] if u != "norm1_bwd"]:
                self.units[(k, b)].fn(st)
            if tp:
                self.comm.all_reduce(self.partial[b % 2][("dxn2p", b)], self.stage, a["dxn2"], ncta, stream=st)
            for k in blk["bwd_attn"]:
                self.units[(k, b)].fn(st)
            if tp:
                self.comm.all_reduce(self.partial[b % 2][("dxn1p", b)], self.stage, a["dxn1"], ncta, stream=st)
            self.units[("norm1_bwd", b)].fn(st)
        self.finalize_norm_grads(st)

    def weight_grad(self, name: str) -> torch.Tensor:
        """This rank's gradient of weight `name` in the reference layout ([gate; up] for wgu)."""
        if name == "wgu" and self.swiglu_fused:
            return ops.deinterleave_gate_up(self.dw[name])
        return self.dw[name]
