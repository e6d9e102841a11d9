"""Non-partition work of a microbatch, executed and measured on the hardware.

The reference gives every microbatch a per-frequency cost table of the work outside its
partitions, `MicrobatchSpec.non_partition_costs` (reference compose.py:79-102), and fills it
analytically from abstract `non_partition_kernels` (cli.py:171-175, `_non_partition_table`
cli.py:227-241: roofline time, e_flop/e_byte energy).  Here the work is real:

  forward microbatch  (first + last pipeline stage of a Llama model):
      embedding (gather)  -> final RMSNorm -> LM head GEMM -> fused cross-entropy (loss + dlogits)
  backward microbatch:
      LM head dgrad GEMM, LM head wgrad GEMM -> final RMSNorm backward -> embedding backward
      (fp32 scatter-add into the gradient table)

over all nanobatches' tokens at once (the embedding and LM head are not nanobatched).  Under TP the
LM head is vocab-parallel (V / world columns per rank) and the cross-entropy runs over the rank's
vocab shard; the two-float cross-rank logsumexp exchange is not modelled.  `measure_costs` replays
the program as a CUDA graph over the reference's profiling protocol and returns
{frequency: (time_ms, dynamic_energy_j)}, exactly the table `MicrobatchSpec` takes.
"""

from __future__ import annotations

import torch

from . import ops
from .domain import KernelSpec, LaunchTiming, ScheduleConfig
from .layer import BF16, CommUnit, LaunchUnit, PartitionProgram
from .model import Workload

FWD_UNITS = ["embedding", "final_norm", "lm_head", "cross_entropy"]
BWD_UNITS = ["lm_head_dgrad", "lm_head_wgrad", "final_norm_bwd", "embedding_bwd"]
GEMM_UNITS = {"lm_head", "lm_head_dgrad", "lm_head_wgrad"}


def unit_specs(wl: Workload, vocab: int | None = None) -> dict[str, KernelSpec]:
    """Algorithmic work of each non-partition launch unit (flops: 2MNK; bytes: read + write)."""
    T = wl.tokens * wl.nanobatches
    h = wl.h
    V = shard_vocab(wl, vocab)
    g = lambda n, M, N, K: KernelSpec(n, flops=2.0 * M * N * K, bytes=2.0 * (M * K + N * K + M * N))
    return {
        "embedding": KernelSpec("embedding", flops=0.0, bytes=4.0 * T + 2.0 * 2 * T * h),
        "final_norm": KernelSpec("final_norm", flops=3.0 * T * h, bytes=4.0 * T * h + 2 * h + 4 * T),
        "lm_head": g("lm_head", T, V, h),
        # pass 1 reads the logits, pass 2 re-reads them and writes dlogits
        "cross_entropy": KernelSpec("cross_entropy", flops=8.0 * T * V, bytes=3.0 * 2 * T * V + 8.0 * T),
        "lm_head_dgrad": g("lm_head_dgrad", T, h, V),
        "lm_head_wgrad": g("lm_head_wgrad", V, h, T),
        "final_norm_bwd": KernelSpec("final_norm_bwd", flops=8.0 * T * h, bytes=2 * 4.0 * T * h),
        # read dy, read-modify-write fp32 table rows
        "embedding_bwd": KernelSpec("embedding_bwd", flops=T * h, bytes=4.0 * T + 2.0 * T * h + 8.0 * T * h),
    }


def shard_vocab(wl: Workload, vocab: int | None = None) -> int:
    V = vocab or wl.model.vocab
    if wl.parallel == "tp":
        V = (V + wl.world - 1) // wl.world
    return (V + 63) // 64 * 64  # GEMM / 16-byte friendly padding (padded columns get zero weights)


class NonPartitionWork:
    """Buffers and the two launch-unit programs ("np_fwd", "np_bwd") of one rank."""

    def __init__(self, wl: Workload, device, vocab: int | None = None, seed: int = 0, data_seed: int = 1000):
        self.wl = wl
        self.device = torch.device(device)
        T, h = wl.tokens * wl.nanobatches, wl.h
        self.vocab_full = vocab or wl.model.vocab
        V = shard_vocab(wl, vocab)
        self.V = V
        dev = self.device
        g = torch.Generator(device=dev).manual_seed(seed)
        self.table = (torch.randn(self.vocab_full, h, generator=g, device=dev) * 0.02).to(BF16)
        w = torch.randn(V, h, generator=g, device=dev) * 0.02
        if V > self.vocab_full and wl.parallel != "tp":
            w[self.vocab_full:] = 0.0
        self.w_lm = w.to(BF16)
        self.g_final = torch.ones(h, dtype=BF16, device=dev)
        gd = torch.Generator(device=dev).manual_seed(data_seed)
        self.ids = torch.randint(0, self.vocab_full, (T,), generator=gd, device=dev, dtype=torch.int32)
        self.labels = torch.randint(0, min(V, self.vocab_full), (T,), generator=gd, device=dev, dtype=torch.int32)
        # the last layer's output and its gradient come from the partitions; synthetic here
        self.x_last = torch.randn(T, h, generator=gd, device=dev).to(BF16)
        self.dx_first = torch.randn(T, h, generator=gd, device=dev).to(BF16)
        E = lambda *s, dt=BF16: torch.zeros(*s, dtype=dt, device=dev)
        self.emb_out = E(T, h)
        self.bad = torch.zeros(1, dtype=torch.int32, device=dev)
        self.xn = E(T, h)
        self.rstd = E(T, dt=torch.float32)
        self.logits = E(T, V)  # dlogits are written in place
        self.loss = E(T, dt=torch.float32)
        self.dxn = E(T, h)
        self.dw_lm = E(V, h)
        self.dx_last = E(T, h)
        self.dwp = E(ops.rmsnorm_partials(T, h), h, dt=torch.float32)
        self.dtable = E(self.vocab_full, h, dt=torch.float32)
        self.grad_scale = 1.0 / T
        self.sched = ops.GemmScheduler(dev, slots=8)
        self._build()

    def _build(self) -> None:
        US = unit_specs(self.wl, self.vocab_full)
        s = {k: self.sched.slot() for k in GEMM_UNITS}
        eps = self.wl.model.norm_eps
        fns = {
            "embedding": lambda st: ops.embedding_fwd(self.ids, self.table, self.emb_out, self.bad, stream=st),
            "final_norm": lambda st: ops.rmsnorm_fwd(self.x_last, self.g_final, self.xn, self.rstd, eps, stream=st),
            "lm_head": lambda st: ops.linear(self.xn, self.w_lm, self.logits, sched=s["lm_head"], stream=st),
            "cross_entropy": lambda st: ops.cross_entropy(self.logits, self.labels, self.loss, self.logits,
                                                          self.grad_scale, stream=st),
            "lm_head_dgrad": lambda st: ops.linear_dgrad(self.logits, self.w_lm, self.dxn, sched=s["lm_head_dgrad"],
                                                         stream=st),
            "lm_head_wgrad": lambda st: ops.linear_wgrad(self.logits, self.xn, self.dw_lm, sched=s["lm_head_wgrad"],
                                                         stream=st),
            "final_norm_bwd": lambda st: ops.rmsnorm_bwd(self.dxn, self.x_last, self.g_final, self.rstd,
                                                         self.dx_last, self.dwp, stream=st),
            "embedding_bwd": lambda st: ops.embedding_bwd(self.ids, self.dx_first, self.dtable, stream=st),
        }
        kind = lambda n: "gemm" if n in GEMM_UNITS else "memory"
        none = CommUnit("none", KernelSpec("none", comm_bytes=1.0), lambda st, ncta: None, n_kernels=0)
        self.programs = {
            "np_fwd": PartitionProgram("np_fwd", [LaunchUnit(n, US[n], fns[n], kind(n)) for n in FWD_UNITS], none, 1),
            "np_bwd": PartitionProgram("np_bwd", [LaunchUnit(n, US[n], fns[n], kind(n)) for n in BWD_UNITS], none, 1),
        }

    def run(self, stream=None) -> None:
        """Forward then backward non-partition work once (dependency order)."""
        st = stream or torch.cuda.current_stream(self.device)
        for name in ("np_fwd", "np_bwd"):
            for u in self.programs[name].units:
                u.fn(st)


def measure_costs(engine, program: PartitionProgram, freqs, protocol=None) -> dict[float, tuple[float, float]]:
    """{f: (time_ms, dynamic_energy_j)} of one execution of `program` per frequency, measured with the
    reference protocol fields (warmup_s / window_s / cooldown_s).  Frequencies the GPU cannot be locked
    to are not reported (NVML locked clocks are NOT_SUPPORTED on some pools): the table then holds the
    single clock the GPU ran at, keyed by f_max, like every partition measurement of that pool."""
    engine.programs[program.name] = program
    warm = getattr(protocol, "warmup_s", 0.5)
    win = getattr(protocol, "window_s", 1.0)
    cool = getattr(protocol, "cooldown_s", 0.0)
    out = {}
    fs = list(freqs) if engine.freq.available else [engine.gpu.f_max_mhz]
    for f in fs:
        cfg = ScheduleConfig(float(f), 1, LaunchTiming.sequential())
        t_ms, e_j, _ = engine.measure_local(program.name, cfg, warm, win, cool, 1)
        out[float(f)] = (t_ms, e_j - engine.gpu.p_static_w * t_ms / 1e3)
    return out


def microbatch_spec(name: str, partition_sequence, costs: dict[float, tuple[float, float]], spec_cls=None):
    """A `MicrobatchSpec` (the reference's own class when given) carrying measured costs."""
    if spec_cls is None:
        from schedfront.compose import MicrobatchSpec as spec_cls  # noqa: N813
    return spec_cls(name, tuple(partition_sequence), dict(costs))


def unit_times(work: NonPartitionWork, iters: int = 3, stream=None) -> dict[str, float]:
    """Average per-unit durations (ms) with CUDA events on the launching stream."""
    st = stream or torch.cuda.Stream(work.device)
    marks = []
    for _ in range(iters):
        for name in ("np_fwd", "np_bwd"):
            for u in work.programs[name].units:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                u.fn(st)
                e1.record(st)
                marks.append((u.name, e0, e1))
    st.synchronize()
    out: dict[str, float] = {}
    for n, e0, e1 in marks:
        out[n] = out.get(n, 0.0) + e0.elapsed_time(e1) / iters
    return out
