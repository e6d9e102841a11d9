"""1F1B pipeline validation harness: run a real PP x TP iteration and compare it with
the reference's 1F1B emulator (`compose.simulate_pipeline`, compose.py:376-395, with the frequency-
switch gaps of `_switch_delays`, compose.py:398-406).

Rank grid: `pp` stages x `tp` ranks, rank = stage * tp + tp_rank (torch.distributed world of pp*tp).
Every rank of stage s executes the reference's per-stage 1F1B op order (`stage_op_order`, restated
from compose.py:263-272 and checked against it in tests/test_pipeline_gloo.py):

    warmup forwards, then one-forward-one-backward, then the draining backwards.

F(m) on stage s > 0 first receives microbatch m's activations from the same tp rank of stage s-1;
B(m) on stage s < pp-1 first receives its gradients from stage s+1; results are sent on after the
op.  Sends are asynchronous (isend), so a stage never waits for its consumer; receives block, which
is exactly the dependency edge structure of `_PipelineGraph` (compose.py:297-330).

The stage work is pluggable:
  * `SleepStageWork` -- CPU stand-in for the control-plane test (gloo, tests/test_pipeline_gloo.py);
  * `LayerStageWork` -- the B200 path: `layers` layer iterations of this stage's PartitionedLayer
    (TP over the stage's tp group with the engine's P2P collectives), forward = the fwd partitions
    under their schedule, backward = the bwd partitions, transfers of [T, h] bf16 activations /
    gradients per nanobatch over NCCL send/recv (plumbing; the hot-path collectives stay P2P).
Each op is timed on its own clock (CUDA events on the compute stream, or perf_counter), together
with the time the stage spent waiting for its input; `emulate()` then feeds the measured per-op
durations to the reference emulator and compares the emulated makespan with the measured one (max
over ranks).  Given per-op energies (`op_energy`, e.g. NVML windows of each op type run back to back,
tools/pipeline_1f1b.py), the emulator's energy (sum of op energies + static power over idle time) is
compared with the NVML energy of the whole iteration.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import torch
import torch.distributed as dist


def stage_op_order(num_stages: int, num_microbatches: int, stage: int) -> list[tuple[str, int]]:
    """The 1F1B op sequence of one stage (reference PipelineSpec.stage_op_order, compose.py:263-272)."""
    warmup = min(num_stages - 1 - stage, num_microbatches)
    ops = [("F", m) for m in range(warmup)]
    for m in range(warmup, num_microbatches):
        ops.append(("F", m))
        ops.append(("B", m - warmup))
    for m in range(num_microbatches - warmup, num_microbatches):
        ops.append(("B", m))
    return ops


@dataclass
class OpRecord:
    stage: int
    microbatch: int
    direction: str
    start_ms: float      # relative to the iteration start (after the start barrier)
    end_ms: float
    wait_ms: float       # time spent blocked in the receive before the op
    duration_ms: float   # the op itself (device time on GPU)


@dataclass
class PipelineRun:
    pp: int
    tp: int
    microbatches: int
    rank: int
    records: list[OpRecord] = field(default_factory=list)
    makespan_ms: float = 0.0
    energy_j: float | None = None
    transfers_ok: bool = True

    def durations(self) -> dict[tuple[int, int, str], float]:
        return {(r.stage, r.microbatch, r.direction): r.duration_ms for r in self.records}


class Grid:
    """pp x tp rank grid over the default process group; tp groups and p2p peers."""

    def __init__(self, pp: int, tp: int):
        world, rank = dist.get_world_size(), dist.get_rank()
        if pp * tp != world:
            raise ValueError(f"pp*tp = {pp * tp} != world size {world}")
        self.pp, self.tp, self.rank = pp, tp, rank
        self.stage, self.tp_rank = divmod(rank, tp)
        self.tp_groups = [dist.new_group([s * tp + t for t in range(tp)]) for s in range(pp)]
        self.tp_group = self.tp_groups[self.stage]

    def peer(self, stage: int) -> int:
        return stage * self.tp + self.tp_rank


# ------------------------------------------------------------------------------------ stage work
class SleepStageWork:
    """CPU stand-in: each op sleeps (F, B durations in ms) and all-reduces a scalar over the tp group,
    the stage's TP collective.  Payloads carry the microbatch id so routing errors are detected."""

    device = torch.device("cpu")

    def __init__(self, f_ms: float, b_ms: float, numel: int = 1024, tp_group=None):
        self.f_ms, self.b_ms, self.numel, self.tp_group = f_ms, b_ms, numel, tp_group
        self.seen: list[tuple[str, int, float]] = []

    def buffer(self, direction: str) -> torch.Tensor:
        return torch.empty(self.numel)

    def forward(self, m: int, inp: torch.Tensor | None) -> torch.Tensor:
        if inp is not None:
            self.seen.append(("F", m, float(inp[0])))
        time.sleep(self.f_ms / 1e3)
        if self.tp_group is not None:
            dist.all_reduce(torch.ones(1), group=self.tp_group)
        return torch.full((self.numel,), float(m))

    def backward(self, m: int, grad: torch.Tensor | None) -> torch.Tensor:
        if grad is not None:
            self.seen.append(("B", m, float(grad[0])))
        time.sleep(self.b_ms / 1e3)
        if self.tp_group is not None:
            dist.all_reduce(torch.ones(1), group=self.tp_group)
        return torch.full((self.numel,), 1000.0 + m)

    def timed(self, fn):
        t0 = time.perf_counter()
        out = fn()
        return out, (time.perf_counter() - t0) * 1e3

    def now_ms(self) -> float:
        return time.perf_counter() * 1e3


class LayerStageWork:
    """B200 stage: `layers` iterations of a PartitionedLayer's forward / backward partitions per op,
    executed through the engine's schedule executor (captured graphs; collective on its SM budget)."""

    def __init__(self, layer, engine, schedule, layers: int):
        self.layer, self.engine, self.schedule, self.layers = layer, engine, schedule, layers
        self.device = engine.device
        self.stream = engine.exec.compute
        self.fwd = [n for n in layer.order if n.startswith("fwd")]
        self.bwd = [n for n in layer.order if n.startswith("bwd")]
        for n in layer.order:
            engine.exec.graph(layer.programs[n], schedule[n], engine.default_ncta())
        T, h = layer.wl.tokens, layer.wl.h
        nb = layer.wl.nanobatches
        self._act = torch.empty(nb, T, h, dtype=torch.bfloat16, device=self.device)
        self._grad = torch.empty(nb, T, h, dtype=torch.bfloat16, device=self.device)

    def buffer(self, direction: str) -> torch.Tensor:
        return self._act if direction == "F" else self._grad

    def _run(self, names):
        ex = self.engine.exec
        for _ in range(self.layers):
            for n in names:
                ex.run(self.layer.programs[n], self.schedule[n], self.engine.default_ncta(), 1)

    def forward(self, m: int, inp):
        self.stream.wait_stream(torch.cuda.current_stream(self.device))  # the receive (NCCL, current stream)
        with torch.cuda.stream(self.stream):
            if inp is not None:
                for b, a in enumerate(self.layer.nb):
                    a["x"].copy_(inp[b])
            self._run(self.fwd)
            for b, a in enumerate(self.layer.nb):
                self._act[b].copy_(a["y"])
        torch.cuda.current_stream(self.device).wait_stream(self.stream)  # before the send
        return self._act

    def backward(self, m: int, grad):
        self.stream.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(self.stream):
            if grad is not None:
                for b, a in enumerate(self.layer.nb):
                    a["dy"].copy_(grad[b])
            self._run(self.bwd)
            for b, a in enumerate(self.layer.nb):
                self._grad[b].copy_(a["dx"])
        torch.cuda.current_stream(self.device).wait_stream(self.stream)
        return self._grad

    def timed(self, fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(self.stream)
        out = fn()
        e1.record(self.stream)
        e1.synchronize()
        return out, e0.elapsed_time(e1)

    def now_ms(self) -> float:
        torch.cuda.synchronize(self.device)
        return time.perf_counter() * 1e3


# ------------------------------------------------------------------------------------ the runner
def run_iteration(grid: Grid, work, microbatches: int, sampler=None) -> PipelineRun:
    """Execute one 1F1B iteration on this rank; returns its op records (times relative to a common
    start barrier) and, with an NVML `sampler`, this rank's energy over the iteration."""
    S, s = grid.pp, grid.stage
    order = stage_op_order(S, microbatches, s)
    run = PipelineRun(S, grid.tp, microbatches, grid.rank)
    pending = []
    dist.barrier()
    t0 = work.now_ms()
    w0 = time.perf_counter()
    for d, m in order:
        inp = None
        tw = work.now_ms()
        if d == "F" and s > 0:
            inp = work.buffer("F")
            dist.recv(inp, src=grid.peer(s - 1))
        elif d == "B" and s < S - 1:
            inp = work.buffer("B")
            dist.recv(inp, src=grid.peer(s + 1))
        start = work.now_ms()
        fn = (lambda: work.forward(m, inp)) if d == "F" else (lambda: work.backward(m, inp))
        out, dur = work.timed(fn)
        end = start + dur
        run.records.append(OpRecord(s, m, d, start - t0, end - t0, start - tw, dur))
        if d == "F" and s < S - 1:
            pending.append(dist.isend(out.clone() if out.device.type == "cpu" else out, dst=grid.peer(s + 1)))
            if out.device.type != "cpu":
                pending[-1].wait()  # the stage's single activation buffer is reused by the next op
        elif d == "B" and s > 0:
            pending.append(dist.isend(out.clone() if out.device.type == "cpu" else out, dst=grid.peer(s - 1)))
            if out.device.type != "cpu":
                pending[-1].wait()
    for p in pending:
        p.wait()
    t_end = work.now_ms()
    w1 = time.perf_counter()
    run.makespan_ms = t_end - t0
    if sampler is not None:
        run.energy_j = sampler.window_j(w0, w1)
    dist.barrier()
    return run


def gather_runs(run: PipelineRun) -> list[PipelineRun]:
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, run)
    return out


def emulate(runs: list[PipelineRun], pp: int, microbatches: int, p_static_w: float,
            op_energy: dict[tuple[int, str], float] | None = None, freq_switch_ms: float = 0.0,
            schedfront_module=None) -> dict:
    """Feed the measured per-op durations (max over a stage's tp ranks) into the reference emulator
    (compose.simulate_pipeline) and compare with the measured makespan (max over ranks)."""
    import importlib

    sf = schedfront_module or importlib.import_module("schedfront")
    compose = importlib.import_module(sf.__name__ + ".compose")
    dur: dict[tuple[int, int, str], float] = {}
    for r in runs:
        for k, v in r.durations().items():
            dur[k] = max(dur.get(k, 0.0), v)
    assignment = {k: compose.PipelineOpChoice(v, (op_energy or {}).get((k[0], k[2]), 0.0), 0.0)
                  for k, v in dur.items()}
    spec = compose.PipelineSpec(pp, microbatches)
    t_emu, e_emu = compose.simulate_pipeline(spec, assignment, p_static_w, freq_switch_ms)
    t_meas = max(r.makespan_ms for r in runs)
    out = {"makespan_measured_ms": t_meas, "makespan_emulated_ms": t_emu,
           "rel_error": (t_meas - t_emu) / t_emu if t_emu else None,
           "ops": len(dur), "bubble_fraction_measured": 1.0 - sum(dur.values()) / (pp * t_meas) if t_meas else None}
    if op_energy is not None:
        out["energy_emulated_j"] = e_emu
        meas = [r.energy_j for r in runs if r.energy_j is not None]
        if meas:
            out["energy_measured_j"] = sum(meas)
    return out
