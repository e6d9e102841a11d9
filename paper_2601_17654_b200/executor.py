"""Partition executor: one (PartitionProgram, schedule) -> two CUDA streams (optionally a CUDA graph).

Implements the reference's execution semantics on hardware (simgpu.py:181-261):

  sequential (simgpu.py:181-188, the Megatron baseline PAPER.md:226):
      all compute units, then the collective at its default CTA count, on ONE stream.
  overlap(start, span) (simgpu.py:191-261, LaunchTiming domain.py:88-118):
      compute units [0, start) on the compute stream;
      fork: the high-priority comm stream waits for them, then launches the collective with
            exactly `sm_alloc` CTAs (each CTA owns a whole SM — comm.cu);
      the launch-completion event of the collective (cudaLaunchAttributeLaunchCompletionEvent)
            gates compute unit `start`, so the collective's CTAs are resident before the compute
            kernels fill the remaining SMs;
      units [start, start+span_eff) run concurrently on the other SMs (GEMMs use a dynamic tile
            scheduler, so SMs released by the collective are picked up mid-kernel);
      sync point: unit start+span_eff waits for the collective (the exposed tail);
      the remaining units follow; the partition ends when both streams are done.

`overlap_launch_overhead_ms` of the simulator is not modelled: it is whatever the real fork/join
costs, and it is inside every measured time.
"""

from __future__ import annotations

import torch

from .device import validate_schedule


class ScheduleExecutor:
    def __init__(self, device, comm=None, use_graphs: bool = True, launch_gate: bool = True):
        self.device = torch.device(device)
        self.comm = comm
        self.compute = torch.cuda.Stream(self.device, priority=0)
        lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
        self.comm_stream = torch.cuda.Stream(self.device, priority=-1)
        self.ev_fork = torch.cuda.Event()
        self.ev_launched = torch.cuda.Event()
        self.ev_done = torch.cuda.Event()
        self.use_graphs = use_graphs
        self.launch_gate = launch_gate
        self.gate_status = "disabled" if not launch_gate else "unprobed"
        self.graphs: dict[tuple, torch.cuda.CUDAGraph] = {}
        self.graph_failures: dict[tuple, str] = {}
        # graph-set tag: callers that swap the tensors a program reads (LayerRunner's host-staging
        # slots) keep one captured graph per (program, schedule, variant)
        self.variant = None

    # ------------------------------------------------------------------ launch gate
    def probe_gate(self) -> bool:
        """Probe once whether collectives can carry the launch-completion event (a profiler replaying
        kernels, for one, rejects it); on failure the executor forks the collective ungated."""
        if not self.launch_gate or self.comm is None:
            return False
        if self.gate_status != "unprobed":
            return self.launch_gate
        from . import _lib

        ev = torch.cuda.Event()
        try:
            ev.record(self.compute)
            _lib.call("kpo_probe_launch_completion", ev.cuda_event, self.comm_stream.cuda_stream)
            self.compute.wait_event(ev)
            self.compute.synchronize()
            self.gate_status = "ok"
        except Exception as ex:  # noqa: BLE001 - any refusal means: no gate
            self.launch_gate = False
            self.gate_status = f"off: {type(ex).__name__}: {ex}"
            try:
                torch.cuda.synchronize(self.device)
            except Exception:
                pass
        return self.launch_gate

    # ------------------------------------------------------------------ enqueue
    def issue(self, prog, config, default_ncta: int) -> None:
        """Enqueue one execution of `prog` under `config` (eager, or inside a capture)."""
        comp, side = self.compute, self.comm_stream
        units = prog.units
        n = len(units)
        t = config.timing
        if t.is_sequential:
            for u in units:
                u.fn(comp)
            prog.comm.fn(comp, default_ncta)
            return
        start = t.start
        span = min(t.span, n - start)
        for u in units[:start]:
            u.fn(comp)
        self.ev_fork.record(comp)
        side.wait_event(self.ev_fork)
        gate = self.launch_gate and self.comm is not None and self.probe_gate()
        if gate:
            self.comm.arm_launch_event(self.ev_launched)
        try:
            prog.comm.fn(side, int(config.sm_alloc))
        finally:
            if gate:
                self.comm.disarm_launch_event()
        self.ev_done.record(side)
        if gate:
            try:
                comp.wait_event(self.ev_launched)
            except Exception as ex:  # noqa: BLE001 - e.g. a profiler replaying the launch drops the event
                # the gate only orders residency (the collective's CTAs before the span's kernels);
                # without it the schedule is still correct, so continue ungated from here on
                self.launch_gate = False
                self.gate_status = f"off after first use: {type(ex).__name__}: {ex}"
        for u in units[start:start + span]:
            u.fn(comp)
        comp.wait_event(self.ev_done)  # sync point (or the join at the end when span reaches n)
        for u in units[start + span:]:
            u.fn(comp)

    # ------------------------------------------------------------------ graphs
    def _key(self, prog, config, default_ncta):
        t = config.timing
        key = (prog.name, "seq", default_ncta) if t.is_sequential else (prog.name, int(config.sm_alloc), t.start,
                                                                         min(t.span, len(prog.units) - t.start))
        return key if self.variant is None else key + (self.variant,)

    def graph(self, prog, config, default_ncta: int):
        key = self._key(prog, config, default_ncta)
        if key in self.graphs:
            return self.graphs[key]
        if key in self.graph_failures or not self.use_graphs:
            return None
        # warm up eagerly once (first-call attribute setup happens outside capture)
        self.issue(prog, config, default_ncta)
        self.compute.synchronize()
        g = torch.cuda.CUDAGraph()
        try:
            with torch.cuda.graph(g, stream=self.compute, capture_error_mode="thread_local"):
                self.issue(prog, config, default_ncta)
        except Exception as ex:  # fall back to eager streams for this schedule
            self.graph_failures[key] = repr(ex)
            torch.cuda.synchronize(self.device)
            return None
        self.graphs[key] = g
        return g

    def run(self, prog, config, default_ncta: int, reps: int = 1) -> None:
        """Enqueue `reps` executions on the compute stream (graph replay when available)."""
        g = self.graph(prog, config, default_ncta)
        with torch.cuda.stream(self.compute):
            for _ in range(reps):
                if g is not None:
                    g.replay()
                else:
                    self.issue(prog, config, default_ncta)

    def time_ms(self, prog, config, default_ncta: int, reps: int = 10, warmup: int = 2) -> float:
        self.run(prog, config, default_ncta, warmup)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(self.compute)
        self.run(prog, config, default_ncta, reps)
        e1.record(self.compute)
        e1.synchronize()
        return e0.elapsed_time(e1) / reps

    def check(self, partition, config, gpu) -> None:
        validate_schedule(partition, config, gpu)
