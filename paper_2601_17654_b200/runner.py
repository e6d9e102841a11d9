"""Layer-iteration runner: all partitions of one layer (fwd + bwd, 2 nanobatches) under a schedule
assignment, plus the host-buffer entry point used for end-to-end timing.

The default assignment is the paper's baseline "nanobatching" schedule (BASELINE.md
§3): every partition at f_max, the collective at its default CTA count, launched with the first
kernel and free to run to the end — ScheduleConfig(f_max, default_ncta, overlap(0, n)).
"""

from __future__ import annotations

import torch

from .domain import LaunchTiming, ScheduleConfig


def default_schedule(layer, gpu) -> dict[str, ScheduleConfig]:
    return {name: ScheduleConfig(gpu.f_max_mhz, int(gpu.sm_bw_saturation),
                                 LaunchTiming.overlap(0, len(layer.programs[name].units)))
            for name in layer.order}


def sequential_schedule(layer, gpu) -> dict[str, ScheduleConfig]:
    return {name: ScheduleConfig(gpu.f_max_mhz, int(gpu.sm_bw_saturation), LaunchTiming.sequential())
            for name in layer.order}


class LayerRunner:
    def __init__(self, layer, engine, schedule: dict[str, ScheduleConfig] | None = None):
        self.layer = layer
        self.engine = engine
        self.schedule = schedule or default_schedule(layer, engine.gpu)
        self.ncta = engine.default_ncta()

    def kernels_per_step(self) -> int:
        n = 0
        for name in self.layer.order:
            p = self.layer.programs[name]
            n += sum(u.n_kernels for u in p.units) + p.comm.n_kernels
        return n

    def step(self) -> None:
        """Enqueue one layer iteration on the engine's compute stream (graph replays)."""
        ex = self.engine.exec
        for name in self.layer.order:
            ex.run(self.layer.programs[name], self.schedule[name], self.ncta, 1)

    def warm(self) -> None:
        for name in self.layer.order:
            self.engine.exec.graph(self.layer.programs[name], self.schedule[name], self.ncta)
        torch.cuda.synchronize(self.engine.device)

    # ---------------------------------------------------------------- host-buffer entry point
    def step_host(self, xs_host: list[torch.Tensor], dys_host: list[torch.Tensor],
                  dxs_host: list[torch.Tensor]) -> None:
        """One iteration from pinned host inputs to pinned host input-gradients: H2D of every
        nanobatch's activations and upstream grads, the partitioned iteration, D2H of dx."""
        st = self.engine.exec.compute
        with torch.cuda.stream(st):
            for a, x, dy in zip(self.layer.nb, xs_host, dys_host):
                a["x"].copy_(x, non_blocking=True)
                a["dy"].copy_(dy, non_blocking=True)
        self.step()
        with torch.cuda.stream(st):
            for a, dx in zip(self.layer.nb, dxs_host):
                dx.copy_(a["dx"], non_blocking=True)
        st.synchronize()

    # ---------------------------------------------------------------- instrumentation
    def unit_times(self, iters: int = 3) -> dict[str, list[float]]:
        """Per-launch-unit durations (ms) inside real iterations: eager issue with CUDA events
        recorded on the stream each unit is launched on (the compute stream), comm overlapping."""
        ex = self.engine.exec
        out: dict[str, list[float]] = {}
        for _ in range(iters):
            marks = []
            for name in self.layer.order:
                prog, cfg = self.layer.programs[name], self.schedule[name]
                wrapped = []
                for u in prog.units:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    marks.append((u.name, e0, e1))

                    def fn(st, u=u, e0=e0, e1=e1):
                        e0.record(st)
                        u.fn(st)
                        e1.record(st)
                    wrapped.append(type(u)(u.name, u.spec, fn, u.kind, u.n_kernels))
                tmp = type(prog)(prog.name, wrapped, prog.comm, prog.comm_group_size)
                ex.issue(tmp, cfg, self.ncta)
            torch.cuda.synchronize(self.engine.device)
            for nm, e0, e1 in marks:
                out.setdefault(nm, []).append(e0.elapsed_time(e1))
        return out
