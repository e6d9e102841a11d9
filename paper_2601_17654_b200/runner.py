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
        self.k = 0          # iterations enqueued so far (selects the layer-parity buffers)
        self._slot = None   # host-staging slot the layer currently points at (None: its own tensors)

    def kernels_per_step(self) -> int:
        n = 0
        for name in self.layer.order:
            p = self.layer.programs[name]
            n += sum(u.n_kernels for u in p.units) + p.comm.n_kernels
        return n

    def _select(self, parity: int) -> None:
        """Point the layer at layer-parity `parity` and the executor at the matching graph set."""
        self.layer.set_parity(parity)
        self.engine.exec.variant = (self.layer.parity, self._slot)

    def step(self) -> None:
        """Enqueue one layer iteration on the engine's compute stream (graph replays).  Consecutive
        iterations alternate the FSDP layer-parity buffers (PartitionedLayer.set_parity), so the
        weights gathered by iteration k are the ones iteration k+1 computes with."""
        ex = self.engine.exec
        self._select(self.k % self.layer.parity_period)
        for name in self.layer.order:
            ex.run(self.layer.programs[name], self.schedule[name], self.ncta, 1)
        self.k += 1

    def warm(self) -> None:
        """Capture every partition's graph for every layer parity (executes each once)."""
        k0 = self.k
        for par in range(self.layer.parity_period):
            self._select(par)
            for name in self.layer.order:
                self.engine.exec.graph(self.layer.programs[name], self.schedule[name], self.ncta)
        self._select(k0 % self.layer.parity_period)
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

    # ---------------------------------------------------------------- pipelined host-buffer entry point
    def _use_slot(self, s) -> None:
        """Point the layer's input / output activations at host-staging slot s (None: the layer's own
        tensors); the executor keeps a separate graph set per slot."""
        for a, own, slot in zip(self.layer.nb, self._own, self._slots[s] if s is not None else self._own):
            a["x"], a["dy"], a["dx"] = slot
        self._slot = s
        self.engine.exec.variant = (self.layer.parity, s)

    def prepare_host_pipeline(self) -> None:
        """Allocate the two host-staging slots and capture their graphs (this executes every partition
        once per slot on the current inputs); step_host_async does it on first use otherwise."""
        if not hasattr(self, "_pipe_k"):
            self._pipe_init()

    def _pipe_init(self) -> None:
        dev = self.engine.device
        self._h2d = torch.cuda.Stream(dev)
        self._d2h = torch.cuda.Stream(dev)
        # two device slots, each with its own x / dy / dx and its own captured graphs: step k reads its
        # inputs and writes dx in slot k % 2 directly (no staging copies on the compute stream), so the
        # H2D of step k+1 and the D2H of step k-1 run on copy engines while step k computes
        self._own = [(a["x"], a["dy"], a["dx"]) for a in self.layer.nb]
        self._slots = [[(a["x"].clone(), a["dy"].clone(), torch.empty_like(a["dx"])) for a in self.layer.nb]
                       for _ in range(2)]
        for s in range(2):
            self._use_slot(s)
            self.warm()  # capture this slot's graphs before any pipelined step is queued
        self._use_slot(None)
        ev = lambda: [torch.cuda.Event(), torch.cuda.Event()]
        self._in_ready, self._in_free, self._out_ready, self._out_free = ev(), ev(), ev(), ev()
        self._pipe_k = 0
        self._pipe_used = [False, False]

    def step_host_async(self, xs_host: list[torch.Tensor], dys_host: list[torch.Tensor],
                        dxs_host: list[torch.Tensor]) -> None:
        """Enqueue one iteration from pinned host buffers without waiting for it.

        The H2D of this step's inputs runs on a copy stream into this step's device slot and overlaps
        the previous step's compute; the D2H of this step's dx overlaps the next step's compute. The
        host buffers of a step must stay untouched until `drain()` (or two steps later) returns.
        Call `drain()` to wait for every enqueued step."""
        if not hasattr(self, "_pipe_k"):
            self._pipe_init()
        s = self._pipe_k & 1
        comp = self.engine.exec.compute
        used = self._pipe_used[s]
        slot = self._slots[s]
        with torch.cuda.stream(self._h2d):
            if used:
                self._h2d.wait_event(self._in_free[s])  # step k-2 has finished reading this slot
            for (sx, sdy, _), x, dy in zip(slot, xs_host, dys_host):
                sx.copy_(x, non_blocking=True)
                sdy.copy_(dy, non_blocking=True)
            self._in_ready[s].record(self._h2d)
        comp.wait_event(self._in_ready[s])
        if used:
            comp.wait_event(self._out_free[s])  # step k-2's dx has left this slot
        self._use_slot(s)
        self.step()
        self._in_free[s].record(comp)
        self._out_ready[s].record(comp)
        self._d2h.wait_event(self._out_ready[s])
        with torch.cuda.stream(self._d2h):
            for (_, _, sdx), dx in zip(slot, dxs_host):
                dx.copy_(sdx, non_blocking=True)
            self._out_free[s].record(self._d2h)
        self._pipe_used[s] = True
        self._pipe_k += 1

    def drain(self) -> None:
        if hasattr(self, "_pipe_k"):
            self._d2h.synchronize()
            self._h2d.synchronize()
            self._use_slot(None)
        self.engine.exec.compute.synchronize()

    # ---------------------------------------------------------------- instrumentation
    def unit_times_graph(self, iters: int = 3) -> dict[str, list[float]]:
        """Per-launch-unit durations (ms) inside real iterations executed the way the step executes
        them: every partition (with timing events recorded around each unit on the compute stream,
        the stream the unit's kernels are launched on) captured as a CUDA graph and replayed, comm
        overlapping.  Unlike the eager variant, host-side launch work is not inside the intervals."""
        ex = self.engine.exec
        marks, graphs = [], []
        for name in self.layer.order:
            prog, cfg = self.layer.programs[name], self.schedule[name]
            wrapped = []
            for u in prog.units:
                e0 = torch.cuda.Event(enable_timing=True, external=True)
                e1 = torch.cuda.Event(enable_timing=True, external=True)
                marks.append((u.name, e0, e1))

                def fn(st, u=u, e0=e0, e1=e1):
                    e0.record(st)
                    u.fn(st)
                    e1.record(st)
                wrapped.append(type(u)(u.name, u.spec, fn, u.kind, u.n_kernels))
            tmp = type(prog)(prog.name, wrapped, prog.comm, prog.comm_group_size)
            ex.issue(tmp, cfg, self.ncta)  # eager once (first-call setup outside the capture)
            torch.cuda.synchronize(self.engine.device)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=ex.compute):
                ex.issue(tmp, cfg, self.ncta)
            graphs.append(g)
        out: dict[str, list[float]] = {}
        for _ in range(iters):
            with torch.cuda.stream(ex.compute):
                for g in graphs:
                    g.replay()
            torch.cuda.synchronize(self.engine.device)
            for nm, e0, e1 in marks:
                out.setdefault(nm, []).append(e0.elapsed_time(e1))
        return out

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
