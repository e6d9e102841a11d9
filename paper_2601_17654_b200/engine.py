"""Engine: the drop-in replacement for the reference's hot path.

  reference (schedfront)                                  here
  ------------------------------------------------------  ------------------------------------
  simulate_schedule(partition, config, gpu)               Engine.execute(partition, config, gpu)
      simgpu.py:264-286                                   one real execution (short window)
  measure(partition, config, gpu, thermal, protocol,      Engine.measure(...same signature...)
          state)  simgpu.py:321-364                       thermally-stable window on hardware
  InvalidConfigError  simgpu.py:85, :270-279              same checks, before any native call

`measure` follows the reference protocol field by field: warm up for `warmup_s` (graph replays),
execute back-to-back for reps = max(1, window_s // exec_s) (simgpu.py:347), read time from CUDA
events and energy from the NVML counter over the same window, cool down for `cooldown_s`, and
write the GPU temperature into `state.temperature_c`.  Dynamic energy is what the counter saw
minus static power x time, and the result is `Measurement.build(t, E - P_s t, P_s)`
(domain.py:245-248), so total == dyn + static exactly as the reference guarantees.

The reference optimizer calls `measure` as a module global (mbo.py:290-292); `install()` swaps it
(and the `simulate_schedule` imports of oracle.py / compose.py) for this engine.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import torch

from .device import GpuModel, InvalidConfigError, validate_schedule
from .domain import Measurement
from .executor import ScheduleExecutor
from .power import EnergySampler, FrequencyController, Nvml


@dataclass
class Observation:
    """Side-channel facts of the last measurement (not part of Measurement)."""

    reps: int = 0
    window_s: float = 0.0
    gpu_ms: float = 0.0
    energy_j: float = 0.0
    sm_mhz: float = 0.0
    temperature_c: float = 0.0
    reasons: tuple = ()
    clock_control: str = ""
    graph: bool = False


class Engine:
    def __init__(self, programs, gpu: GpuModel, device=None, comm=None, clock_control: bool = False,
                 use_graphs: bool = True, launch_gate: bool = True, measurement_cls=Measurement):
        self.gpu = gpu
        self.device = torch.device(device or "cuda")
        self.comm = comm
        self.programs = {}
        for p in (programs.values() if isinstance(programs, dict) else programs):
            self.programs[p.name] = p
        self.exec = ScheduleExecutor(self.device, comm=comm, use_graphs=use_graphs, launch_gate=launch_gate)
        self.exec.ev_launched.record(self.exec.compute)  # materialise the CUDA event
        self.nvml = Nvml(self.device.index or 0)
        self.freq = FrequencyController(self.nvml, enable=clock_control)
        self.sampler = EnergySampler(self.nvml)
        self.sampler.start()
        self.measurement_cls = measurement_cls
        self.last = Observation()
        self._exec_ms: dict[tuple, float] = {}

    @classmethod
    def for_layer(cls, layer, gpu: GpuModel, **kw) -> "Engine":
        return cls(layer.programs, gpu, device=layer.device, comm=layer.comm, **kw)

    def close(self) -> None:
        self.sampler.stop()
        self.freq.release()

    # ------------------------------------------------------------------ resolution
    def program_for(self, partition):
        prog = self.programs.get(getattr(partition, "name", None))
        if prog is None:
            raise KeyError(f"no registered program for partition {getattr(partition, 'name', partition)!r}")
        if len(partition.comp_kernels) != len(prog.units):
            raise ValueError(f"partition {prog.name!r}: {len(partition.comp_kernels)} kernels vs "
                             f"{len(prog.units)} launch units")
        return prog

    def default_ncta(self, gpu=None) -> int:
        return int((gpu or self.gpu).sm_bw_saturation)

    # ------------------------------------------------------------------ core window
    def _window(self, prog, config, ncta, warmup_s: float, window_s: float) -> tuple[float, float, int]:
        ex = self.exec
        key = ex._key(prog, config, ncta)
        est = self._exec_ms.get(key)
        if est is None:
            est = ex.time_ms(prog, config, ncta, reps=3, warmup=1)
            self._exec_ms[key] = est
        if warmup_s > 0:
            ex.run(prog, config, ncta, max(1, int(warmup_s * 1e3 / est)))
        reps = max(1, int(window_s // (est / 1e3)))
        torch.cuda.synchronize(self.device)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(ex.compute)
        ex.run(prog, config, ncta, reps)
        e1.record(ex.compute)
        e1.synchronize()
        t1 = time.perf_counter()
        gpu_ms = e0.elapsed_time(e1)
        energy = self.sampler.window_j(t0, t1)
        idle = max(0.0, (t1 - t0) - gpu_ms / 1e3)
        energy -= idle * self.gpu.p_static_w  # host-side launch latency at the window edges
        self._exec_ms[key] = gpu_ms / reps
        clocks = self.sampler.clocks_summary(t0, t1)
        self.last = Observation(reps=reps, window_s=t1 - t0, gpu_ms=gpu_ms, energy_j=energy,
                                sm_mhz=clocks.get("sm_mhz", 0.0), reasons=tuple(clocks.get("reasons", ())),
                                clock_control=self.freq.reason, graph=key in ex.graphs)
        return gpu_ms / reps, energy / reps, reps

    def _prepare(self, partition, config, gpu):
        gpu = gpu or self.gpu
        validate_schedule(partition, config, gpu)  # InvalidConfigError before any native call
        prog = self.program_for(partition)
        self.freq.set(config.frequency_mhz)
        return gpu, prog

    # ------------------------------------------------------------------ public API
    def execute(self, partition, config, gpu: GpuModel | None = None, window_s: float = 0.3):
        """One noise-free execution (reference simulate_schedule)."""
        gpu, prog = self._prepare(partition, config, gpu)
        t_ms, e_j, _ = self._window(prog, config, self.default_ncta(gpu), 0.05, window_s)
        return self.measurement_cls.build(t_ms, e_j - gpu.p_static_w * t_ms / 1e3, gpu.p_static_w)

    def measure_local(self, name: str, config, warmup_s: float, window_s: float, cooldown_s: float,
                      ncta: int | None = None) -> tuple[float, float, float]:
        """This rank's (time_ms, energy_j per execution, temperature) for a registered program;
        the SPMD driver (spmd.py) combines ranks."""
        prog = self.programs[name]
        self.freq.set(config.frequency_mhz)
        t_ms, e_j, _ = self._window(prog, config, ncta or self.default_ncta(), warmup_s, window_s)
        if cooldown_s > 0:
            time.sleep(cooldown_s)
        temp = self.nvml.temperature_c()
        self.last.temperature_c = temp
        return t_ms, e_j, temp

    def measure(self, partition, config, gpu: GpuModel | None = None, thermal=None, protocol=None, state=None):
        """Thermally-stable profiling pass (reference measure, simgpu.py:321-364)."""
        gpu, prog = self._prepare(partition, config, gpu)
        t_ms, e_j, temp = self.measure_local(prog.name, config, getattr(protocol, "warmup_s", 2.0),
                                             getattr(protocol, "window_s", 5.0), getattr(protocol, "cooldown_s", 5.0),
                                             self.default_ncta(gpu))
        if state is not None:
            state.temperature_c = temp
        return self.measurement_cls.build(t_ms, e_j - gpu.p_static_w * t_ms / 1e3, gpu.p_static_w)

    # reference-shaped free functions bound to this engine
    def measure_fn(self):
        def measure(partition, config, gpu, thermal, protocol, state):
            return self.measure(partition, config, gpu, thermal, protocol, state)
        return measure

    def simulate_fn(self):
        def simulate_schedule(partition, config, gpu):
            return self.execute(partition, config, gpu)
        return simulate_schedule


def install(engine, schedfront_module=None):
    """Swap the reference's hot path for `engine` (mbo.py:30,291; oracle.py:24; compose.py:29).
    Returns a function restoring the previous bindings."""
    from .compat import patch_reference, reference_measurement_cls

    engine.measurement_cls = reference_measurement_cls(schedfront_module)
    return patch_reference(engine.measure_fn(), engine.simulate_fn(), schedfront_module)


__all__ = ["Engine", "Observation", "install", "InvalidConfigError", "math"]
