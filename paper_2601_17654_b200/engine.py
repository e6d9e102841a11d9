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
events and energy from the NVML counter over the same window, cool down for `cooldown_s` (and,
optionally, until the GPU is below `cooldown_target_c`), and write the GPU
temperature into `state.temperature_c`.  Dynamic energy is what the counter saw minus static
power x time, and the result is `Measurement.build(t, E - P_s t, P_s)` (domain.py:245-248), so
total == dyn + static exactly as the reference guarantees.

Frequency (ScheduleConfig.frequency_mhz, domain.py:151): the reference always honours f
(simgpu.py:144-178).  Here f is applied with NVML locked clocks when the driver permits it and
the clock the GPU actually ran is checked against it after the window.  When locked clocks are
refused (this pool: profiles/r2_clock_probe.json), the only frequency the engine can honour is the
unlocked default f_max (the boost ceiling); any other f raises `FrequencyUnavailableError` (an
`InvalidConfigError`) before anything runs, so a profile table can never carry a mislabelled
frequency.

Multi-rank: every rank must launch the same number of collectives (their per-CTA flag barriers
wait for the peers), so the warm-up and window repetition counts are derived from one execution-
time estimate agreed across ranks (`agree_ms`, the MAX over ranks; spmd.py sets it).

The reference optimizer calls `measure` as a module global (mbo.py:290-292); `install()` swaps it
(and the `simulate_schedule` imports of oracle.py / compose.py) for this engine.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import torch

from .device import GpuModel, InvalidConfigError, validate_schedule
from .domain import Measurement
from .executor import ScheduleExecutor
from .power import EnergySampler, FrequencyController, Nvml

# throttle reasons that invalidate a sample (re-measured once, then flagged); sw_power_cap is the
# normal state of a dense-GEMM partition at ~1 kW and is only recorded
BAD_REASONS = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "hw_power_brake_slowdown")


def rep_counts(est_ms: float, warmup_s: float, window_s: float) -> tuple[int, int]:
    """(warm-up executions, window executions) for an execution-time estimate: the window count is
    the reference's reps = max(1, window // exec) (simgpu.py:347)."""
    warm = max(1, int(warmup_s * 1e3 / est_ms)) if warmup_s > 0 else 0
    return warm, max(1, int(window_s // (est_ms / 1e3)))


class FrequencyUnavailableError(InvalidConfigError):
    """The requested SM clock cannot be applied on this GPU (locked clocks refused, or the GPU ran
    above the requested clock).  Subclass of InvalidConfigError so callers that screen invalid
    configurations (reference mbo / cli) treat it the same way."""


@dataclass
class Observation:
    """Side-channel facts of the last measurement (not part of Measurement)."""

    reps: int = 0
    window_s: float = 0.0
    gpu_ms: float = 0.0
    energy_j: float = 0.0
    sm_mhz: float = 0.0
    requested_mhz: float = 0.0
    temperature_c: float = 0.0
    temperature_start_c: float = 0.0
    cooldown_s: float = 0.0
    reasons: tuple = ()
    flags: tuple = ()
    clock_control: str = ""
    graph: bool = False
    retried: int = 0
    energy_trials_j: tuple = ()

    def as_dict(self) -> dict:
        return {k: (list(v) if isinstance(v, tuple) else v) for k, v in self.__dict__.items()}


class Engine:
    def __init__(self, programs, gpu: GpuModel, device=None, comm=None, clock_control: bool = True,
                 use_graphs: bool = True, launch_gate: bool = True, measurement_cls=Measurement,
                 cooldown_target_c: float | None = None, cooldown_max_s: float = 30.0,
                 energy_outlier_frac: float | None = 0.10,
                 reject_throttled: bool = True, clock_tolerance_mhz: float = 30.0):
        self.gpu = gpu
        self.device = torch.device(device or "cuda")
        self.comm = comm
        self.programs = {}
        for p in (programs.values() if isinstance(programs, dict) else programs):
            self.programs[p.name] = p
        self.exec = ScheduleExecutor(self.device, comm=comm, use_graphs=use_graphs, launch_gate=launch_gate)
        self.exec.ev_launched.record(self.exec.compute)  # materialise the CUDA event
        self.exec.probe_gate()
        self.nvml = Nvml(self.device.index or 0)
        self.freq = FrequencyController(self.nvml, enable=clock_control)
        self.sampler = EnergySampler(self.nvml)
        self.sampler.start()
        self.measurement_cls = measurement_cls
        self.cooldown_target_c = cooldown_target_c
        self.cooldown_max_s = cooldown_max_s
        self.reject_throttled = reject_throttled
        self.clock_tolerance_mhz = clock_tolerance_mhz
        self.last = Observation()
        self.history: list[Observation] = []
        self._exec_ms: dict[tuple, float] = {}
        # multi-rank: maps this rank's execution-time estimate to the value every rank uses
        self.agree_ms = None
        # energy-outlier re-measurement: a window whose average power departs from this program's
        # running median by more than energy_outlier_frac (after 5 windows) is measured twice more and
        # the median-energy window of the three is kept (NVML counter outliers)
        self.energy_outlier_frac = energy_outlier_frac
        self._power_hist: dict[str, list[float]] = {}

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

    # ------------------------------------------------------------------ frequency
    def frequencies(self, gpu: GpuModel | None = None) -> list[float]:
        """The SM clocks this engine can honour: the NVML grid when clocks can be locked, else f_max."""
        gpu = gpu or self.gpu
        if self.freq.available:
            return [f for f in self.nvml.supported_sm_clocks() if f <= gpu.f_max_mhz]
        return [float(gpu.f_max_mhz)]

    def check_frequency(self, f_mhz: float, gpu: GpuModel | None = None) -> None:
        gpu = gpu or self.gpu
        if self.freq.available:
            return
        if abs(float(f_mhz) - float(gpu.f_max_mhz)) > 0.5:
            raise FrequencyUnavailableError(
                f"frequency {f_mhz} MHz cannot be applied: NVML locked clocks are unavailable on this GPU "
                f"({self.freq.reason}); only the unlocked default f_max = {gpu.f_max_mhz} MHz is measurable")

    def _apply_frequency(self, f_mhz: float, gpu: GpuModel | None = None) -> None:
        self.check_frequency(f_mhz, gpu)
        if self.freq.available and not self.freq.set(f_mhz):
            raise FrequencyUnavailableError(f"NVML refused locked clocks at {f_mhz} MHz")

    # ------------------------------------------------------------------ core window
    def estimate_ms(self, prog, config, ncta) -> float:
        ex = self.exec
        key = ex._key(prog, config, ncta)
        est = self._exec_ms.get(key)
        if est is None:
            est = ex.time_ms(prog, config, ncta, reps=3, warmup=1)
            self._exec_ms[key] = est
        return est

    def _window(self, prog, config, ncta, warmup_s: float, window_s: float) -> tuple[float, float, int]:
        ex = self.exec
        key = ex._key(prog, config, ncta)
        est = self.estimate_ms(prog, config, ncta)
        if self.agree_ms is not None:
            est = float(self.agree_ms(est))  # identical repetition counts on every rank
        warm, reps = rep_counts(est, warmup_s, window_s)
        if warm:
            ex.run(prog, config, ncta, warm)
        torch.cuda.synchronize(self.device)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        temp0 = self.nvml.temperature_c()
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
        reasons = tuple(clocks.get("reasons", ()))
        flags = tuple(r for r in reasons if r in BAD_REASONS)
        if "sw_power_cap" in reasons:
            flags += ("power_capped",)
        self.last = Observation(reps=reps, window_s=t1 - t0, gpu_ms=gpu_ms, energy_j=energy,
                                sm_mhz=clocks.get("sm_mhz", 0.0), requested_mhz=float(config.frequency_mhz),
                                temperature_start_c=temp0, reasons=reasons, flags=flags,
                                clock_control=self.freq.reason, graph=key in ex.graphs)
        return gpu_ms / reps, energy / reps, reps

    def _cooldown(self, cooldown_s: float) -> float:
        """Idle for cooldown_s, then (if a target is set) until the GPU is below it; returns the idle time."""
        t0 = time.perf_counter()
        if cooldown_s > 0:
            time.sleep(cooldown_s)
        if self.cooldown_target_c is not None:
            while (self.nvml.temperature_c() > self.cooldown_target_c
                   and time.perf_counter() - t0 < cooldown_s + self.cooldown_max_s):
                time.sleep(0.25)
        return time.perf_counter() - t0

    def _verify_clock(self, config) -> None:
        """With locked clocks the GPU must not run above the requested clock (it may run below it
        under a power cap, which is flagged, not rejected)."""
        obs = self.last
        if self.freq.available and obs.sm_mhz > float(config.frequency_mhz) + self.clock_tolerance_mhz:
            raise FrequencyUnavailableError(
                f"requested {config.frequency_mhz} MHz but the GPU ran at {obs.sm_mhz} MHz (median of the window)")
        if obs.sm_mhz and obs.sm_mhz < float(config.frequency_mhz) - self.clock_tolerance_mhz:
            obs.flags = tuple(obs.flags) + ("below_requested_clock",)

    def _prepare(self, partition, config, gpu):
        gpu = gpu or self.gpu
        validate_schedule(partition, config, gpu)  # InvalidConfigError before any native call
        self.check_frequency(config.frequency_mhz, gpu)
        prog = self.program_for(partition)
        return gpu, prog

    # ------------------------------------------------------------------ public API
    def execute(self, partition, config, gpu: GpuModel | None = None, window_s: float = 1.0):
        """One noise-free execution (reference simulate_schedule).  The window defaults to 1 s, about
        ten steps of the NVML energy counter (power.py)."""
        gpu, prog = self._prepare(partition, config, gpu)
        self._apply_frequency(config.frequency_mhz, gpu)
        t_ms, e_j, _ = self._window(prog, config, self.default_ncta(gpu), 0.05, window_s)
        self._verify_clock(config)
        self.history.append(self.last)
        return self.measurement_cls.build(t_ms, e_j - gpu.p_static_w * t_ms / 1e3, gpu.p_static_w)

    def measure_local(self, name: str, config, warmup_s: float, window_s: float, cooldown_s: float,
                      ncta: int | None = None) -> tuple[float, float, float]:
        """This rank's (time_ms, energy_j per execution, temperature) for a registered program;
        the SPMD driver (spmd.py) combines ranks.  A window that saw a hardware / thermal slowdown
        is re-measured once (after the cooldown) and flagged if it happens again."""
        prog = self.programs[name]
        self._apply_frequency(config.frequency_mhz)
        ncta = ncta or self.default_ncta()
        retried = 0
        while True:
            t_ms, e_j, _ = self._window(prog, config, ncta, warmup_s, window_s)
            self._verify_clock(config)
            obs = self.last
            obs.cooldown_s = self._cooldown(cooldown_s)
            # every rank takes the same branch: the decision must not depend on rank-local flags when
            # ranks are coupled by collectives, so the retry is driven by the agreed hook if present
            bad = any(f in BAD_REASONS for f in obs.flags)
            if self.agree_ms is not None:
                bad = bool(self.agree_ms(1.0 if bad else 0.0) > 0.5)
            if not (self.reject_throttled and bad and retried == 0):
                break
            retried += 1
        t_ms, e_j, obs = self._energy_outlier_check(name, prog, config, ncta, warmup_s, window_s, cooldown_s,
                                                    t_ms, e_j, obs)
        temp = self.nvml.temperature_c()
        obs.temperature_c = temp
        obs.retried = retried
        self.history.append(obs)
        return t_ms, e_j, temp

    def _energy_outlier_check(self, name, prog, config, ncta, warmup_s, window_s, cooldown_s, t_ms, e_j, obs):
        """Re-measure a window whose average power is an outlier for this program (see __init__);
        returns the (time, energy, observation) of the median-energy window of the three."""
        hist = self._power_hist.setdefault(name, [])
        power = e_j / max(t_ms / 1e3, 1e-12)
        frac = self.energy_outlier_frac
        suspect = False
        if frac is not None and len(hist) >= 5:
            med = sorted(hist)[len(hist) // 2]
            suspect = abs(power - med) > frac * med
        if self.agree_ms is not None and frac is not None and len(hist) >= 5:
            suspect = bool(self.agree_ms(1.0 if suspect else 0.0) > 0.5)  # same branch on every rank
        if suspect:
            trials = [(e_j, t_ms, obs)]
            for _ in range(2):
                t2, e2, _ = self._window(prog, config, ncta, warmup_s, window_s)
                o2 = self.last
                o2.cooldown_s = self._cooldown(cooldown_s)
                trials.append((e2, t2, o2))
            energies = tuple(round(x[0], 6) for x in trials)  # in measurement order
            e_j, t_ms, obs = sorted(trials, key=lambda x: x[0])[1]
            obs.flags = tuple(obs.flags) + ("energy_outlier_remeasured",)
            obs.energy_trials_j = energies
            power = e_j / max(t_ms / 1e3, 1e-12)
        hist.append(power)
        return t_ms, e_j, obs

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


__all__ = ["Engine", "Observation", "install", "rep_counts", "InvalidConfigError", "FrequencyUnavailableError", "BAD_REASONS",
           "math", "field"]
