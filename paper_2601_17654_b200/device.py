"""Device descriptor and profiling-protocol types for the B200 engine.

`GpuModel` keeps the reference's field names (simgpu.py:35-82) so the reference optimizer's
space enumeration (`mbo.enumerate_space`, mbo.py:85-127) and analytic pruning keep working when
handed a B200 descriptor; on hardware the descriptor no longer *predicts* execution, it only
prunes the candidate space and carries the static power used by `Measurement.build`.

`ThermalModel`, `ProfilingProtocol`, `ThermalState` mirror simgpu.py:89-141.  On hardware:
warmup_s / window_s / cooldown_s are real durations; noise_std_frac and counter_quantum_j are
simulation knobs and are ignored; ThermalState.temperature_c is refreshed from NVML.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np


class InvalidConfigError(ValueError):
    """Schedule configuration is not executable on this GPU (reference simgpu.py:85-86)."""


@dataclass(frozen=True)
class GpuModel:
    num_sms: int = 108
    peak_flops_per_sm_mhz: float = 2.0e9
    mem_bw_gbps: float = 1555.0
    net_bw_gbps: float = 240.0
    sm_bw_saturation: int = 8
    p_static_w: float = 60.0
    kappa: float = 1.2e-7
    f_max_mhz: float = 1410.0
    freq_switch_ms: float = 5.0
    e_flop_j: float = 1.1e-12
    e_byte_j: float = 1.0e-10
    e_comm_byte_j: float = 2.5e-10
    overlap_launch_overhead_ms: float = 0.05

    def __post_init__(self):
        if self.sm_bw_saturation > self.num_sms:
            raise ValueError("sm_bw_saturation cannot exceed num_sms")
        for name in ("num_sms", "peak_flops_per_sm_mhz", "mem_bw_gbps", "net_bw_gbps", "sm_bw_saturation",
                     "p_static_w", "kappa", "f_max_mhz"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")

    @property
    def mem_bw_bps(self) -> float:
        return self.mem_bw_gbps * 1e9

    @property
    def net_bw_bps(self) -> float:
        return self.net_bw_gbps * 1e9

    def flop_rate(self, sm_count: float, freq_mhz: float) -> float:
        return sm_count * self.peak_flops_per_sm_mhz * freq_mhz

    def comm_rate_bps(self, sm_count: int) -> float:
        return self.net_bw_bps * min(1.0, sm_count / self.sm_bw_saturation)


def b200_model(hbm_gbs: float = 6539.9, bf16_tflops: float = 1640.5, f_max_mhz: float = 1965.0,
               net_bw_gbps: float = 770.0, sm_bw_saturation: int = 16, p_static_w: float = 205.0,
               num_sms: int = 148) -> GpuModel:
    """B200 descriptor.  Defaults: HBM copy bandwidth and cuBLAS bf16 burst peak from
    MEASURED_PEAKS.json (driver-measured on this pool), f_max = NVML max SM clock (1965 MHz),
    idle power measured on the box (tools/box_probe.py: 204.6 W), NVLink peer bandwidth 770 GB/s
    (B200_PROFILING.md).  `sm_bw_saturation` is the comm CTA count that saturates the link; it
    is re-measured by the collective microbench (bench_comm)."""
    return GpuModel(
        num_sms=num_sms,
        peak_flops_per_sm_mhz=bf16_tflops * 1e12 / (num_sms * f_max_mhz),
        mem_bw_gbps=hbm_gbs,
        net_bw_gbps=net_bw_gbps,
        sm_bw_saturation=sm_bw_saturation,
        p_static_w=p_static_w,
        f_max_mhz=f_max_mhz,
        overlap_launch_overhead_ms=0.0,
    )


DESCRIPTOR_PATH = "profiles/r2_descriptor.json"


def b200_model_measured(path: str | None = None) -> GpuModel:
    """The B200 descriptor built from committed measurements (tools/calibrate_descriptor.py ->
    profiles/r2_descriptor.json): effective tensor / HBM rates of the layer's own kernels, the
    collective's bus bandwidth and its CTA-saturation knee, idle power, NVML f_max.  This is what the
    optimizer's space pruning (mbo.py:107-114) and the default comm CTA count use; falls back to
    `b200_model()` when the file is absent."""
    import json
    import os

    path = path or os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), DESCRIPTOR_PATH)
    try:
        with open(path) as f:
            d = json.load(f)["descriptor"]
    except (OSError, KeyError, ValueError):
        return b200_model()
    return GpuModel(num_sms=int(d["num_sms"]), peak_flops_per_sm_mhz=float(d["peak_flops_per_sm_mhz"]),
                    mem_bw_gbps=float(d["mem_bw_gbps"]), net_bw_gbps=float(d["net_bw_gbps"]),
                    sm_bw_saturation=int(d["sm_bw_saturation"]), p_static_w=float(d["p_static_w"]),
                    f_max_mhz=float(d["f_max_mhz"]), overlap_launch_overhead_ms=float(d["overlap_launch_overhead_ms"]))


def load_measured_peaks(path: str | None = None) -> dict:
    import json
    import os

    path = path or os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return json.load(f)
    except OSError:
        return {}


@dataclass(frozen=True)
class ThermalModel:
    ambient_c: float = 30.0
    heat_coeff: float = 0.0
    cool_tau_s: float = 0.0
    power_temp_coeff: float = 0.0

    def __post_init__(self):
        for name in ("heat_coeff", "cool_tau_s", "power_temp_coeff"):
            if getattr(self, name) < 0:
                raise ValueError(f"{name} must be >= 0")


@dataclass(frozen=True)
class ProfilingProtocol:
    warmup_s: float = 2.0
    window_s: float = 5.0
    cooldown_s: float = 5.0
    noise_std_frac: float = 0.0
    counter_quantum_j: float = 0.0
    seed: int = 0

    def __post_init__(self):
        if self.window_s <= 0:
            raise ValueError("window_s must be positive")
        if self.cooldown_s < 0 or self.warmup_s < 0:
            raise ValueError("durations must be >= 0")
        if self.noise_std_frac < 0 or self.counter_quantum_j < 0:
            raise ValueError("noise magnitudes must be >= 0")


@dataclass
class ThermalState:
    temperature_c: float
    rng: np.random.Generator = field(default_factory=lambda: np.random.default_rng(0))

    @classmethod
    def new(cls, thermal: ThermalModel, protocol: ProfilingProtocol) -> "ThermalState":
        return cls(thermal.ambient_c, np.random.default_rng(protocol.seed))


def analytic_kernel_ms(kernel, freq_mhz: float, sm_count: int, gpu, bw_frac: float = 1.0) -> float:
    """Roofline duration used only for candidate pruning (reference simgpu.py:144-168)."""
    if sm_count < 1:
        raise InvalidConfigError("kernel needs at least one SM")
    if not 0 < bw_frac <= 1:
        raise ValueError("bw_frac must be in (0, 1]")
    if kernel.comm_bytes > 0:
        return kernel.comm_bytes / gpu.comm_rate_bps(sm_count) * 1e3
    if kernel.flops == 0 and kernel.bytes == 0:
        return 0.0
    tc = kernel.flops / gpu.flop_rate(sm_count, freq_mhz) if kernel.flops else 0.0
    tm = kernel.bytes / (gpu.mem_bw_bps * bw_frac) if kernel.bytes else 0.0
    return max(tc, tm) * 1e3


def validate_schedule(partition, config, gpu) -> None:
    """The executor's admission check, identical in effect to reference simgpu.py:269-279."""
    t = config.timing
    if t.is_sequential:
        return
    if config.sm_alloc >= gpu.num_sms:
        raise InvalidConfigError(
            f"sm_alloc {config.sm_alloc} must leave SMs for computation (GPU has {gpu.num_sms})")
    n = len(partition.comp_kernels)
    if t.start >= n:
        raise InvalidConfigError(f"overlap start {t.start} out of range for {n} computation kernels")


def span_eff(partition, config) -> int:
    n = len(partition.comp_kernels)
    return min(config.timing.span, n - config.timing.start)


__all__ = ["GpuModel", "b200_model", "b200_model_measured", "ThermalModel", "ProfilingProtocol", "ThermalState", "InvalidConfigError",
           "analytic_kernel_ms", "validate_schedule", "span_eff", "load_measured_peaks", "replace", "math"]
