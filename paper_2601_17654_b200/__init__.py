"""paper_2601_17654_b200 ("kpo") — B200-native partitioned-overlap execution engine for Kareus
(arXiv 2601.17654), a drop-in for the reference `schedfront` hot path
(`simgpu.simulate_schedule` / `simgpu.measure`).

Host side: Python + PyTorch (memory, streams, torch.distributed plumbing).
Device side: hand-written sm_100a kernels in libkpo.so behind the C ABI of include/kpo.h.
There is no CPU fallback on the product path; `oracle/` (repo root) is test infrastructure only.
"""

from .domain import (FrequencyGrid, FrontierPoint, KernelSpec, LaunchTiming, Measurement, PartitionSpec,
                     ScheduleConfig, SmGrid, get_frontier)
from .device import (GpuModel, InvalidConfigError, ProfilingProtocol, ThermalModel, ThermalState, analytic_kernel_ms,
                     b200_model, validate_schedule)
from .model import PRESETS, ModelConfig, Workload, baseline_workload

__all__ = [
    "FrequencyGrid", "FrontierPoint", "KernelSpec", "LaunchTiming", "Measurement", "PartitionSpec", "ScheduleConfig",
    "SmGrid", "get_frontier", "GpuModel", "InvalidConfigError", "ProfilingProtocol", "ThermalModel", "ThermalState",
    "analytic_kernel_ms", "b200_model", "validate_schedule", "PRESETS", "ModelConfig", "Workload",
    "baseline_workload",
]
__version__ = "0.1.0"
