"""SPMD measurement driver for N-GPU partitions (one process per GPU).

Rank 0 runs the optimizer and calls `SpmdEngine.measure` with the reference `measure` signature
(simgpu.py:321-328).  The command (partition name, schedule, protocol windows) is broadcast over
`torch.distributed`; every rank executes the same schedule at the same time on its own GPU
(`local.measure_local`), and the results are combined as SURVEY.md §8e prescribes:
time = max over ranks, energy = sum over ranks.  With `gpu.p_static_w` set to the group's static
power (sum of per-GPU idle power), `Measurement.build` and the optimizer's static-energy passes
(mbo.py:190-192) stay consistent.  Other ranks sit in `serve()` until rank 0 calls `stop()`.

Every rank must launch the same number of collectives (their per-CTA flag barriers wait for the
peers), so the warm-up / window repetition counts come from one execution-time estimate agreed
across ranks: `SpmdEngine` installs `local.agree_ms` = MAX over ranks, which `Engine._window` applies
before deriving the counts.

Invalid configurations raise `InvalidConfigError` on rank 0 before anything is broadcast.  The
scalar reductions run on the local CUDA device when the group's backend is NCCL (which cannot
reduce CPU tensors) and on the CPU otherwise.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .device import validate_schedule
from .domain import Measurement


def default_reduce_device(group=None, device=None) -> torch.device:
    """CUDA for an NCCL group (NCCL cannot reduce CPU tensors), CPU for gloo."""
    backend = str(dist.get_backend(group)).lower()
    if "nccl" in backend:
        if device is not None and torch.device(device).type == "cuda":
            return torch.device(device)
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


class SpmdEngine:
    def __init__(self, local, gpu, group=None, measurement_cls=Measurement, reduce_device=None):
        self.local = local
        self.gpu = gpu
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.measurement_cls = measurement_cls
        self.reduce_device = reduce_device or default_reduce_device(group, getattr(local, "device", None))
        local.agree_ms = self._max

    def _max(self, v: float) -> float:
        t = torch.tensor([float(v)], dtype=torch.float64, device=self.reduce_device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def _reduce(self, t_ms: float, e_j: float) -> tuple[float, float]:
        v = torch.tensor([t_ms, e_j], dtype=torch.float64, device=self.reduce_device)
        t = v[:1].clone()
        e = v[1:].clone()
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        dist.all_reduce(e, op=dist.ReduceOp.SUM, group=self.group)
        return float(t.item()), float(e.item())

    def _bcast(self, obj):
        box = [obj]
        dist.broadcast_object_list(box, src=0, group=self.group)
        return box[0]

    def _run(self, cmd) -> tuple[float, float]:
        _, name, (f, sm, timing), (warm, win, cool) = cmd
        from .domain import LaunchTiming, ScheduleConfig

        cfg = ScheduleConfig(f, sm, LaunchTiming.decode(timing))
        t_ms, e_j, _ = self.local.measure_local(name, cfg, warm, win, cool)
        return self._reduce(t_ms, e_j)

    def measure(self, partition, config, gpu=None, thermal=None, protocol=None, state=None):
        if self.rank != 0:
            raise RuntimeError("SpmdEngine.measure is called on rank 0; other ranks call serve()")
        gpu = gpu or self.gpu
        validate_schedule(partition, config, gpu)
        if hasattr(self.local, "check_frequency"):
            self.local.check_frequency(config.frequency_mhz, gpu)  # before anything is broadcast
        cmd = ("measure", partition.name, (float(config.frequency_mhz), int(config.sm_alloc), config.timing.encode()),
               (getattr(protocol, "warmup_s", 2.0), getattr(protocol, "window_s", 5.0),
                getattr(protocol, "cooldown_s", 5.0)))
        self._bcast(cmd)
        t_ms, e_j = self._run(cmd)
        return self.measurement_cls.build(t_ms, e_j - gpu.p_static_w * t_ms / 1e3, gpu.p_static_w)

    def serve(self) -> int:
        """Non-zero ranks: execute rank 0's commands until it stops; returns #commands served."""
        n = 0
        while True:
            cmd = self._bcast(None)
            if cmd is None or cmd[0] == "stop":
                return n
            self._run(cmd)
            n += 1

    def stop(self) -> None:
        if self.rank == 0:
            self._bcast(("stop",))
