"""N > 1 host logic on CPU: world_size-2 `gloo` process groups on 127.0.0.1.

Covers the multi-GPU control plane that cannot run on the single-GPU box: IPC-handle exchange for
the symmetric buffers, and the SPMD measurement protocol (rank 0 drives, all ranks execute in
lockstep, time = max over ranks, energy = sum over ranks, invalid configs rejected on rank 0
before anything is broadcast)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class FakeLocal:
    """Stands in for Engine.measure_local on a CPU-only host."""

    def __init__(self, rank):
        self.rank = rank
        self.calls = []
        self.reps = []

    def measure_local(self, name, cfg, warm, win, cool):
        from paper_2601_17654_b200.engine import rep_counts
        self.calls.append((name, cfg.sm_alloc, cfg.timing.encode(), warm, win, cool))
        # as Engine._window: each rank's own estimate differs; the agreed one sets the counts
        est = 0.37 + 0.011 * self.rank
        if getattr(self, "agree_ms", None) is not None:
            est = self.agree_ms(est)
        self.reps.append(rep_counts(est, warm, win))
        return 1.0 + self.rank, 10.0 * (self.rank + 1), 40.0


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2601_17654_b200 import (GpuModel, InvalidConfigError, KernelSpec, LaunchTiming, PartitionSpec,
                                       ProfilingProtocol, ScheduleConfig)
    from paper_2601_17654_b200.comm import exchange_blobs
    from paper_2601_17654_b200.spmd import SpmdEngine
    res = {}
    blobs = exchange_blobs(bytes([rank]) * 64)
    res["blobs"] = [b[0] for b in blobs]
    local = FakeLocal(rank)
    gpu = GpuModel(num_sms=148, sm_bw_saturation=16, p_static_w=100.0 * world)
    eng = SpmdEngine(local, gpu)
    part = PartitionSpec((KernelSpec("k", flops=1e9),) * 3, KernelSpec("ar", comm_bytes=1e6), world, "p0")
    proto = ProfilingProtocol(0.1, 0.5, 0.0)
    if rank == 0:
        m = eng.measure(part, ScheduleConfig(1965.0, 8, LaunchTiming.overlap(1, 2)), gpu, None, proto, None)
        res["m"] = (m.time_ms, m.dyn_energy_j, m.static_energy_j, m.total_energy_j)
        try:
            eng.measure(part, ScheduleConfig(1965.0, 148, LaunchTiming.overlap(0, 1)), gpu, None, proto, None)
        except InvalidConfigError:
            res["invalid_raised"] = True
        m2 = eng.measure(part, ScheduleConfig(1500.0, 16, LaunchTiming.sequential()), gpu, None, proto, None)
        res["m2"] = m2.time_ms
        eng.stop()
    else:
        res["served"] = eng.serve()
    res["calls"] = local.calls
    res["reps"] = local.reps
    out[rank] = res
    dist.destroy_process_group()


def test_spmd_protocol_world2():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    r0, r1 = out[0], out[1]
    assert r0["blobs"] == [0, 1] and r1["blobs"] == [0, 1]
    t, dyn, static, total = r0["m"]
    assert t == 2.0                                  # max over ranks
    assert total == pytest.approx(30.0)              # sum over ranks (10 + 20 J per execution)
    assert static == 2.0 / 1000.0 * 200.0 and total == dyn + static
    assert r0.get("invalid_raised")
    assert r1["served"] == 2                         # the invalid config never reached rank 1
    assert r0["calls"] == r1["calls"] == [("p0", 8, "ov1x2", 0.1, 0.5, 0.0), ("p0", 16, "seq", 0.1, 0.5, 0.0)]
    assert r0["m2"] == 2.0
    # every rank launches the same number of executions (collectives) per window
    assert r0["reps"] == r1["reps"] and len(r0["reps"]) == 2
    from paper_2601_17654_b200.engine import rep_counts
    assert r0["reps"][0] == rep_counts(0.381, 0.1, 0.5) != rep_counts(0.37, 0.1, 0.5)
