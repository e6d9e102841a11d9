"""Boundary value types: behaviour and field-for-field compatibility with the reference."""
import dataclasses
import itertools
import random

import pytest

from paper_2601_17654_b200 import (FrequencyGrid, KernelSpec, LaunchTiming, Measurement, PartitionSpec,
                                   ScheduleConfig, SmGrid, get_frontier)
from paper_2601_17654_b200.domain import FrontierPoint


def test_launch_timing_encode_decode_roundtrip():
    for t in [LaunchTiming.sequential()] + [LaunchTiming.overlap(s, k) for s in range(4) for k in range(1, 5)]:
        assert LaunchTiming.decode(t.encode()) == t
    assert LaunchTiming.overlap(2, 3).encode() == "ov2x3"
    with pytest.raises(ValueError):
        LaunchTiming.decode("bogus")
    with pytest.raises(ValueError):
        LaunchTiming.overlap(0, 0)


def test_schedule_sort_key_orders_like_reference():
    cs = [ScheduleConfig(f, sm, t) for f in (900.0, 1410.0) for sm in (3, 1)
          for t in (LaunchTiming.overlap(1, 1), LaunchTiming.sequential(), LaunchTiming.overlap(0, 2))]
    keys = [c.sort_key() for c in sorted(cs, key=lambda c: c.sort_key())]
    assert keys[0] == (900.0, 1, 0, 0, 0)
    assert keys == sorted(keys)


def test_kernel_kind_and_partition_class():
    assert KernelSpec("a", flops=150.0 * 10, bytes=10).kind == "compute-bound"
    assert KernelSpec("a", flops=149.0 * 10, bytes=10).kind == "memory-bound"
    assert KernelSpec("c", comm_bytes=1).kind == "communication"
    with pytest.raises(ValueError):
        KernelSpec("x", flops=1, comm_bytes=1)
    comm = KernelSpec("c", comm_bytes=1)
    k = KernelSpec("k", flops=1)
    assert PartitionSpec((k,), comm).partition_class == "small"
    assert PartitionSpec((k,) * 3, comm).partition_class == "medium"
    assert PartitionSpec((k,) * 4, comm).partition_class == "large"
    with pytest.raises(ValueError):
        PartitionSpec((comm,), comm)


def test_measurement_build_exact():
    m = Measurement.build(3.25, 1.5, 205.0)
    assert m.static_energy_j == 3.25 / 1000.0 * 205.0
    assert m.total_energy_j == m.dyn_energy_j + m.static_energy_j


def test_frontier_matches_brute_force():
    rng = random.Random(0)
    for trial in range(50):
        pts = [(rng.randint(0, 20) / 2, rng.randint(0, 20) / 2) for _ in range(rng.randint(1, 40))]
        got = [p.objectives for p in get_frontier(pts)]
        want = sorted({p for p in pts if not any(q[0] <= p[0] and q[1] <= p[1] and q != p for q in pts)})
        assert got == want


def test_frontier_tie_break_by_config_sort_key():
    a = ScheduleConfig(1410.0, 8, LaunchTiming.overlap(1, 1))
    b = ScheduleConfig(900.0, 2, LaunchTiming.sequential())
    f = get_frontier([(1.0, 1.0, a), (1.0, 1.0, b)])
    assert len(f) == 1 and f[0].payload is b


def test_grids():
    assert len(FrequencyGrid.default()) == 18
    assert SmGrid.default_for_group(8).values == tuple(range(3, 31, 3))
    g = FrequencyGrid.b200([1965.0 - 7.5 * i for i in range(200)])
    assert g.max == 1965.0 and g.min >= 990.0
    with pytest.raises(ValueError):
        SmGrid((3, 2))


def test_fields_match_reference(schedfront):
    """Same field names and order as the reference dataclasses, so either side's objects can be
    passed to the other (reference domain.py:88-248, simgpu.py:35-141)."""
    from schedfront import domain as rd, simgpu as rs
    import paper_2601_17654_b200 as kpo
    pairs = [(kpo.LaunchTiming, rd.LaunchTiming), (kpo.ScheduleConfig, rd.ScheduleConfig),
             (kpo.KernelSpec, rd.KernelSpec), (kpo.PartitionSpec, rd.PartitionSpec),
             (kpo.Measurement, rd.Measurement), (kpo.FrequencyGrid, rd.FrequencyGrid), (kpo.SmGrid, rd.SmGrid),
             (kpo.GpuModel, rs.GpuModel), (kpo.ThermalModel, rs.ThermalModel),
             (kpo.ProfilingProtocol, rs.ProfilingProtocol)]
    for mine, ref in pairs:
        assert [f.name for f in dataclasses.fields(mine)] == [f.name for f in dataclasses.fields(ref)], mine
    # defaults of the descriptor types are the reference's A100 defaults
    assert dataclasses.asdict(kpo.GpuModel()) == dataclasses.asdict(rs.GpuModel())
    assert issubclass(kpo.InvalidConfigError, ValueError)
