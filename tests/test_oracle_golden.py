"""Pin the CPU timing-model port (oracle/simgpu_port.py) and the product's analytic pruning model
(device.analytic_kernel_ms) against vectors produced by the UNMODIFIED reference
(tools/make_golden.py -> tests/golden/simgpu_golden.json), plus the reference tests' known answers
(reference pkg/tests/test_simgpu.py)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import simgpu_port as sp
from paper_2601_17654_b200 import (GpuModel, KernelSpec, LaunchTiming, PartitionSpec, ProfilingProtocol,
                                   ScheduleConfig, ThermalModel, analytic_kernel_ms)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "simgpu_golden.json")))
GPU = GpuModel(**GOLD["gpu"])


def _part(d):
    return PartitionSpec(tuple(KernelSpec(n, flops=f, bytes=b) for n, f, b in d["comp"]),
                         KernelSpec(d["comm"][0], comm_bytes=d["comm"][1]), d["comm_group_size"], d["name"])


def _cfg(f, sm, t):
    return ScheduleConfig(f, sm, LaunchTiming.decode(t))


@pytest.mark.parametrize("idx", range(len(GOLD["partitions"])))
def test_simulate_matches_reference_vectors(idx):
    block = GOLD["partitions"][idx]
    p = _part(block["partition"])
    exact = 0
    for f, sm, t, time_ms, dyn, static, total in block["rows"]:
        ms, d = sp.simulate(p, _cfg(f, sm, t), GPU)
        assert ms == pytest.approx(time_ms, rel=1e-12, abs=0)
        assert d == dyn  # dynamic energy is closed form: bit-exact
        st = ms / 1000.0 * GPU.p_static_w
        assert st + d == pytest.approx(total, rel=1e-12)
        exact += ms == time_ms
    assert exact >= 0.99 * len(block["rows"])  # guard only perturbs at the 1e-16 level


def test_kernel_duration_vectors_bit_exact():
    for name, fl, by, cb, f, sm, want in GOLD["kernel_duration"]:
        k = KernelSpec(name, flops=fl, bytes=by, comm_bytes=cb)
        assert sp.roofline_ms(k, f, sm, GPU) == want
        assert analytic_kernel_ms(k, f, sm, GPU) == want


def test_measure_sequence_with_thermal_noise_and_quantum():
    ms = GOLD["measure_sequence"]
    p = _part(ms["partition"])
    thermal = ThermalModel(**ms["thermal"])
    proto = ProfilingProtocol(**ms["protocol"])
    rng = np.random.default_rng(proto.seed)
    temp = thermal.ambient_c
    for f, sm, t, time_ms, dyn, static, total, temp_after in ms["rows"]:
        got = sp.measure(p, _cfg(f, sm, t), GPU, thermal, proto, temp, rng)
        temp = got[4]
        assert got[0] == pytest.approx(time_ms, rel=1e-12)
        assert got[1] == pytest.approx(dyn, rel=1e-10, abs=1e-12)
        assert got[3] == pytest.approx(total, rel=1e-10, abs=1e-12)
        assert temp == pytest.approx(temp_after, rel=1e-12)


# ---- known answers restated from reference pkg/tests/test_simgpu.py
def test_exposed_tail_15ms():
    gpu = GpuModel(overlap_launch_overhead_ms=0.0)
    comp = KernelSpec("gemm", flops=gpu.flop_rate(gpu.num_sms - 8, gpu.f_max_mhz) * 0.010)
    comm = KernelSpec("ar", comm_bytes=gpu.comm_rate_bps(8) * 0.015)
    ms, _ = sp.simulate(PartitionSpec((comp,), comm), ScheduleConfig(gpu.f_max_mhz, 8, LaunchTiming.overlap(0, 1)), gpu)
    assert ms == pytest.approx(15.0, rel=1e-9)


def test_sync_point_12ms():
    gpu = GpuModel(overlap_launch_overhead_ms=0.0)
    c1 = KernelSpec("c", flops=gpu.flop_rate(gpu.num_sms - 4, gpu.f_max_mhz) * 0.001)
    c2 = KernelSpec("c2", flops=gpu.flop_rate(gpu.num_sms, gpu.f_max_mhz) * 0.002)
    comm = KernelSpec("ar", comm_bytes=gpu.comm_rate_bps(4) * 0.010)
    p = PartitionSpec((c1, c2), comm)
    spanned, _ = sp.simulate(p, ScheduleConfig(gpu.f_max_mhz, 4, LaunchTiming.overlap(0, 1)), gpu)
    free, _ = sp.simulate(p, ScheduleConfig(gpu.f_max_mhz, 4, LaunchTiming.overlap(0, 2)), gpu)
    assert spanned == pytest.approx(12.0, rel=1e-9) and free < spanned


def test_hbm_contention_closed_form():
    gpu = GpuModel(overlap_launch_overhead_ms=0.0)
    sm = gpu.sm_bw_saturation
    mem = KernelSpec("norm", bytes=1e9)
    rate = gpu.comm_rate_bps(sm)
    solo = sp.roofline_ms(mem, gpu.f_max_mhz, gpu.num_sms, gpu)
    stretched = solo * (gpu.mem_bw_bps + rate) / gpu.mem_bw_bps
    comm = KernelSpec("ar", comm_bytes=rate * 1.0)
    ms, _ = sp.simulate(PartitionSpec((mem,), comm), ScheduleConfig(gpu.f_max_mhz, sm, LaunchTiming.overlap(0, 1)), gpu)
    moved = rate * (gpu.mem_bw_bps / (gpu.mem_bw_bps + rate)) * stretched / 1e3
    assert ms == pytest.approx(stretched + (comm.comm_bytes - moved) / rate * 1e3, rel=1e-9)


def test_invalid_configs_and_span_clamp():
    p = _part(GOLD["partitions"][0]["partition"])
    with pytest.raises(sp.InvalidConfig):
        sp.simulate(p, ScheduleConfig(1410.0, GPU.num_sms, LaunchTiming.overlap(0, 1)), GPU)
    with pytest.raises(sp.InvalidConfig):
        sp.simulate(p, ScheduleConfig(1410.0, 4, LaunchTiming.overlap(9, 1)), GPU)
    a, _ = sp.simulate(p, ScheduleConfig(1410.0, 8, LaunchTiming.overlap(4, 1)), GPU)
    b, _ = sp.simulate(p, ScheduleConfig(1410.0, 8, LaunchTiming.overlap(4, 5)), GPU)
    assert a == b


def _spinning_case():
    from paper_2601_17654_b200 import b200_model, specs
    from paper_2601_17654_b200.model import baseline_workload
    p = next(x for x in specs.partition_specs(baseline_workload(1)) if x.name == "bwd_mlp0")
    return p, b200_model(), (1965.0, 4, 2, 4)


def test_guard_terminates_where_reference_loop_spins():
    """SURVEY §0 finding 1: at B200-scale parameters the reference event loop can spin forever on a
    ~1e-9-byte comm residual; the port's guard terminates with a finite makespan."""
    p, gpu, (f, sm, s, k) = _spinning_case()
    with pytest.raises(RuntimeError):
        sp.overlap_ms(p, f, sm, s, k, gpu, guard=False, max_steps=5000)
    ms = sp.overlap_ms(p, f, sm, s, k, gpu, guard=True)
    assert 0 < ms < 1e3


def test_reference_itself_hangs_on_that_case(schedfront):
    """Run the unmodified reference in a subprocess with a 20 s budget: it must not finish."""
    p, gpu, (f, sm, s, k) = _spinning_case()
    code = f"""
import sys; sys.path.insert(0, {os.path.join(os.path.dirname(os.path.dirname(__file__)), 'baseline', '_ref')!r})
from schedfront.domain import KernelSpec, PartitionSpec, ScheduleConfig, LaunchTiming
from schedfront.simgpu import GpuModel, simulate_schedule
gpu = GpuModel(**{ {fl.name: getattr(gpu, fl.name) for fl in __import__('dataclasses').fields(gpu)}!r})
p = PartitionSpec(tuple(KernelSpec(*x) for x in {[(kk.name, kk.flops, kk.bytes) for kk in p.comp_kernels]!r}),
                  KernelSpec({p.comm_kernel.name!r}, comm_bytes={p.comm_kernel.comm_bytes!r}), 8, 'x')
simulate_schedule(p, ScheduleConfig({f!r}, {sm!r}, LaunchTiming.overlap({s}, {k})), gpu)
print('finished')
"""
    with pytest.raises(subprocess.TimeoutExpired):
        subprocess.run([sys.executable, "-c", code], timeout=20, capture_output=True)
