"""Check 2 of north_star: given the same profile table, the optimizer's selected Pareto schedule set
is bit-exact with the reference's.

Fixture: BASELINE config-1 partitions (GPT layer, h 1024, T 2048) projected to
KernelSpecs, reference GpuModel defaults, FrequencyGrid.default() x SmGrid.default_for_group(8);
a profile table made by the reference `measure` (default thermal model, noise 0.02, counter quantum
6 J, seed 1234) over the full space in space order.
  reference side: run_mbo with `measure` monkeypatched to a dict lookup of that table;
  engine side:    the table written through profiler.ProfileTable (JSON lines), read back, and
                  installed with compat.patch_reference; run_mbo driven with OUR PartitionSpec and
                  GpuModel objects.
Records (config, measurement, batch, pass), frontier points and HV history must be identical.
"""
import pytest

from paper_2601_17654_b200 import GpuModel, specs
from paper_2601_17654_b200.compat import patch_reference
from paper_2601_17654_b200.model import baseline_workload
from paper_2601_17654_b200.profiler import ProfileTable


def _to_ref(sf, p):
    d = sf.domain
    return d.PartitionSpec(tuple(d.KernelSpec(k.name, k.flops, k.bytes, k.comm_bytes) for k in p.comp_kernels),
                           d.KernelSpec(p.comm_kernel.name, comm_bytes=p.comm_kernel.comm_bytes), p.comm_group_size,
                           p.name)


def _run(sf, part, gpu, measure):
    from schedfront import mbo, workloads
    restore = patch_reference(measure=measure, schedfront_module=sf)
    try:
        proto = sf.simgpu.ProfilingProtocol(2.0, 5.0, 5.0, 0.02, 6.0, 1234)
        return mbo.run_mbo(part, gpu, workloads.default_thermal(), proto, mbo.MboHyperparams.for_partition(part, 0),
                           sf.domain.FrequencyGrid.default(), sf.domain.SmGrid.default_for_group(8))
    finally:
        restore()


@pytest.mark.parametrize("pname", ["fwd_attn0", "fwd_mlp0"])
def test_table_replay_bitexact(schedfront, tmp_path, pname):
    sf = schedfront
    import schedfront.mbo as mbo
    import schedfront.simgpu as simgpu
    import schedfront.workloads as workloads
    mine = next(p for p in specs.partition_specs(baseline_workload(0)) if p.name == pname)
    ref_part = _to_ref(sf, mine)
    ref_gpu = workloads.default_gpu()
    space = mbo.enumerate_space(ref_part, ref_gpu, sf.domain.FrequencyGrid.default(),
                                sf.domain.SmGrid.default_for_group(8))
    thermal = workloads.default_thermal()
    proto = simgpu.ProfilingProtocol(2.0, 5.0, 5.0, 0.02, 6.0, 1234)
    state = simgpu.ThermalState.new(thermal, proto)
    lookup, table = {}, ProfileTable(pname, {"note": "reference measure over the full space in space order"})
    for c in space:
        m = simgpu.measure(ref_part, c, ref_gpu, thermal, proto, state)
        lookup[c] = m
        table.add(c, m)
    path = tmp_path / f"{pname}.jsonl"
    table.write(str(path))
    back = ProfileTable.read(str(path))
    assert len(back) == len(space)

    r_ref = _run(sf, ref_part, ref_gpu, lambda part, c, *a: lookup[c])
    r_kpo = _run(sf, mine, GpuModel(), back.evaluator(sf.domain.Measurement))

    assert len(r_ref.records) == len(r_kpo.records) > 0
    for a, b in zip(r_ref.records, r_kpo.records):
        assert (a.config, a.measurement, a.batch, a.pass_label) == (b.config, b.measurement, b.batch, b.pass_label)
    assert [(p.time_ms, p.energy_j, p.payload) for p in r_ref.frontier] == \
           [(p.time_ms, p.energy_j, p.payload) for p in r_kpo.frontier]
    assert r_ref.hv_history == r_kpo.hv_history
    assert r_ref.rel_improvements == r_kpo.rel_improvements
    assert len(r_ref.frontier) >= 3


def test_profile_table_roundtrip_exact(tmp_path):
    from paper_2601_17654_b200 import LaunchTiming, Measurement, ScheduleConfig
    t = ProfileTable("p", {"gpu": {"num_sms": 148}})
    vals = [0.1 + 0.2, 1 / 3, 2.0 ** -40, 123456.789e-7]
    for i, v in enumerate(vals):
        t.add(ScheduleConfig(1965.0, 4 + i, LaunchTiming.overlap(i, 1)), Measurement.build(v, v / 7, 205.0),
              {"sm_mhz": 1965.0})
    t.write(str(tmp_path / "t.jsonl"))
    u = ProfileTable.read(str(tmp_path / "t.jsonl"))
    ev = u.evaluator()
    for i, v in enumerate(vals):
        m = ev(None, ScheduleConfig(1965.0, 4 + i, LaunchTiming.overlap(i, 1)))
        assert m == Measurement.build(v, v / 7, 205.0)
    with pytest.raises(ValueError):
        u.add(ScheduleConfig(1965.0, 4, LaunchTiming.overlap(0, 1)), Measurement.build(1, 1, 1))
