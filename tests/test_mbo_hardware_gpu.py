"""The drop-in end to end: the UNMODIFIED reference optimizer (baseline/_ref) drives real B200
executions through Engine.measure (installed over schedfront.mbo.measure), and the measured profile
table replays bit-exactly."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_reference_run_mbo_on_hardware(cuda, schedfront, tmp_path):
    from schedfront import mbo
    from schedfront.domain import FrequencyGrid, SmGrid
    from schedfront.simgpu import ProfilingProtocol, ThermalModel

    from paper_2601_17654_b200 import b200_model
    from paper_2601_17654_b200.comm import Communicator
    from paper_2601_17654_b200.compat import patch_reference
    from paper_2601_17654_b200.engine import Engine, install
    from paper_2601_17654_b200.layer import PartitionedLayer
    from paper_2601_17654_b200.model import ModelConfig, Workload
    from paper_2601_17654_b200.profiler import ProfileTable

    m = ModelConfig("mbo", hidden=2048, ffn=5632, n_heads=16, n_kv_heads=4, head_dim=128, n_layers=1)
    wl = Workload(m, "fsdp", 8, tokens=2048)
    comm = Communicator.loopback_group(8, 512 << 20, device=cuda)
    layer = PartitionedLayer(wl, comm)
    gpu = b200_model()
    eng = Engine.for_layer(layer, gpu)
    restore = install(eng, schedfront)
    part = layer.programs["fwd_mlp0"].spec()
    seen = []
    orig = eng.measure

    def recording(partition, config, *a):
        res = orig(partition, config, *a)
        seen.append((config, res))
        return res

    mbo.measure = recording
    try:
        hyper = mbo.MboHyperparams(n_init=6, b_max=2, batch_k=4, seed=0)
        proto = ProfilingProtocol(warmup_s=0.02, window_s=0.1, cooldown_s=0.0)
        res = mbo.run_mbo(part, gpu, ThermalModel(), proto, hyper, FrequencyGrid((1965.0,)), SmGrid((4, 8, 16, 32)))
    finally:
        restore()
    assert len(res.records) >= 6 and len(res.frontier) >= 1
    assert all(r.measurement.time_ms > 0 for r in res.records)
    assert type(res.records[0].measurement).__module__.startswith("schedfront")
    # the measured table replays bit-exactly through the reference optimizer
    table = ProfileTable(part.name)
    for cfg, meas in seen:
        table.add(cfg, meas)
    path = tmp_path / "t.jsonl"
    table.write(str(path))
    ev = ProfileTable.read(str(path)).evaluator(schedfront.domain.Measurement)
    r2 = patch_reference(measure=lambda p, c, *a: ev(p, c), schedfront_module=schedfront)
    try:
        res2 = mbo.run_mbo(part, gpu, ThermalModel(), proto, hyper, FrequencyGrid((1965.0,)), SmGrid((4, 8, 16, 32)))
    finally:
        r2()
    assert [(r.config, r.measurement) for r in res.records] == [(r.config, r.measurement) for r in res2.records]
    eng.close()
    comm.close()
