"""Engine / executor on the B200: schedule semantics, admission errors, measurements, graphs."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup(cuda):
    from paper_2601_17654_b200.comm import Communicator
    from paper_2601_17654_b200.device import b200_model
    from paper_2601_17654_b200.engine import Engine
    from paper_2601_17654_b200.layer import PartitionedLayer
    from paper_2601_17654_b200.model import ModelConfig, Workload
    m = ModelConfig("mid", hidden=2048, ffn=4096, n_heads=16, n_kv_heads=4, head_dim=128, n_layers=1)
    wl = Workload(m, "fsdp", 8, tokens=1024)
    comm = Communicator.loopback_group(8, 512 << 20, device=cuda)
    L = PartitionedLayer(wl, comm)
    eng = Engine.for_layer(L, b200_model())
    yield L, eng
    eng.close()
    comm.close()


def test_invalid_configs_rejected(setup):
    from paper_2601_17654_b200 import InvalidConfigError, LaunchTiming, ScheduleConfig
    L, eng = setup
    part = L.programs["fwd_attn0"].spec()
    with pytest.raises(InvalidConfigError):
        eng.execute(part, ScheduleConfig(1965.0, 148, LaunchTiming.overlap(0, 1)))
    with pytest.raises(InvalidConfigError):
        eng.execute(part, ScheduleConfig(1965.0, 8, LaunchTiming.overlap(5, 1)))


def test_schedules_do_not_change_results(setup):
    from paper_2601_17654_b200 import LaunchTiming, ScheduleConfig
    L, eng = setup
    prog = L.programs["fwd_mlp0"]
    outs = []
    for cfg in [ScheduleConfig(1965.0, 16, LaunchTiming.sequential()),
                ScheduleConfig(1965.0, 16, LaunchTiming.overlap(0, 4)),
                ScheduleConfig(1965.0, 40, LaunchTiming.overlap(1, 2)),
                ScheduleConfig(1965.0, 4, LaunchTiming.overlap(3, 1))]:
        eng.exec.run(prog, cfg, 16, reps=2)
        torch.cuda.synchronize()
        outs.append((L.nb[0]["y"].clone(), L.w_next["wgu"].clone()))
    for y, w in outs[1:]:
        assert torch.equal(y, outs[0][0])
        assert torch.equal(w, outs[0][1])
    assert torch.equal(outs[0][1], L.w["wgu"])  # the overlapped all-gather delivered the real weights


def test_measure_protocol(setup):
    from paper_2601_17654_b200 import LaunchTiming, ProfilingProtocol, ScheduleConfig, ThermalModel, ThermalState
    L, eng = setup
    part = L.programs["fwd_attn1"].spec()
    proto = ProfilingProtocol(warmup_s=0.1, window_s=0.4, cooldown_s=0.0)
    st = ThermalState.new(ThermalModel(), proto)
    for cfg in [ScheduleConfig(1965.0, 16, LaunchTiming.sequential()),
                ScheduleConfig(1965.0, 16, LaunchTiming.overlap(0, 5))]:
        m = eng.measure(part, cfg, eng.gpu, ThermalModel(), proto, st)
        assert m.time_ms > 0
        assert m.total_energy_j == m.dyn_energy_j + m.static_energy_j
        assert m.total_energy_j > 0
        assert eng.last.reps >= 1
    assert st.temperature_c > 0
    assert len(eng.exec.graphs) >= 1, eng.exec.graph_failures


def test_all_partitions_run_under_overlap(setup):
    from paper_2601_17654_b200 import LaunchTiming, ScheduleConfig
    L, eng = setup
    for name in L.order:
        prog = L.programs[name]
        n = len(prog.units)
        ms = eng.exec.time_ms(prog, ScheduleConfig(1965.0, 16, LaunchTiming.overlap(0, n)), 16, reps=3)
        assert ms > 0
    torch.cuda.synchronize()
