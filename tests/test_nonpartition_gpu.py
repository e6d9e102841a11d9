"""Non-partition work: embedding, fused cross-entropy, LM head program, and
the measured cost table feeding the reference's microbatch composition.

Tolerances: the cross-entropy loss is fp32 math over bf16 logits (<= 1e-4 abs vs fp32 on the same
bf16 inputs); dlogits are bf16 (<= 1e-2 relative Frobenius); the embedding gather is bit-exact; the
fp32 scatter-add reorders sums of repeated ids (<= 1e-6 relative).
"""
import pytest
import torch

from oracle import nonpart_ref

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = a.float().cpu(), b.float().cpu()
    return ((a - b).norm() / b.norm().clamp_min(1e-12)).item()


@pytest.mark.parametrize("T,V", [(64, 1000), (37, 50304), (8, 128256)])
def test_cross_entropy_matches_oracle(cuda, T, V):
    from paper_2601_17654_b200 import ops
    g = torch.Generator().manual_seed(T + V)
    logits = (torch.randn(T, V, generator=g) * 3).to(torch.bfloat16)
    labels = torch.randint(0, V, (T,), generator=g, dtype=torch.int32)
    labels[1] = -100  # ignored row
    loss_ref, d_ref = nonpart_ref.cross_entropy(logits, labels, grad_scale=0.5)
    lg = logits.to(cuda)
    loss = torch.empty(T, device=cuda)
    dl = torch.empty_like(lg)
    ops.cross_entropy(lg, labels.to(cuda), loss, dl, grad_scale=0.5)
    torch.cuda.synchronize()
    assert (loss.cpu() - loss_ref).abs().max().item() < 1e-4
    assert rel(dl, d_ref) < 1e-2
    assert torch.count_nonzero(dl[1]).item() == 0
    # in place (dlogits aliasing logits) gives the same result
    ops.cross_entropy(lg, labels.to(cuda), loss, lg, grad_scale=0.5)
    torch.cuda.synchronize()
    assert torch.equal(lg, dl)


def test_embedding_fwd_bitexact_and_bwd(cuda):
    from paper_2601_17654_b200 import ops
    V, h, T = 5000, 256, 300
    g = torch.Generator().manual_seed(3)
    table = torch.randn(V, h, generator=g).to(torch.bfloat16)
    ids = torch.randint(0, V, (T,), generator=g, dtype=torch.int32)
    ids[:50] = 7  # repeated token: scatter-add collisions
    out = torch.empty(T, h, dtype=torch.bfloat16, device=cuda)
    bad = torch.zeros(1, dtype=torch.int32, device=cuda)
    ops.embedding_fwd(ids.to(cuda), table.to(cuda), out, bad)
    torch.cuda.synchronize()
    assert torch.equal(out.cpu(), table[ids.long()])
    assert bad.item() == 0
    dy = torch.randn(T, h, generator=g).to(torch.bfloat16)
    dt = torch.zeros(V, h, device=cuda)
    ops.embedding_bwd(ids.to(cuda), dy.to(cuda), dt)
    torch.cuda.synchronize()
    assert rel(dt, nonpart_ref.embedding_bwd(ids, dy, V)) < 1e-6
    ids[5] = V + 3  # out of range: zero row and the flag
    ops.embedding_fwd(ids.to(cuda), table.to(cuda), out, bad)
    torch.cuda.synchronize()
    assert bad.item() == 1 and torch.count_nonzero(out[5]).item() == 0


def test_head_program_matches_oracle(cuda):
    from paper_2601_17654_b200.model import ModelConfig, Workload
    from paper_2601_17654_b200.nonpartition import NonPartitionWork
    m = ModelConfig("tiny", hidden=256, ffn=512, n_heads=4, n_kv_heads=2, head_dim=64, n_layers=1, vocab=4000)
    wl = Workload(m, "fsdp", 2, tokens=128)
    npw = NonPartitionWork(wl, cuda)
    npw.run()
    torch.cuda.synchronize()
    ref = nonpart_ref.head_fwd_bwd(npw.x_last.cpu(), npw.w_lm.cpu(), npw.g_final.cpu(), npw.labels.cpu(),
                                   m.norm_eps, npw.grad_scale)
    assert (npw.loss.cpu() - ref["loss"]).abs().max().item() < 2e-2
    assert rel(npw.dx_last, ref["dx"]) < 3e-2
    assert rel(npw.dw_lm, ref["dw"]) < 3e-2
    assert rel(npw.dtable, nonpart_ref.embedding_bwd(npw.ids.cpu(), npw.dx_first.cpu(), m.vocab)) < 1e-6
    assert torch.equal(npw.emb_out.cpu(), npw.table.cpu()[npw.ids.long().cpu()])


def test_measured_costs_feed_reference_composition(cuda, schedfront):
    """Measured {f: (ms, J)} tables drive the reference's microbatch_frontier unchanged."""
    from schedfront.compose import microbatch_frontier

    from paper_2601_17654_b200 import b200_model
    from paper_2601_17654_b200.device import ProfilingProtocol
    from paper_2601_17654_b200.engine import Engine
    from paper_2601_17654_b200.model import ModelConfig, Workload
    from paper_2601_17654_b200.nonpartition import NonPartitionWork, measure_costs, microbatch_spec
    m = ModelConfig("tiny", hidden=512, ffn=1024, n_heads=8, n_kv_heads=2, head_dim=64, n_layers=1, vocab=8192)
    wl = Workload(m, "fsdp", 2, tokens=256)
    npw = NonPartitionWork(wl, cuda)
    gpu = b200_model()
    eng = Engine(npw.programs, gpu, device=cuda)
    proto = ProfilingProtocol(warmup_s=0.05, window_s=0.2, cooldown_s=0.0)
    costs = measure_costs(eng, npw.programs["np_fwd"], [gpu.f_max_mhz], proto)
    eng.close()
    assert set(costs) == {gpu.f_max_mhz}
    t, e = costs[gpu.f_max_mhz]
    assert t > 0
    spec = microbatch_spec("mb_fwd", ["p"], costs, schedfront.compose.MicrobatchSpec)
    from schedfront.compose import TypeChoice
    from schedfront.domain import LaunchTiming, ScheduleConfig
    cfg = ScheduleConfig(gpu.f_max_mhz, 8, LaunchTiming.sequential())
    per_freq = {"p": {gpu.f_max_mhz: [TypeChoice(1.0, 2.0, cfg)]}}
    front = microbatch_frontier(spec, per_freq, gpu.p_static_w)
    pts = list(front.points)
    assert len(pts) == 1
    assert abs(pts[0].time_ms - (1.0 + t)) < 1e-9 and abs(pts[0].payload.dyn_energy_j - (2.0 + e)) < 1e-9


def test_clock_controller_drives_real_microbatches(cuda):
    """freqctl on hardware: the non-partition programs as 'microbatches' with assigned clocks.  Where
    NVML refuses locked clocks (this pool) the sequence runs at the current clock and no switch is
    recorded; where it permits them every frequency change is one recorded switch."""
    from paper_2601_17654_b200 import b200_model
    from paper_2601_17654_b200.engine import Engine
    from paper_2601_17654_b200.freqctl import MicrobatchClockController
    from paper_2601_17654_b200.model import ModelConfig, Workload
    from paper_2601_17654_b200.nonpartition import NonPartitionWork
    m = ModelConfig("tiny", hidden=512, ffn=1024, n_heads=8, n_kv_heads=2, head_dim=64, n_layers=1, vocab=8192)
    npw = NonPartitionWork(Workload(m, "fsdp", 2, tokens=256), cuda)
    eng = Engine(npw.programs, b200_model(), device=cuda, clock_control=True)
    progs = [npw.programs["np_fwd"], npw.programs["np_bwd"]] * 2
    st = eng.exec.compute

    def enqueue(i):
        for u in progs[i].units:
            u.fn(st)
        ev = torch.cuda.Event()
        ev.record(st)
        return ev

    f0 = eng.gpu.f_max_mhz
    freqs = [f0, f0 - 300.0, f0 - 300.0, f0]
    res = MicrobatchClockController(eng.freq, eng.nvml.sm_clock_mhz).run(freqs, enqueue, "async")
    eng.close()
    if eng.freq.available:
        assert [s.index for s in res.switches] == [0, 1, 3]
    else:
        assert res.switches == [] and res.clock_control.startswith("unavailable")
    assert res.total_s > 0
