"""Host-side logic that needs no GPU: partition specs, profiler batching/resume, bench contract."""
import json
import os
import subprocess
import sys

import pytest

from paper_2601_17654_b200 import (LaunchTiming, Measurement, ScheduleConfig, analytic_kernel_ms, b200_model, specs)
from paper_2601_17654_b200.model import PRESETS, Workload, baseline_workload
from paper_2601_17654_b200.profiler import ProfileTable, Profiler

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("idx", [0, 1, 2, 3])
def test_partition_specs_shapes(idx):
    wl = baseline_workload(idx)
    parts = specs.partition_specs(wl)
    assert [p.name for p in parts] == ["fwd_attn0", "fwd_attn1", "fwd_mlp0", "fwd_mlp1", "bwd_mlp0", "bwd_mlp1",
                                       "bwd_attn0", "bwd_attn1"]
    n_fa = 4 if specs.fused_rope(wl) else 5  # head_dim 128: RoPE runs in the QKV GEMM epilogue
    n_fm = 3 if specs.fused_swiglu(wl) else 4  # SwiGLU in the gate|up GEMM epilogue
    n_bm = 5 if specs.fused_swiglu_bwd(wl) else 6  # SwiGLU backward in the down dgrad epilogue
    # the last backward partition also runs the dγ column sums ("norm_grads")
    assert [len(p.comp_kernels) for p in parts] == [n_fa, n_fa, n_fm, n_fm, n_bm, n_bm, n_fa + 2, n_fa + 3]
    assert parts[-1].comp_kernels[-1].name == "norm_grads"
    for p in parts:
        assert p.comm_kernel.is_comm and p.comm_group_size == wl.world
        kinds = {k.name: k.kind for k in p.comp_kernels}
        for name, kind in kinds.items():
            if name.startswith(("linear", "o_", "qkv_", "gu_", "down_", "attention")):
                assert kind == "compute-bound", name
            else:
                assert kind == "memory-bound", name
    # backward GEMM FLOPs = 2x forward GEMM FLOPs per nanobatch
    us = specs.unit_specs(wl)
    fwd = sum(us[k].flops for k in ("linear_qkv", "linear_proj", "linear_up", "linear_down"))
    bwd = sum(us[k].flops for k in us if k.endswith(("_dgrad", "_wgrad")))
    assert bwd == pytest.approx(2 * fwd)


def test_fsdp_comm_bytes_cover_every_weight_once_per_direction():
    wl = baseline_workload(1)
    parts = specs.partition_specs(wl)
    total = sum(p.comm_kernel.comm_bytes for p in parts)
    w = sum(wl.weight_numels().values()) * 2 * (wl.world - 1) / wl.world
    gn = specs.fsdp_numel(wl, "gn") * 2 * (wl.world - 1) / wl.world
    # forward all-gathers once, backward re-gathers once and reduce-scatters once; plus the
    # reduce-scatter of the RMSNorm gradients
    assert total == pytest.approx(3 * w + gn)


def test_tp_shapes_per_rank():
    wl = baseline_workload(2)
    assert (wl.hq, wl.hkv, wl.ffn, wl.qkv_dim) == (4, 1, 1792, 768)
    assert Workload(PRESETS["llama-3-70b"], "tp", 8, 4096).hkv == 1


def test_analytic_pruning_model_on_b200_descriptor():
    gpu = b200_model()
    assert gpu.num_sms == 148 and gpu.f_max_mhz == 1965.0
    part = specs.partition_specs(baseline_workload(1))[2]
    gemm = next(k for k in part.comp_kernels if k.name == "linear_up")
    t = analytic_kernel_ms(gemm, gpu.f_max_mhz, gpu.num_sms, gpu)
    assert t == pytest.approx(gemm.flops / 1640.5e12 * 1e3, rel=1e-9)


class _FakeEngine:
    def __init__(self):
        self.calls = 0
        self.last = None

    def measure(self, part, cfg, gpu, thermal, protocol, state):
        self.calls += 1
        return Measurement.build(1.0 + cfg.sm_alloc / 100.0, 0.5, gpu.p_static_w)


def test_profiler_collects_and_resumes(tmp_path):
    gpu = b200_model()
    part = specs.partition_specs(baseline_workload(1))[0]
    cfgs = [ScheduleConfig(1965.0, sm, LaunchTiming.overlap(0, 5)) for sm in (4, 8, 16)]
    eng = _FakeEngine()
    t = Profiler(eng, gpu, None).collect(part, cfgs[:2])
    assert len(t) == 2 and eng.calls == 2
    t = Profiler(eng, gpu, None).collect(part, cfgs, table=t)  # resume: only the missing config runs
    assert len(t) == 3 and eng.calls == 3
    t.write(str(tmp_path / "t.jsonl"))
    assert ProfileTable.read(str(tmp_path / "t.jsonl")).lookup(cfgs[2]).time_ms == 1.16


def test_bench_reference_arm_contract():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--tokens", "128"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "port" and line["value"] > 0


def test_gate_up_block_layout_roundtrip_and_index_map():
    """ops.interleave_gate_up puts gate block b at rows [256b, 256b+128) and its up block right after —
    the column map gate_col(j) = (j // 128) * 256 + j % 128 (+128 for up) of elementwise.cu / the GEMM
    epilogues; deinterleave inverts it exactly."""
    import torch
    from paper_2601_17654_b200 import ops
    f, h = 512, 3
    w = torch.arange(2 * f * h, dtype=torch.float32).view(2 * f, h)
    wb = ops.interleave_gate_up(w)
    assert torch.equal(ops.deinterleave_gate_up(wb), w)
    for j in (0, 5, 127, 128, 300, f - 1):
        g = (j // 128) * 256 + j % 128
        assert torch.equal(wb[g], w[j]) and torch.equal(wb[g + 128], w[f + j])


def test_bench_reference_cpu_path_reports_per_candidate_costs():
    """bench.py's cpu_baseline.reference_path times the unmodified reference simulator over every
    partition's schedule space; skipped where the reference package is absent."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_2601_17654_b200.model import baseline_workload
    r = bench.reference_cpu_path(baseline_workload(0), with_mbo=False)
    if r is None:
        pytest.skip("reference package not installed (baseline/_ref)")
    assert r["partitions"] == 8 and r["candidates"] > 1000
    assert r["simulate_schedule_us"] > 0 and r["measure_us"] > 0 and r["cores"] == 1


def test_energy_outlier_remeasured_median_of_three():
    """Engine._energy_outlier_check (no GPU): after 5 windows of a program, a window whose average power
    departs from the running median by more than energy_outlier_frac is measured twice more and the
    median-energy window is kept; a consistent window is kept as is."""
    from paper_2601_17654_b200.engine import Engine, Observation

    eng = object.__new__(Engine)
    eng.energy_outlier_frac = 0.10
    eng._power_hist = {"p": [1000.0] * 5}
    eng.agree_ms = None
    queue = [(1.0, 0.99e-3 * 1000), (1.0, 1.01e-3 * 1000)]  # two re-measurements near 1 kW

    def window(prog, config, ncta, warmup_s, window_s):
        t, e = queue.pop(0)
        eng.last = Observation(window_s=1.0)
        return t, e, 1

    eng._window = window
    eng._cooldown = lambda s: 0.0
    # a 560 W outlier (1 ms per execution, 0.56 J) -> re-measured, the median (0.99 J) is kept
    t, e, obs = eng._energy_outlier_check("p", None, None, 8, 0.1, 1.0, 0.0, 1.0, 0.56, Observation())
    assert e == 0.99 and "energy_outlier_remeasured" in obs.flags and obs.energy_trials_j == (0.56, 0.99, 1.01)
    # a consistent window: no re-measurement
    t, e, obs = eng._energy_outlier_check("p", None, None, 8, 0.1, 1.0, 0.0, 1.0, 1.02, Observation())
    assert e == 1.02 and "energy_outlier_remeasured" not in obs.flags and not queue
