"""Parity of the executed partition schedules at BASELINE layer widths (north_star check 1).

`LayerRunner.step()` — the call bench.py times: every partition's CUDA graph replayed with the
collective on `sm_alloc` SMs of a side stream, the launch gate and the sync point — runs under the
default nanobatching schedule and two non-default ones (`ov1x2@8`, `seq`), three iterations each
after NaN-poisoning every produced buffer (tests/step_parity.py).  Then this rank's y, h, dx, all
weight gradients and both RMSNorm γ gradients must match the CPU fp32 oracle (oracle/layer_ref.py,
rel. Frobenius <= 3e-2), and the FSDP collectives must be bit-exact: the all-gathers delivered the
full weights the NEXT iteration computes with, and the reduce-scatters reduced the PREVIOUS
iteration's real gradients (plus the virtual peers' fixed gradients) exactly as the numpy
collective oracle does.

Widths (tokens per nanobatch reduced where the CPU oracle would take minutes; 2 nanobatches):
  config 1  Llama-3.2-3B  FSDP8 loopback: h 3072, ffn 8192, 24/8 heads x 128   (T 1024, and T 4096)
  config 2  Llama-3-8B    TP8 per-rank shapes: h 4096, ffn 1792, 4/1 heads x 128 (world-1 layer of
            those shapes here; the real cross-rank all-reduce inside the step is
            test_ipc_step_parity below, two processes on one GPU)
  config 3  Llama-3-70B   FSDP8 loopback: h 8192, ffn 28672, 64/8 heads x 128  (T 512)
"""
import json
import os
import subprocess
import sys

import pytest
import torch

import step_parity as sp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _wl(case):
    from paper_2601_17654_b200.model import PRESETS, ModelConfig, Workload
    if case == "cfg1_T1024":
        return Workload(PRESETS["llama-3.2-3b"], "fsdp", 8, 1024)
    if case == "cfg1_T4096":
        return Workload(PRESETS["llama-3.2-3b"], "fsdp", 8, 4096)
    if case == "cfg2_tp8_rank":
        m = ModelConfig("llama-3-8b-tp8-rank", hidden=4096, ffn=1792, n_heads=4, n_kv_heads=1, head_dim=128,
                        n_layers=32)
        return Workload(m, "tp", 1, 1024)
    if case == "cfg3_T512":
        return Workload(PRESETS["llama-3-70b"], "fsdp", 8, 512)
    raise KeyError(case)


def _run_case(cuda, case, sched_names):
    from paper_2601_17654_b200.comm import Communicator
    from paper_2601_17654_b200.device import b200_model
    from paper_2601_17654_b200.engine import Engine
    from paper_2601_17654_b200.layer import PartitionedLayer, sym_bytes_for
    from paper_2601_17654_b200.runner import LayerRunner

    wl = _wl(case)
    comm = Communicator.loopback_group(wl.world, sym_bytes_for(wl), device=cuda)
    L = PartitionedLayer(wl, comm)
    gpu = b200_model()
    eng = Engine.for_layer(L, gpu, clock_control=False)
    ref = sp.oracle_for(L)
    scheds = sp.schedules(L, gpu)
    k = 0
    report = {}
    try:
        for name in sched_names:
            run = LayerRunner(L, eng, schedule=scheds[name])
            run.k = k
            run.warm()
            sp.poison(L, run.k)
            for _ in range(3):
                run.step()
            torch.cuda.synchronize()
            k = run.k
            errs = sp.check_outputs(L, ref)
            bad = {e: v for e, v in errs.items() if not v < sp.TOL}
            report[name] = errs
            assert not bad, f"{case} {name}: {bad}"
            if wl.parallel == "fsdp":
                coll = sp.check_fsdp_collectives_loopback(L)
                assert all(coll.values()), f"{case} {name}: {coll}"
                prev = sp.previous_grads_rel(L, ref)
                assert all(v < sp.TOL for v in prev.values()), f"{case} {name}: {prev}"
            assert eng.exec.graph_failures == {}, eng.exec.graph_failures
    finally:
        eng.close()
        comm.close()
        del L
        torch.cuda.empty_cache()
    print(case, json.dumps({s: {k: round(v, 5) for k, v in e.items()} for s, e in report.items()}))


@pytest.mark.parametrize("case", ["cfg1_T1024", "cfg2_tp8_rank", "cfg3_T512"])
def test_step_matches_oracle_under_schedules(cuda, case):
    _run_case(cuda, case, ["default", "ov1x2@8", "seq"])


def test_step_matches_oracle_cfg1_full_tokens(cuda):
    """Config 1 at its full 4096 tokens per nanobatch, the bench's own shape, default schedule."""
    _run_case(cuda, "cfg1_T4096", ["default"])


@pytest.mark.parametrize("parallel", ["tp", "fsdp"])
def test_ipc_step_parity(cuda, parallel):
    """Two processes on one GPU, CUDA-IPC peer mapping (no loopback): the TP all-reduces / FSDP
    all-gathers and reduce-scatters inside LayerRunner.step() are the real cross-rank ones.  TP at
    the TP8 per-rank shapes (the model is sized so that 2 ranks hold 4/1 heads and ffn 1792 each)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ipc_step_parity.py"), parallel],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-4000:])
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["ok"], line
