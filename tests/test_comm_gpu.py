"""SM-budgeted P2P collectives in loopback mode: bit-exact against the numpy oracle, exact CTA
budget (one CTA per distinct SM), graph-replay-safe epochs."""
import numpy as np
import pytest
import torch

from oracle import collectives as oc

pytestmark = pytest.mark.gpu
W = 8


def _comm(cuda, nbytes):
    from paper_2601_17654_b200.comm import Communicator
    return Communicator.loopback_group(W, nbytes, device=cuda)


def _rand_bf16(n, seed):
    g = torch.Generator().manual_seed(seed)
    return torch.randn(n, generator=g).to(torch.bfloat16)


def _bits(t):
    return t.cpu().view(torch.int16).numpy().view(np.uint16)


@pytest.fixture(params=["auto", "lsu", "bulk"])
def copy_path(request, monkeypatch):
    """Copy engine of the gather phases: size-based choice, forced 16-byte LSU, forced TMA bulk."""
    if request.param == "lsu":
        monkeypatch.setenv("KPO_COMM_BULK", "0")
    elif request.param == "bulk":
        monkeypatch.setenv("KPO_COMM_BULK", "1")
    else:
        monkeypatch.delenv("KPO_COMM_BULK", raising=False)
    return request.param


@pytest.mark.parametrize("count,ncta", [(8, 1), (4096, 3), (1 << 20, 16), (123456 * 8, 148), (3 << 20, 2)])
def test_all_gather_bitexact(cuda, count, ncta, copy_path):
    c = _comm(cuda, count * 2 + 4096)
    reg = c.alloc(count * 2)
    shards = [_rand_bf16(count, p) for p in range(W)]
    for p in range(W):
        (reg.local() if p == 0 else reg.peer(p)).copy_(shards[p].to(cuda))
    out = torch.empty(W * count, dtype=torch.bfloat16, device=cuda)
    for _ in range(3):  # repeated launches exercise the device-side epoch counters
        out.zero_()
        c.all_gather(reg, out, ncta)
    torch.cuda.synchronize()
    assert np.array_equal(_bits(out), oc.all_gather([_bits(s) for s in shards]))
    c.close()


@pytest.mark.parametrize("count,ncta", [(64, 1), (8192, 5), (1 << 19, 32)])
def test_reduce_scatter_bitexact(cuda, count, ncta):
    n = count * W
    c = _comm(cuda, n * 2 + 4096)
    reg = c.alloc(n * 2)
    ins = [_rand_bf16(n, 100 + p) for p in range(W)]
    for p in range(W):
        (reg.local() if p == 0 else reg.peer(p)).copy_(ins[p].to(cuda))
    out = torch.empty(count, dtype=torch.bfloat16, device=cuda)
    c.reduce_scatter(reg, out, ncta)
    torch.cuda.synchronize()
    assert np.array_equal(_bits(out), oc.reduce_scatter([_bits(x) for x in ins], 0))
    c.close()


@pytest.mark.parametrize("count,ncta", [(W * 8, 1), (W * 4096, 7), (4096 * 3072, 24), (4096 * 3072, 2)])
def test_all_reduce_bitexact(cuda, count, ncta, copy_path):
    c = _comm(cuda, 2 * count * 2 + 8192)
    src = c.alloc(count * 2)
    stage = c.alloc(count * 2)
    ins = [_rand_bf16(count, 200 + p) for p in range(W)]
    for p in range(W):
        (src.local() if p == 0 else src.peer(p)).copy_(ins[p].to(cuda))
    ref = oc.all_reduce([_bits(x) for x in ins])
    chunk = count // W
    # loopback: the virtual peers' phase-1 results (their reduced chunks) are provided by the oracle
    for p in range(1, W):
        st = stage.peer(p)
        st[p * chunk:(p + 1) * chunk].copy_(torch.from_numpy(ref[p * chunk:(p + 1) * chunk].view(np.int16)).view(torch.bfloat16).to(cuda))
    out = torch.empty(count, dtype=torch.bfloat16, device=cuda)
    c.all_reduce(src, stage, out, ncta)
    torch.cuda.synchronize()
    assert np.array_equal(_bits(out), ref)
    assert np.array_equal(_bits(stage.local()[:chunk]), ref[:chunk])  # rank 0's phase-1 chunk
    c.close()


def test_sm_budget_exact(cuda):
    """Every comm CTA runs on its own SM and owns it: ncta distinct SM ids, concurrent with a GEMM."""
    from paper_2601_17654_b200 import ops
    count = 1 << 22
    c = _comm(cuda, count * 2 + 4096)
    reg = c.alloc(count * 2)
    out = torch.empty(W * count, dtype=torch.bfloat16, device=cuda)
    trace = torch.zeros(256 * 4, dtype=torch.int64, device=cuda)
    c.trace(trace, 1)
    side = torch.cuda.Stream(priority=-1)
    x = torch.randn(8192, 4096, device=cuda).bfloat16()
    w = torch.randn(8192, 4096, device=cuda).bfloat16()
    y = torch.empty(8192, 8192, device=cuda, dtype=torch.bfloat16)
    ncta = 20
    with torch.cuda.stream(side):
        c.all_gather(reg, out, ncta, stream=side)
    ops.linear(x, w, y)
    torch.cuda.synchronize()
    t = trace.view(256, 4)[:ncta].cpu()
    assert bool((t[:, 3] == 1).all())
    assert len(set(t[:, 0].tolist())) == ncta
    c.trace(None)
    c.close()
