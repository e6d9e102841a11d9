"""The N > 1 data path on real hardware: two processes, CUDA-IPC peer mapping, cross-rank per-CTA
flag barriers and graph-replayed epochs (tools/ipc_two_rank.py), on the single GPU of the box."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_two_rank_ipc_collectives_bitexact(cuda):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ipc_two_rank.py")], capture_output=True,
                       text=True, timeout=240)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-3000:])
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["ok"], line


def test_bench_two_ranks_same_device(cuda, tmp_path):
    """bench.py's N > 1 branch under torchrun (2 ranks, both on cuda:0, gloo plumbing): IPC peer
    mapping, SPMD timing with max-over-ranks, one JSON line from rank 0."""
    env = dict(os.environ, KPO_SAME_DEVICE="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29541", os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--steps", "2", "--warmup", "3", "--tokens", "512", "--no-sweep", "--no-cpu"],
                       capture_output=True, text=True, timeout=400, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["config"]["parallelism"] == "fsdp2" and line["value"] > 0
    assert line["comm"]["mode"].startswith("cuda-ipc")


def test_comm_bench_two_ranks_same_device(cuda):
    """tools/comm_bench.py's torchrun path (2 ranks, CUDA-IPC, cross-rank flag barriers), results
    checked bit-exactly against the numpy collective oracle through the peer mappings."""
    env = dict(os.environ, KPO_SAME_DEVICE="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29543",
                        os.path.join(ROOT, "tools", "comm_bench.py"), "--sizes-mb", "1,4", "--ctas", "1,4,16",
                        "--reps", "2", "--check"], capture_output=True, text=True, timeout=400, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["world"] == 2 and line["mode"].startswith("cuda-ipc")
    assert len(line["rows"]) == 2 * 3 * 3 and all(row["bitexact"] for row in line["rows"])
