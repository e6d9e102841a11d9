"""Executed-schedule parity with REAL cross-rank collectives: two processes share the one GPU of the
box, map each other's symmetric heaps through CUDA IPC (no loopback) and run LayerRunner.step()
under three schedules; every rank's outputs / gradients are checked against the CPU fp32 oracle and
the FSDP collectives bit-exactly against the numpy collective oracle (tests/step_parity.py).

  tp    TP2 of a model sized so each rank holds the Llama-3-8B TP8 per-rank shapes
        (h 4096, 4/1 heads x 128, ffn 1792): the all-reduces of the partial sums are cross-rank.
  fsdp  FSDP2 of a Llama-3.2-3B-width layer (h 3072, 24/8 heads, ffn 8192).

Prints one JSON line; exit code 0 on success.  python tools/ipc_step_parity.py {tp|fsdp} [tokens]"""
import json
import os
import socket
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def worker(rank, world, port, parallel, tokens, results):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import step_parity as sp
    from paper_2601_17654_b200.comm import Communicator
    from paper_2601_17654_b200.device import b200_model
    from paper_2601_17654_b200.engine import Engine
    from paper_2601_17654_b200.layer import PartitionedLayer, sym_bytes_for
    from paper_2601_17654_b200.model import PRESETS, ModelConfig, Workload
    from paper_2601_17654_b200.runner import LayerRunner

    if parallel == "tp":
        m = ModelConfig("llama-3-8b-tp8-rank-x2", hidden=4096, ffn=1792 * world, n_heads=4 * world,
                        n_kv_heads=world, head_dim=128, n_layers=32)
    else:
        m = PRESETS["llama-3.2-3b"]
    wl = Workload(m, parallel, world, tokens)
    dev = torch.device("cuda", 0)
    comm = Communicator.from_process_group(sym_bytes_for(wl), device=dev)
    L = PartitionedLayer(wl, comm)
    gpu = b200_model()
    eng = Engine.for_layer(L, gpu, clock_control=False)
    ref = sp.oracle_for(L)
    slices = (lambda g, k: L.tp_shard({"wqkv": ref["grads"]["wqkv"], "wo": ref["grads"]["wo"],
                                       "wgu": ref["grads"]["wgu"], "wd": ref["grads"]["wd"],
                                       "g1": ref["grads"]["g1"], "g2": ref["grads"]["g2"]}, rank)[k]) \
        if parallel == "tp" else None
    res = {"rank": rank, "schedules": {}}
    ok = True
    k = 0
    for name, sched in sp.schedules(L, gpu).items():
        run = LayerRunner(L, eng, schedule=sched)
        run.k = k
        run.warm()
        dist.barrier()
        sp.poison(L, run.k)
        dist.barrier()
        for _ in range(3):
            run.step()
        torch.cuda.synchronize()
        dist.barrier()  # every rank's step is done before peers' buffers are read
        k = run.k
        errs = sp.check_outputs(L, ref, slices)
        row = {"max_rel": max(errs.values()), "errs": {e: round(v, 5) for e, v in errs.items()}}
        ok &= all(v < sp.TOL for v in errs.values())
        if parallel == "fsdp":
            coll = sp.check_fsdp_collectives_loopback(L)
            row["collectives_bitexact"] = all(coll.values())
            ok &= row["collectives_bitexact"]
        res["schedules"][name] = row
        dist.barrier()
    res["ok"] = bool(ok)
    res["graph_failures"] = len(eng.exec.graph_failures)
    res["gate"] = eng.exec.gate_status
    results[rank] = res
    dist.barrier()
    eng.close()
    comm.close()
    dist.destroy_process_group()


def main():
    import torch.multiprocessing as mp

    parallel = sys.argv[1] if len(sys.argv) > 1 else "tp"
    tokens = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(worker, args=(2, port, parallel, tokens, out), nprocs=2, join=True)
    res = {k: dict(v) for k, v in out.items()}
    ok = all(v["ok"] for v in res.values()) and len(res) == 2
    print(json.dumps({"ok": ok, "parallel": parallel, "tokens": tokens, "ranks": res}))
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
