"""Real 2-rank (non-loopback) collectives on ONE GPU: two processes, CUDA-IPC mapped symmetric
buffers exchanged over gloo, per-CTA cross-rank flag barriers.  Checks bit-exactness against the
numpy oracle and replays a captured CUDA graph to exercise the device-side epochs.
Prints one JSON line; exit code 0 on success.  python tools/ipc_two_rank.py"""
import json
import os
import socket
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, world, port, results):
    import numpy as np
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from oracle import collectives as oc
    from paper_2601_17654_b200.comm import Communicator

    count = 1 << 16  # elements per rank shard (all-gather) / chunk (reduce-scatter)
    c = Communicator.from_process_group(4 * count * world * 2 + (1 << 20), device=torch.device("cuda", 0))
    res = {"rank": rank}
    g = torch.Generator().manual_seed(1234)
    shards = [torch.randn(count, generator=g).to(torch.bfloat16) for _ in range(world)]
    full = [torch.randn(count * world, generator=g).to(torch.bfloat16) for _ in range(world)]
    bits = lambda t: t.cpu().view(torch.int16).numpy().view(np.uint16)
    # all-gather
    ag_src = c.alloc(count * 2)
    ag_src.local().copy_(shards[rank].cuda())
    out = torch.empty(count * world, dtype=torch.bfloat16, device="cuda")
    torch.cuda.synchronize()
    dist.barrier()
    for _ in range(3):
        c.all_gather(ag_src, out, 8)
    torch.cuda.synchronize()
    res["all_gather"] = bool(np.array_equal(bits(out), oc.all_gather([bits(s) for s in shards])))
    # reduce-scatter
    rs_src = c.alloc(count * world * 2)
    rs_src.local().copy_(full[rank].cuda())
    rs_out = torch.empty(count, dtype=torch.bfloat16, device="cuda")
    torch.cuda.synchronize()
    dist.barrier()
    c.reduce_scatter(rs_src, rs_out, 8)
    torch.cuda.synchronize()
    res["reduce_scatter"] = bool(np.array_equal(bits(rs_out), oc.reduce_scatter([bits(x) for x in full], rank)))
    # all-reduce, captured in a CUDA graph and replayed (device-side epochs must keep ranks in step)
    ar_src = c.alloc(count * world * 2)
    stage = c.alloc(count * world * 2)
    ar_src.local().copy_(full[rank].cuda())
    ar_out = torch.empty(count * world, dtype=torch.bfloat16, device="cuda")
    torch.cuda.synchronize()
    dist.barrier()
    c.all_reduce(ar_src, stage, ar_out, 4)  # eager once
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        c.all_reduce(ar_src, stage, ar_out, 4, stream=s)
    torch.cuda.synchronize()
    dist.barrier()
    for _ in range(4):
        ar_out.zero_()
        graph.replay()
    torch.cuda.synchronize()
    res["all_reduce_graph"] = bool(np.array_equal(bits(ar_out), oc.all_reduce([bits(x) for x in full])))
    dist.barrier()
    results[rank] = res
    c.close()
    dist.destroy_process_group()


def main():
    import torch.multiprocessing as mp

    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(worker, args=(2, port, out), nprocs=2, join=True)
    res = {k: dict(v) for k, v in out.items()}
    ok = all(v[t] for v in res.values() for t in ("all_gather", "reduce_scatter", "all_reduce_graph"))
    print(json.dumps({"ok": ok, "ranks": res}))
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
