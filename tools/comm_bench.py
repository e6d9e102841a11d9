"""Collective microbench (BASELINE.json configs[4]): the engine's SM-budgeted P2P all-gather /
reduce-scatter / all-reduce bus bandwidth vs CTA budget and message size, next to NCCL.

Modes
  single process (default)   loopback group of --world virtual ranks on cuda:0: the peers' buffers
                             live in local HBM, so "bus" bytes move through HBM (a one-GPU box).
  torchrun, one GPU per rank  real ranks: CUDA-IPC peer mapping, the kernels load / store peer HBM
                             over NVLink; device time is the max over ranks.  With the NCCL backend
                             the same sizes are timed through torch.distributed (all_gather_into_tensor,
                             reduce_scatter_tensor, all_reduce) as the default-collective baseline
                             (SURVEY §5).  KPO_SAME_DEVICE=1 runs every rank on cuda:0 over gloo (a
                             functional check of this path on a one-GPU box; no NCCL column, timings
                             meaningless under context time-slicing).
  bus bytes: (W-1)/W * S for all-gather / reduce-scatter, 2(W-1)/W * S for all-reduce (S = the full
  tensor).  Against 900 GB/s per direction per GPU on NVLink 5 (public spec).

NVLink counters for one configuration (one GPU's view; ncu on a single rank of a multi-rank run is
not possible here, so profile rank 0 with the others running un-profiled):
  ncu --metrics nvltx__bytes.sum,nvlrx__bytes.sum,gpu__time_duration.sum -k regex:all_gather_kernel \\
      --clock-control none -c 5 python tools/comm_bench.py ...   (under torchrun, rank 0 only:
      `ncu --target-processes all` is NOT used; wrap rank 0's command)

python tools/comm_bench.py [--world 8] [--sizes-mb 1,16,128,512] [--ctas 1,2,4,8,16,32,64] [--check]
torchrun --nproc-per-node 8 --master-addr 127.0.0.1 tools/comm_bench.py --sizes-mb 1,16,128,1024
Prints one JSON line (rank 0)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=8, help="loopback group size (single process)")
    ap.add_argument("--sizes-mb", default="1,16,128,512")
    ap.add_argument("--ctas", default="1,2,4,8,16,32,64")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--check", action="store_true", help="verify every result bit-exactly (numpy oracle)")
    ap.add_argument("--out", default="")
    a = ap.parse_args()

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2601_17654_b200.comm import Communicator

    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    multi = world_env > 1
    same_dev = os.environ.get("KPO_SAME_DEVICE") == "1"
    local = 0 if same_dev else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if multi:
        dist.init_process_group("gloo" if same_dev else "nccl", **({} if same_dev else {"device_id": dev}))
        W, rank = dist.get_world_size(), dist.get_rank()
    else:
        W, rank = a.world, 0
    nccl = multi and not same_dev
    sizes = [int(float(x) * (1 << 20)) for x in a.sizes_mb.split(",")]
    ctas = [int(x) for x in a.ctas.split(",")]
    rows = []

    def tmax(v):
        if not multi:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cpu" if same_dev else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t)

    def timed(fn, st):
        fn()
        if multi:
            torch.cuda.synchronize(dev)
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(a.reps):
            fn()
        e1.record(st)
        e1.synchronize()
        return tmax(e0.elapsed_time(e1) / a.reps)

    bits = lambda t: t.contiguous().cpu().view(torch.int16).numpy().view(np.uint16).reshape(-1)
    st = torch.cuda.Stream(dev)
    for total in sizes:  # total = full (gathered / reduced) tensor bytes
        total = total // (16 * W) * 16 * W
        count = total // 2
        sym = 2 * total + total // W + (4 << 20)
        c = (Communicator.from_process_group(sym, device=dev) if multi
             else Communicator.loopback_group(W, sym, device=dev))
        src = c.alloc(total)
        stage = c.alloc(total)
        shard = c.alloc(total // W)
        g = torch.Generator(device=dev).manual_seed(17 + rank)
        src.local().copy_(torch.randn(count, generator=g, device=dev).bfloat16())
        shard.local().copy_(torch.randn(count // W, generator=g, device=dev).bfloat16())
        if not multi:
            for p in range(1, W):
                src.peer(p).normal_()
                shard.peer(p).normal_()
        torch.cuda.synchronize(dev)
        if multi:
            dist.barrier()
        out_ag = torch.empty(count, dtype=torch.bfloat16, device=dev)
        out_rs = torch.empty(count // W, dtype=torch.bfloat16, device=dev)
        out_ar = torch.empty(count, dtype=torch.bfloat16, device=dev)
        ops = {
            "all_gather": (lambda n: c.all_gather(shard, out_ag, n, stream=st), (W - 1) / W * total),
            "reduce_scatter": (lambda n: c.reduce_scatter(src, out_rs, n, stream=st), (W - 1) / W * total),
            "all_reduce": (lambda n: c.all_reduce(src, stage, out_ar, n, stream=st), 2 * (W - 1) / W * total),
        }
        for name, (fn, bus) in ops.items():
            for n in ctas:
                if n > c.max_ctas:
                    continue
                ms = timed(lambda: fn(n), st)
                row = {"op": name, "bytes": total, "ncta": n, "ms": round(ms, 5),
                       "busbw_gbs": round(bus / (ms / 1e3) / 1e9, 1), "impl": "kpo-p2p"}
                if a.check:
                    torch.cuda.synchronize(dev)
                    row["bitexact"] = check(name, c, src, shard, out_ag, out_rs, out_ar, W, rank, multi, bits)
                rows.append(row)
            if nccl:
                ref_in = src.local()
                with torch.cuda.stream(st):
                    if name == "all_gather":
                        fn_n = lambda: dist.all_gather_into_tensor(out_ag, shard.local())
                    elif name == "reduce_scatter":
                        fn_n = lambda: dist.reduce_scatter_tensor(out_rs, ref_in)
                    else:
                        buf = ref_in.clone()
                        fn_n = lambda: dist.all_reduce(buf)
                    ms = timed(fn_n, st)
                rows.append({"op": name, "bytes": total, "ncta": None, "ms": round(ms, 5),
                             "busbw_gbs": round(bus / (ms / 1e3) / 1e9, 1), "impl": "nccl"})
        c.close()
    res = {"mode": ("cuda-ipc p2p (NVLink)" if nccl else "cuda-ipc p2p, same device (gloo)") if multi
           else "loopback (HBM)", "world": W, "nccl_baseline": nccl, "rows": rows}
    if rank == 0:
        line = json.dumps(res)
        print(line)
        if a.out:
            open(a.out, "w").write(line + "\n")
    if multi:
        dist.barrier()
        dist.destroy_process_group()


def check(name, c, src, shard, out_ag, out_rs, out_ar, W, rank, multi, bits):
    """Bit-exact check against the numpy collective oracle (reads every rank's input through the
    peer mapping; single process: the loopback peers)."""
    import numpy as np

    from oracle import collectives as oc

    if name == "all_gather":
        ins = [bits(shard.local()) if p == rank else bits(shard.peer(p)) for p in range(W)]
        return bool(np.array_equal(bits(out_ag), oc.all_gather(ins)))
    ins = [bits(src.local()) if p == rank else bits(src.peer(p)) for p in range(W)]
    if name == "reduce_scatter":
        return bool(np.array_equal(bits(out_rs), oc.reduce_scatter(ins, rank)))
    if multi:  # all-reduce inputs are read in place by every rank: identical on all
        return bool(np.array_equal(bits(out_ar), oc.all_reduce(ins)))
    return bool(np.array_equal(bits(out_ar)[rank * (out_ar.numel() // W):(rank + 1) * (out_ar.numel() // W)],
                               oc.all_reduce(ins)[rank * (out_ar.numel() // W):(rank + 1) * (out_ar.numel() // W)]))


if __name__ == "__main__":
    main()
