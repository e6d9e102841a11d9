"""Collective microbench (BASELINE.json configs[4]): SM-budgeted all-gather / reduce-scatter /
all-reduce bus bandwidth vs CTA budget and message size.  On a single-GPU box the group runs in
loopback (virtual peers' buffers in local HBM, so 'bus' bytes move through HBM); under torchrun
with one GPU per rank it measures NVLink.  Device-timed with CUDA events on the launching stream.

python tools/comm_bench.py [--world 8] [--sizes-mb 1,16,256] [--ctas 1,2,4,8,16,32]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2601_17654_b200.comm import Communicator

ap = argparse.ArgumentParser()
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--sizes-mb", default="1,16,128,512")
ap.add_argument("--ctas", default="1,2,4,8,16,32,64")
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
W = a.world
dev = torch.device("cuda", 0)
sizes = [int(float(x) * (1 << 20)) for x in a.sizes_mb.split(",")]
ctas = [int(x) for x in a.ctas.split(",")]
rows = []
for total in sizes:  # total = full (gathered / reduced) tensor bytes
    total = total // (16 * W) * 16 * W
    count = total // 2
    c = Communicator.loopback_group(W, 2 * total + total // W + (4 << 20), device=dev)
    src = c.alloc(total)
    stage = c.alloc(total)
    for p in range(W):
        (src.local() if p == 0 else src.peer(p)).normal_()
    out_ag = torch.empty(total // 2, dtype=torch.bfloat16, device=dev)
    out_rs = torch.empty(count // W, dtype=torch.bfloat16, device=dev)
    out_ar = torch.empty(count, dtype=torch.bfloat16, device=dev)
    shard = c.alloc(total // W)
    st = torch.cuda.Stream(dev)
    ops = {
        # bus bytes: (W-1)/W * total for all-gather / reduce-scatter, 2(W-1)/W * total for all-reduce
        "all_gather": (lambda n: c.all_gather(shard, out_ag, n, stream=st), (W - 1) / W * total),
        "reduce_scatter": (lambda n: c.reduce_scatter(src, out_rs, n, stream=st), (W - 1) / W * total),
        "all_reduce": (lambda n: c.all_reduce(src, stage, out_ar, n, stream=st), 2 * (W - 1) / W * total),
    }
    for name, (fn, bus) in ops.items():
        for n in ctas:
            fn(n)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(a.reps):
                fn(n)
            e1.record(st)
            e1.synchronize()
            ms = e0.elapsed_time(e1) / a.reps
            rows.append({"op": name, "bytes": total, "ncta": n, "ms": round(ms, 4),
                         "busbw_gbs": round(bus / (ms / 1e3) / 1e9, 1)})
    c.close()
print(json.dumps({"mode": "loopback" if True else "nvlink", "world": W, "rows": rows}))
