"""1F1B validation on hardware: PP x TP grid of B200s, e.g. PP2 x TP4 on 8 GPUs.

  torchrun --nproc-per-node 8 --master-addr 127.0.0.1 tools/pipeline_1f1b.py --pp 2 --tp 4

Every stage runs `--layers` Llama-3-8B layers per op (TP over its 4 ranks, engine P2P all-reduces
under the default nanobatching schedule); microbatch activations / gradients move between stages over
NCCL send/recv.  Per-op energies are NVML windows of each op run back to back; the reference emulator
(compose.simulate_pipeline) is fed the measured op durations and energies and compared with the
measured iteration (makespan max over ranks, energy summed over ranks).  Prints one JSON line on rank 0.
Needs pp*tp GPUs (this pool's boxes have one, so it has not been run on hardware; the control plane
is tests/test_pipeline_gloo.py)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.append(os.path.join(ROOT, "baseline", "_ref"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pp", type=int, default=2)
    ap.add_argument("--tp", type=int, default=4)
    ap.add_argument("--microbatches", type=int, default=8)
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--tokens", type=int, default=4096)
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    from paper_2601_17654_b200.comm import Communicator
    from paper_2601_17654_b200.device import b200_model
    from paper_2601_17654_b200.engine import Engine
    from paper_2601_17654_b200.layer import PartitionedLayer, sym_bytes_for
    from paper_2601_17654_b200.model import PRESETS, Workload
    from paper_2601_17654_b200.pipeline import Grid, LayerStageWork, emulate, gather_runs, run_iteration
    from paper_2601_17654_b200.runner import default_schedule

    grid = Grid(a.pp, a.tp)
    wl = Workload(PRESETS["llama-3-8b"], "tp", a.tp, a.tokens)
    comm = Communicator.from_process_group(sym_bytes_for(wl), device=dev, group=grid.tp_group)
    layer = PartitionedLayer(wl, comm)
    gpu = b200_model()
    eng = Engine.for_layer(layer, gpu, clock_control=False)
    work = LayerStageWork(layer, eng, default_schedule(layer, gpu), a.layers)
    run_iteration(grid, work, a.microbatches)  # warm-up iteration
    # per-op energy: each op type back to back for ~1 s (NVML window), per rank
    op_e = {}
    for d in ("F", "B"):
        fn = (lambda: work.forward(0, None)) if d == "F" else (lambda: work.backward(0, None))
        _, ms = work.timed(fn)
        n = max(3, int(1000 / max(ms, 1e-3)))
        dist.barrier()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        for _ in range(n):
            fn()
        torch.cuda.synchronize()
        w1 = time.perf_counter()
        e = torch.tensor([eng.sampler.window_j(w0, w1) / n], device=dev, dtype=torch.float64)
        dist.all_reduce(e, group=grid.tp_group)  # the stage's energy = sum over its tp ranks
        op_e[(grid.stage, d)] = float(e)
    all_e = [None] * dist.get_world_size()
    dist.all_gather_object(all_e, op_e)
    op_energy = {k: v for d_ in all_e for k, v in d_.items()}
    run = run_iteration(grid, work, a.microbatches, sampler=eng.sampler)
    runs = gather_runs(run)
    if dist.get_rank() == 0:
        import schedfront
        rep = emulate(runs, a.pp, a.microbatches, gpu.p_static_w * a.tp, op_energy=op_energy,
                      schedfront_module=schedfront)
        print(json.dumps({"pp": a.pp, "tp": a.tp, "microbatches": a.microbatches, "layers_per_stage": a.layers,
                          "workload": wl.tag, **rep}))
    eng.close()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
