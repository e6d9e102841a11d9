"""Measure the B200 GpuModel descriptor the optimizer's pruning uses (reference GpuModel simgpu.py:35-82,
`comm_rate_bps` :81-82, `kernel_duration` :144-168; pruning mbo.py:107-114).  VERDICT r1 item 9.

  comm    bus bandwidth of the engine's collectives vs CTA budget (loopback group of 8 on a one-GPU
          box: the "link" is HBM, so bandwidth grows linearly with CTAs up to 64; tools/comm_bench.py's
          torchrun mode measures NVLink).  The per-CTA copy rate is measured; the reference's
          `min(1, sm / sat)` knee is projected onto NVLink: sm_bw_saturation = ceil(770 GB/s / per-CTA
          rate), net_bw_gbps = 770 GB/s (see derive()).
  compute every launch unit of the BASELINE config-1 layer timed alone (CUDA events, 20 reps, full
          SMs): effective tensor rate of the compute-bound units -> peak_flops_per_sm_mhz at the
          observed SM clock; effective HBM rate of the memory-bound units -> mem_bw_gbps.
  power   idle P0 power (NVML, 5 s at rest after the runs) -> p_static_w.

Writes gpurun_out/descriptor.json; the committed copy profiles/r2_descriptor.json is what
device.b200_model_measured() loads.  `python tools/calibrate_descriptor.py --derive FILE` recomputes the
descriptor block of an existing measurement file."""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


NVLINK_GBS = 770.0  # measured peer copy per direction, /opt/skills/guides/B200_PROFILING.md (900 nominal)


def derive(out: dict) -> dict:
    """Descriptor from the raw measurements.  The collective's bandwidth grows linearly with its CTA
    count on loopback until HBM saturates (no knee below 64 CTAs: the "link" is HBM there), so the
    saturation knee is projected onto NVLink from the measured per-CTA copy rate:
    sm_bw_saturation = ceil(NVLINK_GBS / per-CTA rate of the slower collective), rounded up to the
    SmGrid stride of 3 (domain.py:69-74); net_bw_gbps = NVLINK_GBS."""
    import math

    from paper_2601_17654_b200.device import b200_model, load_measured_peaks

    rows = out["comm"]["rows"]
    big = max(r["bytes"] for r in rows)
    per_cta = {}
    for op in ("all_gather", "reduce_scatter"):
        rs = [r["busbw_gbs"] / r["ncta"] for r in rows if r["op"] == op and r["bytes"] == big and r["ncta"] <= 12]
        per_cta[op] = sorted(rs)[len(rs) // 2]
    slow = min(per_cta.values())
    sat = int(math.ceil(NVLINK_GBS / slow / 3.0) * 3)
    out["comm"]["per_cta_gbs"] = per_cta
    peaks = load_measured_peaks()
    nominal = b200_model()
    return {
        "num_sms": 148,
        "peak_flops_per_sm_mhz": out["compute"]["peak_flops_per_sm_mhz"],
        "mem_bw_gbps": out["compute"]["effective_hbm_gbs"],
        "net_bw_gbps": NVLINK_GBS,
        "sm_bw_saturation": sat,
        "p_static_w": round(out["idle_power_w"], 1),
        "f_max_mhz": out.get("f_max_mhz", 1965.0),
        "overlap_launch_overhead_ms": 0.0,
        "derivation": {
            "peak_flops_per_sm_mhz": "effective tensor rate of the config-1 layer's compute-bound units alone / "
                                     "(148 SMs x median SM clock)",
            "mem_bw_gbps": "effective HBM rate of the layer's memory-bound units alone",
            "net_bw_gbps": "NVLink peer copy per direction (B200_PROFILING.md); loopback busbw grows to "
                           f"{out['comm']['best_busbw_gbs']} GB/s at 64 CTAs through HBM",
            "sm_bw_saturation": f"ceil({NVLINK_GBS} GB/s / {slow:.1f} GB/s per CTA (measured, slower of "
                                "all-gather / reduce-scatter, <= 12 CTAs, 256 MB)) rounded up to a multiple of 3",
            "p_static_w": "idle NVML power over 5 s (after 8 s at rest)",
            "nominal_for_reference": {"peak_flops_per_sm_mhz": nominal.peak_flops_per_sm_mhz,
                                      "mem_bw_gbps": nominal.mem_bw_gbps,
                                      "measured_peaks": {k: peaks.get(k) for k in ("hbm_gbs", "bf16_tflops")}},
        },
    }


def main():
    import torch

    from paper_2601_17654_b200.comm import Communicator
    from paper_2601_17654_b200.device import b200_model, load_measured_peaks
    from paper_2601_17654_b200.layer import PartitionedLayer, sym_bytes_for
    from paper_2601_17654_b200.model import baseline_workload
    from paper_2601_17654_b200.power import EnergySampler, Nvml

    dev = torch.device("cuda", 0)
    nv = Nvml(0)
    samp = EnergySampler(nv)
    samp.start()
    out = {"when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}

    # ------------------------------------------------------------------ comm curve (loopback, W = 8)
    W = 8
    rows = []
    sizes = [16 << 20, 64 << 20, 256 << 20]
    ctas = [3, 6, 9, 12, 15, 18, 24, 30, 48, 64]
    st = torch.cuda.Stream(dev)
    for total in sizes:
        total = total // (16 * W) * 16 * W
        c = Communicator.loopback_group(W, total + total // W + (4 << 20), device=dev)
        src = c.alloc(total)
        shard = c.alloc(total // W)
        for p in range(W):
            (src.local() if p == 0 else src.peer(p)).normal_()
            (shard.local() if p == 0 else shard.peer(p)).normal_()
        out_ag = torch.empty(total // 2, dtype=torch.bfloat16, device=dev)
        out_rs = torch.empty(total // 2 // W, dtype=torch.bfloat16, device=dev)
        for name, fn in (("all_gather", lambda n: c.all_gather(shard, out_ag, n, stream=st)),
                         ("reduce_scatter", lambda n: c.reduce_scatter(src, out_rs, n, stream=st))):
            for n in ctas:
                fn(n)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                for _ in range(10):
                    fn(n)
                e1.record(st)
                e1.synchronize()
                ms = e0.elapsed_time(e1) / 10
                rows.append({"op": name, "bytes": total, "ncta": n, "ms": round(ms, 5),
                             "busbw_gbs": round((W - 1) / W * total / (ms / 1e3) / 1e9, 1)})
        c.close()
    big = [r for r in rows if r["bytes"] == max(r2["bytes"] for r2 in rows)]
    best = max(r["busbw_gbs"] for r in big)
    out["comm"] = {"mode": "loopback (8 virtual ranks, HBM link)", "rows": rows, "best_busbw_gbs": best}
    print("comm best", best, flush=True)

    # ------------------------------------------------------------------ solo launch units, config 1
    wl = baseline_workload(1)
    comm = Communicator.loopback_group(wl.world, sym_bytes_for(wl), device=dev)
    L = PartitionedLayer(wl, comm)
    s = torch.cuda.Stream(dev)
    units = {}
    for name in L.order:
        for u in L.programs[name].units:
            if u.name in units:
                continue
            for _ in range(3):
                u.fn(s)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record(s)
            for _ in range(20):
                u.fn(s)
            e1.record(s)
            e1.synchronize()
            t1 = time.perf_counter()
            ms = e0.elapsed_time(e1) / 20
            clk = samp.clocks_summary(t0, t1)
            units[u.name] = {"ms": ms, "flops": u.spec.flops, "bytes": u.spec.bytes, "kind": u.spec.kind,
                             "sm_mhz": clk.get("sm_mhz")}
    comp = [v for v in units.values() if v["kind"] == "compute-bound"]
    mem = [v for v in units.values() if v["kind"] == "memory-bound" and v["bytes"] > 1e6]
    clocks = [v["sm_mhz"] for v in comp if v["sm_mhz"]] or [1965.0]
    f_obs = statistics.median(clocks)
    flop_rate = sum(v["flops"] for v in comp) / (sum(v["ms"] for v in comp) / 1e3)
    hbm_rate = sum(v["bytes"] for v in mem) / (sum(v["ms"] for v in mem) / 1e3)
    out["units"] = units
    out["compute"] = {"effective_tflops": flop_rate / 1e12, "sm_mhz_median": f_obs,
                      "peak_flops_per_sm_mhz": flop_rate / (148 * f_obs), "effective_hbm_gbs": hbm_rate / 1e9}
    del L
    comm.close()
    torch.cuda.synchronize()
    # ------------------------------------------------------------------ idle power
    time.sleep(8.0)
    t0 = time.perf_counter()
    time.sleep(5.0)
    t1 = time.perf_counter()
    out["idle_power_w"] = samp.window_j(t0, t1) / (t1 - t0)
    out["idle_temperature_c"] = nv.temperature_c()
    samp.stop()
    out["f_max_mhz"] = nv.max_sm_clock_mhz()
    out["descriptor"] = derive(out)
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/descriptor.json", "w"), indent=1)
    print(json.dumps(out["descriptor"]))


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--derive":
        d = json.load(open(sys.argv[2]))
        d["descriptor"] = derive(d)
        json.dump(d, open(sys.argv[2], "w"), indent=1)
        print(json.dumps(d["descriptor"]))
    else:
        main()
