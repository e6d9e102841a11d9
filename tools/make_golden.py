"""Generate tests/golden/*.json by running the UNMODIFIED reference (schedfront) in this container.

    PYTHONPATH=baseline/_ref python tools/make_golden.py

Outputs (committed; the GPU box never reads /root/reference):
  simgpu_golden.json   reference simulate_schedule / kernel_duration / measure outputs (repr floats)
                       on its four workload partitions (workloads.py:38-93) with the default A100
                       GpuModel, over every config of a reduced enumerated space, plus a measure()
                       sequence with thermal drift, noise and counter quantum.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))

from schedfront import simgpu, workloads  # noqa: E402
from schedfront.domain import FrequencyGrid, KernelSpec, SmGrid  # noqa: E402
from schedfront.mbo import enumerate_space  # noqa: E402


def part_dict(p):
    return {"name": p.name, "comm_group_size": p.comm_group_size,
            "comp": [[k.name, k.flops, k.bytes] for k in p.comp_kernels],
            "comm": [p.comm_kernel.name, p.comm_kernel.comm_bytes]}


def cfg_dict(c):
    return [c.frequency_mhz, c.sm_alloc, c.timing.encode()]


def main():
    gpu = workloads.default_gpu()
    out = {"generator": "tools/make_golden.py", "gpu": vars(gpu) if hasattr(gpu, "__dict__") else {},
           "partitions": [], "kernel_duration": [], "measure_sequence": {}}
    import dataclasses

    out["gpu"] = {f.name: getattr(gpu, f.name) for f in dataclasses.fields(gpu)}
    freqs = FrequencyGrid(tuple(float(f) for f in range(900, 1411, 170)))  # 4 values
    sms = SmGrid((2, 5, 8, 13, 20))
    for p in (workloads.attention_partition(), workloads.mlp_partition(), workloads.small_partition(),
              workloads.interference_partition()):
        space = enumerate_space(p, gpu, freqs, sms, max_overlap_span=9)
        rows = []
        for c in space:
            m = simgpu.simulate_schedule(p, c, gpu)
            rows.append(cfg_dict(c) + [m.time_ms, m.dyn_energy_j, m.static_energy_j, m.total_energy_j])
        out["partitions"].append({"partition": part_dict(p), "rows": rows})
    for k in (KernelSpec("gemm", flops=1e12), KernelSpec("norm", flops=1e6, bytes=1e9),
              KernelSpec("ar", comm_bytes=1e9), KernelSpec("mix", flops=3e11, bytes=2e9)):
        for f in (900.0, 1200.0, 1410.0):
            for sm in (1, 4, 8, 50, 108):
                out["kernel_duration"].append([k.name, k.flops, k.bytes, k.comm_bytes, f, sm,
                                               simgpu.kernel_duration(k, f, sm, gpu)])
    # measure(): thermal drift + noise + counter quantum, state threaded through 40 calls
    p = workloads.attention_partition()
    thermal = workloads.default_thermal()
    proto = simgpu.ProfilingProtocol(2.0, 5.0, 5.0, noise_std_frac=0.02, counter_quantum_j=6.0, seed=1234)
    state = simgpu.ThermalState.new(thermal, proto)
    space = enumerate_space(p, gpu, freqs, sms, max_overlap_span=9)
    seq = []
    for c in space[:: max(1, len(space) // 40)][:40]:
        m = simgpu.measure(p, c, gpu, thermal, proto, state)
        seq.append(cfg_dict(c) + [m.time_ms, m.dyn_energy_j, m.static_energy_j, m.total_energy_j,
                                  state.temperature_c])
    out["measure_sequence"] = {"partition": part_dict(p), "thermal": dataclasses.asdict(thermal),
                               "protocol": dataclasses.asdict(proto), "rows": seq}
    os.makedirs(os.path.join(ROOT, "tests", "golden"), exist_ok=True)
    path = os.path.join(ROOT, "tests", "golden", "simgpu_golden.json")
    with open(path, "w") as f:
        json.dump(out, f)
    print("wrote", path, sum(len(x["rows"]) for x in out["partitions"]), "simulate rows,", len(seq), "measure rows")


if __name__ == "__main__":
    main()
