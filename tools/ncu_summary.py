"""Summarise ncu outputs into profiles/ (tracked).

  python tools/ncu_summary.py launches <launches.csv> <out.md>
  python tools/ncu_summary.py report <file.ncu-rep> <out.md> [label]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def launches(path, out):
    text = open(path).read().splitlines()
    start = next(i for i, ln in enumerate(text) if ln.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(text[start:]))))
    rows = [r for r in rows if r.get("Metric Name") == "gpu__time_duration.sum"]
    per = defaultdict(lambda: [0, 0.0])
    order = []
    for r in rows:
        name = r["Kernel Name"].split("(")[0]
        if name not in per:
            order.append(name)
        per[name][0] += 1
        per[name][1] += float(r["Metric Value"].replace(",", ""))
    total = sum(v[1] for v in per.values())
    lines = [f"# ncu launch list summary ({path.split('/')[-1]})", "",
             f"{len(rows)} launches, {total / 1e6:.3f} ms total (cold-cache, serialised; compare SHARES)", "",
             "| kernel | launches | total ms | share |", "|---|---:|---:|---:|"]
    for name in sorted(per, key=lambda n: -per[n][1]):
        c, t = per[name]
        lines.append(f"| `{name}` | {c} | {t / 1e6:.4f} | {t / total:.3f} |")
    lines += ["", "Per launch (in order):", "", "| # | kernel | grid | block | us |", "|---:|---|---|---|---:|"]
    for i, r in enumerate(rows):
        lines.append(f"| {i} | `{r['Kernel Name'].split('(')[0]}` | {r['Grid Size']} | {r['Block Size']} | "
                     f"{float(r['Metric Value'].replace(',', '')) / 1e3:.1f} |")
    open(out, "w").write("\n".join(lines) + "\n")


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "smsp__inst_executed_pipe_tensor_op_hmma.sum", "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__average_warp_latency_issue_stalled_barrier",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum", "sm__cycles_elapsed.avg.per_second"]


def report(path, out, label=""):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rdr = list(csv.reader(io.StringIO(raw)))
    head, units = rdr[0], rdr[1]
    lines = [f"# ncu --set full: {label or path.split('/')[-1]}", ""]
    for row in rdr[2:]:
        d = dict(zip(head, row))
        u = dict(zip(head, units))
        lines.append(f"## `{d.get('Kernel Name', '?')[:120]}`")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---:|---|")
        for k in head:
            if any(k.startswith(w.split('.')[0]) and k == w for w in WANT) or k in WANT:
                lines.append(f"| {k} | {d[k]} | {u.get(k, '')} |")
        extra = [k for k in head if ("pipe_tc" in k or "pipe_tensor" in k) and "pct" in k and k not in WANT]
        for k in extra[:12]:
            lines.append(f"| {k} | {d[k]} | {u.get(k, '')} |")
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        report(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else "")
