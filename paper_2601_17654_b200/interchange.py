"""Wire formats: hardware profile tables -> the reference's frontier CSV and eval-log JSONL.

The reference exchanges partition / microbatch / iteration frontiers as one CSV schema and the
optimizer's evaluations as a JSON-lines log (reference frontier_io.py:21-48 header and writer,
:97-118 rows of an MBO frontier, :120-144 microbatch rows, :166-190 eval log).  This module writes
the same bytes from a B200 profile table (profiler.ProfileTable) or a composed microbatch frontier,
so hardware measurements feed the reference CLI unchanged, e.g.

    python -m paper_2601_17654_b200.interchange profiles/tables/X.jsonl --out out/
    schedfront compare --frontier-a out/X_frontier.csv --frontier-b other.csv

Floats are written with repr (shortest round trip), as the reference does, so reading a file back
reproduces the measured values exactly.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os

from .profiler import ProfileTable

CSV_HEADER = ["time_ms", "dyn_energy_j", "total_energy_j", "frequency_mhz", "sm_alloc", "timing", "provenance"]


def _fmt(v) -> str:
    if v is None:
        return ""
    if isinstance(v, float):
        return repr(v)
    return str(v)


def render_frontier_csv(rows) -> str:
    """rows: iterables of (time_ms, dyn_energy_j, total_energy_j, frequency_mhz, sm_alloc, timing,
    provenance) in CSV_HEADER order (frontier_io.py:50-66)."""
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(CSV_HEADER)
    for r in rows:
        t, dyn, tot, f, sm, timing, prov = r
        w.writerow([_fmt(t), _fmt(dyn), _fmt(tot), _fmt(f), _fmt(sm), timing, prov])
    return buf.getvalue()


def _nondominated(points):
    """Non-dominated (time, energy) subset, time ascending, energy strictly descending; among equal
    objectives the first in input order is kept (the reference get_frontier tie rule for payloads
    without a sort key, domain.py:315-360)."""
    order = sorted(range(len(points)), key=lambda i: (points[i][0], points[i][1], i))
    out, best = [], float("inf")
    for i in order:
        t, e = points[i][0], points[i][1]
        if e < best:
            out.append(i)
            best = e
    return out


def table_frontier_rows(table: ProfileTable, provenance: str = "hardware"):
    """The (time, dynamic energy) frontier of a profile table as frontier-CSV rows, each with its
    realizing config (the shape of rows_from_mbo, frontier_io.py:97-118)."""
    pts = [(r.time_ms, r.dyn_energy_j) for r in table.rows]
    rows = []
    for i in _nondominated(pts):
        r = table.rows[i]
        rows.append((r.time_ms, r.dyn_energy_j, r.total_energy_j, float(r.frequency_mhz), int(r.sm_alloc), r.timing,
                     r.obs.get("pass", provenance) if isinstance(r.obs, dict) else provenance))
    return rows


def microbatch_frontier_rows(frontier):
    """Rows of a composed microbatch frontier (reference ParetoFrontier of MicrobatchPoint payloads;
    frontier_io.py:120-144)."""
    rows = []
    for fp in frontier:
        p = fp.payload
        timing = "|".join(f"{n}:{c.sm_alloc}:{c.timing.encode()}" for n, c in p.choices)
        rows.append((fp.time_ms, p.dyn_energy_j, fp.energy_j, p.frequency_mhz, None, timing, p.execution_model))
    return rows


def render_eval_log(table: ProfileTable) -> str:
    """The reference eval log (frontier_io.py:166-190) of every measured row, in measurement order.
    `batch` is the row index and `pass` the row's recorded pass label (or "profile")."""
    lines = []
    for i, r in enumerate(table.rows):
        obs = r.obs if isinstance(r.obs, dict) else {}
        lines.append(json.dumps({
            "partition": table.partition,
            "batch": int(obs.get("batch", i)),
            "pass": obs.get("pass", "profile"),
            "config": {"frequency_mhz": r.frequency_mhz, "sm_alloc": r.sm_alloc, "timing": r.timing},
            "measurement": {"time_ms": r.time_ms, "dyn_energy_j": r.dyn_energy_j,
                            "static_energy_j": r.static_energy_j, "total_energy_j": r.total_energy_j},
        }, sort_keys=True))
    return "\n".join(lines) + ("\n" if lines else "")


def export_table(path: str, out_dir: str) -> dict[str, str]:
    t = ProfileTable.read(path)
    os.makedirs(out_dir, exist_ok=True)
    base = os.path.join(out_dir, t.partition)
    files = {base + "_frontier.csv": render_frontier_csv(table_frontier_rows(t)),
             base + "_eval.jsonl": render_eval_log(t)}
    for p, text in files.items():
        with open(p, "w", newline="") as f:
            f.write(text)
    return files


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description="profile table -> reference frontier CSV + eval log")
    ap.add_argument("tables", nargs="+")
    ap.add_argument("--out", default=".")
    a = ap.parse_args(argv)
    for p in a.tables:
        for f in export_table(p, a.out):
            print(f)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
