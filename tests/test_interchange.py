"""Wire formats: a hardware profile table exported by
paper_2601_17654_b200.interchange is read by the reference's own frontier_io and CLI unchanged,
byte-identical to what the reference writes for the same rows."""
import glob
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TABLES = sorted(glob.glob(os.path.join(ROOT, "profiles", "tables", "*.jsonl")))


@pytest.mark.parametrize("path", TABLES)
def test_table_export_reads_back_exactly(schedfront, tmp_path, path):
    from schedfront import frontier_io as fio

    from paper_2601_17654_b200.interchange import export_table, render_frontier_csv, table_frontier_rows
    from paper_2601_17654_b200.profiler import ProfileTable
    t = ProfileTable.read(path)
    files = export_table(path, str(tmp_path))
    csv_path = next(p for p in files if p.endswith(".csv"))
    log_path = next(p for p in files if p.endswith(".jsonl"))
    rows = fio.read_frontier_csv(csv_path)
    mine = table_frontier_rows(t)
    assert [(r.time_ms, r.dyn_energy_j, r.total_energy_j, r.frequency_mhz, r.sm_alloc, r.timing) for r in rows] == \
        [m[:6] for m in mine]
    # the reference writer produces the same bytes for the same rows
    ref_rows = [fio.FrontierRow(*m) for m in mine]
    assert fio.render_frontier_csv(ref_rows) == render_frontier_csv(mine)
    # frontier property against the reference's get_frontier
    front = schedfront.domain.get_frontier([(r.time_ms, r.dyn_energy_j) for r in t.rows])
    assert [(p.time_ms, p.energy_j) for p in front] == [(r.time_ms, r.dyn_energy_j) for r in rows]
    log = fio.parse_eval_log(open(log_path).read())
    assert len(log) == len(t.rows)
    for rec, r in zip(log, t.rows):
        assert rec["partition"] == t.partition
        assert rec["config"] == {"frequency_mhz": r.frequency_mhz, "sm_alloc": r.sm_alloc, "timing": r.timing}
        assert rec["measurement"]["time_ms"] == r.time_ms and rec["measurement"]["total_energy_j"] == r.total_energy_j


@pytest.mark.parametrize("path", TABLES[:1])
def test_reference_cli_compare_consumes_exported_frontiers(schedfront, tmp_path, path, capsys):
    """`schedfront compare --frontier-a/--frontier-b` on two hardware frontiers (the sequential
    Megatron-style rows vs every measured row)."""
    from schedfront.cli import EXIT_OK, cmd_compare

    from paper_2601_17654_b200.interchange import render_frontier_csv, table_frontier_rows
    from paper_2601_17654_b200.profiler import ProfileTable
    t = ProfileTable.read(path)
    seq = ProfileTable(t.partition, t.header)
    for r in t.rows:
        if r.timing == "seq":
            seq.rows.append(r)
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    a.write_text(render_frontier_csv(table_frontier_rows(seq)))
    b.write_text(render_frontier_csv(table_frontier_rows(t)))
    assert cmd_compare(out_dir=str(tmp_path), frontier_a=str(a), frontier_b=str(b)) == EXIT_OK
    out = capsys.readouterr().out
    assert "hv_ratio_b_over_a" in out


def test_microbatch_rows_match_reference_writer(schedfront):
    from schedfront import frontier_io as fio
    from schedfront.compose import MicrobatchSpec, TypeChoice, microbatch_frontier
    from schedfront.domain import LaunchTiming, ScheduleConfig

    from paper_2601_17654_b200.interchange import microbatch_frontier_rows, render_frontier_csv
    f = 1965.0
    choices = {"a": [TypeChoice(1.0, 3.0, ScheduleConfig(f, 8, LaunchTiming.overlap(0, 2))),
                     TypeChoice(1.5, 2.0, ScheduleConfig(f, 16, LaunchTiming.sequential()))],
               "b": [TypeChoice(2.0, 1.0, ScheduleConfig(f, 4, LaunchTiming.overlap(1, 3)))]}
    spec = MicrobatchSpec("mb", ("a", "b", "a"), {f: (0.25, 0.5)})
    front = microbatch_frontier(spec, {k: {f: v} for k, v in choices.items()}, 205.0)
    assert render_frontier_csv(microbatch_frontier_rows(front)) == fio.render_frontier_csv(fio.rows_from_microbatch(front))
