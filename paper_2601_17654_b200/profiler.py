"""Candidate profiler and profile tables.

The profiler batch-measures candidate schedules (frequency x comm SM budget x launch timing) on
hardware through `Engine.measure` — warmup, measurement window, cooldown per candidate, exactly
the reference protocol (simgpu.py:321-364) — and records the results as a
*profile table*: a JSON-lines file whose first line is a header (GPU descriptor, grids, span cap,
seed, engine facts) and whose rows are the reference's eval-log fields (frontier_io.py:166-190)
plus what the hardware observed (SM clock, temperature, throttle reasons, window length).

Floats are written with Python's shortest round-trip repr (json), so a table replayed through
`ProfileTable.evaluator()` returns bit-identical Measurements.  Replaying a table through the
reference optimizer reproduces its records, frontier and pass labels exactly (tests/
test_optimizer_parity.py); the table is also the resumable artefact.
"""

from __future__ import annotations

import dataclasses
import json
import time
from dataclasses import dataclass, field

from .domain import LaunchTiming, Measurement, ScheduleConfig

TABLE_KIND = "kpo-profile-table"


def config_key(cfg) -> tuple:
    return (float(cfg.frequency_mhz), int(cfg.sm_alloc), cfg.timing.encode())


@dataclass
class ProfileRow:
    frequency_mhz: float
    sm_alloc: int
    timing: str
    time_ms: float
    dyn_energy_j: float
    static_energy_j: float
    total_energy_j: float
    obs: dict = field(default_factory=dict)

    @property
    def key(self) -> tuple:
        return (float(self.frequency_mhz), int(self.sm_alloc), self.timing)

    def config(self, cls=ScheduleConfig, timing_cls=LaunchTiming):
        return cls(self.frequency_mhz, self.sm_alloc, timing_cls.decode(self.timing))


class ProfileTable:
    def __init__(self, partition: str, header: dict | None = None):
        self.partition = partition
        self.header = dict(header or {})
        self.rows: list[ProfileRow] = []
        self._index: dict[tuple, int] = {}

    # ------------------------------------------------------------------ content
    def add(self, cfg, m, obs: dict | None = None) -> ProfileRow:
        row = ProfileRow(float(cfg.frequency_mhz), int(cfg.sm_alloc), cfg.timing.encode(), m.time_ms, m.dyn_energy_j,
                         m.static_energy_j, m.total_energy_j, dict(obs or {}))
        if row.key in self._index:
            raise ValueError(f"config measured twice: {row.key}")
        self._index[row.key] = len(self.rows)
        self.rows.append(row)
        return row

    def lookup(self, cfg) -> ProfileRow:
        return self.rows[self._index[config_key(cfg)]]

    def __contains__(self, cfg) -> bool:
        return config_key(cfg) in self._index

    def __len__(self) -> int:
        return len(self.rows)

    # ------------------------------------------------------------------ replay
    def evaluator(self, measurement_cls=Measurement):
        """A function with the reference `measure` signature (simgpu.py:321-328) answering from
        the table (fields copied, not recomputed, so replays are bit-exact)."""

        def measure(partition, config, gpu=None, thermal=None, protocol=None, state=None):
            r = self.lookup(config)
            return measurement_cls(r.time_ms, r.dyn_energy_j, r.static_energy_j, r.total_energy_j)

        return measure

    # ------------------------------------------------------------------ I/O
    def dumps(self) -> str:
        head = {"kind": TABLE_KIND, "version": 1, "partition": self.partition, **self.header}
        lines = [json.dumps(head, sort_keys=True)]
        for r in self.rows:
            lines.append(json.dumps(dataclasses.asdict(r), sort_keys=True))
        return "\n".join(lines) + "\n"

    def write(self, path: str) -> None:
        with open(path, "w") as f:
            f.write(self.dumps())

    @classmethod
    def loads(cls, text: str) -> "ProfileTable":
        lines = [ln for ln in text.splitlines() if ln.strip()]
        head = json.loads(lines[0])
        if head.get("kind") != TABLE_KIND:
            raise ValueError("not a kpo profile table")
        t = cls(head["partition"], {k: v for k, v in head.items() if k not in ("kind", "version", "partition")})
        for ln in lines[1:]:
            d = json.loads(ln)
            row = ProfileRow(**d)
            t._index[row.key] = len(t.rows)
            t.rows.append(row)
        return t

    @classmethod
    def read(cls, path: str) -> "ProfileTable":
        with open(path) as f:
            return cls.loads(f.read())


def gpu_header(gpu) -> dict:
    return {f.name: getattr(gpu, f.name) for f in dataclasses.fields(gpu)}


def observation_dict(last) -> dict:
    """What the hardware observed during a measurement (engine.Observation), for table rows."""
    if last is None:
        return {}
    if hasattr(last, "as_dict"):
        d = last.as_dict()
        d["window_s"] = round(d.get("window_s", 0.0), 4)
        d["gpu_ms"] = round(d.get("gpu_ms", 0.0), 5)
        return d
    return {"reps": last.reps, "window_s": round(last.window_s, 4), "sm_mhz": last.sm_mhz,
            "temperature_c": last.temperature_c, "reasons": list(last.reasons),
            "clock_control": last.clock_control, "graph": last.graph}


class Profiler:
    """Batch-measures candidates through an engine-like object exposing
    measure(partition, config, gpu, thermal, protocol, state) and `last` observations."""

    def __init__(self, engine, gpu, protocol, thermal=None, state=None):
        self.engine, self.gpu, self.protocol = engine, gpu, protocol
        self.thermal, self.state = thermal, state

    def collect(self, partition, configs, table: ProfileTable | None = None, header: dict | None = None,
                progress=None) -> ProfileTable:
        table = table or ProfileTable(partition.name, {"gpu": gpu_header(self.gpu), **(header or {})})
        t0 = time.perf_counter()
        for i, cfg in enumerate(configs):
            if cfg in table:  # resume
                continue
            m = self.engine.measure(partition, cfg, self.gpu, self.thermal, self.protocol, self.state)
            last = getattr(self.engine, "last", None)
            obs = observation_dict(last)
            table.add(cfg, m, obs)
            if progress:
                progress(i, cfg, m, time.perf_counter() - t0)
        return table
