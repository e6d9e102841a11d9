"""Online per-microbatch frequency controller.

The composer picks one SM clock per microbatch (MicrobatchPoint.frequency_mhz, reference
compose.py:117-131) and the 1F1B emulator charges `freq_switch_ms` on every stage edge whose two
microbatches run at different clocks (`_switch_delays`, compose.py:398-406; PAPER.md:681 switches
asynchronously between microbatches).  This module executes such a per-stage sequence on the GPU:

  * `measure_switch_ms` times a real clock switch: lock the new clock through NVML and poll the SM
    clock until it reads the target — the measured value replaces the reference's constant
    `GpuModel.freq_switch_ms` (simgpu.py:53);
  * `MicrobatchClockController.run` enqueues the microbatches on a stream and switches clocks at
    microbatch boundaries.  "sync" reproduces the emulator's model (the next microbatch is enqueued
    after the previous one finished and the clock switched: the switch is a gap); "async" enqueues
    everything and a host thread switches the clock the moment the previous microbatch completes
    (the switch overlaps the start of the next one).

Clock locking needs a driver that permits it; on pools where NVML returns NOT_SUPPORTED the
controller runs the sequence at the current clock and reports `switches == []` with the reason.
Device access goes through three small hooks (enqueue / done-event / clock) so the control logic is
testable on CPU with a simulated clock.
"""

from __future__ import annotations

import threading
import time
from dataclasses import dataclass, field


@dataclass
class SwitchRecord:
    index: int            # microbatch that needed the new clock
    from_mhz: float | None
    to_mhz: float
    requested_s: float    # host time the lock was requested
    settled_s: float | None  # host time the SM clock read the target (None: not observed)

    @property
    def latency_ms(self) -> float | None:
        return None if self.settled_s is None else (self.settled_s - self.requested_s) * 1e3


@dataclass
class RunResult:
    mode: str
    total_s: float
    switches: list[SwitchRecord] = field(default_factory=list)
    clock_control: str = ""


def measure_switch_ms(freq, read_clock, target_mhz: float, tol_mhz: float = 15.0, timeout_s: float = 0.5,
                      poll_s: float = 0.0005) -> float | None:
    """Lock `target_mhz` through `freq` (FrequencyController-like: .available, .set) and poll
    `read_clock()` until it is within tol of the target.  None when clocks cannot be locked or the
    clock never settles within `timeout_s`."""
    if not getattr(freq, "available", False):
        return None
    t0 = time.perf_counter()
    freq.set(target_mhz)
    while time.perf_counter() - t0 < timeout_s:
        if abs(read_clock() - target_mhz) <= tol_mhz:
            return (time.perf_counter() - t0) * 1e3
        time.sleep(poll_s)
    return None


class MicrobatchClockController:
    """Runs [(enqueue_fn, freq_mhz), ...] with clock switches at microbatch boundaries.

    hooks:
      enqueue(i)      -> enqueue microbatch i (non-blocking) and return a handle with .synchronize()
                         (a CUDA event recorded after it on the stream);
      freq            -> FrequencyController-like (.available, .set(mhz), .release(), .reason);
      read_clock()    -> current SM clock in MHz (NVML).
    """

    def __init__(self, freq, read_clock, tol_mhz: float = 15.0):
        self.freq = freq
        self.read_clock = read_clock
        self.tol = tol_mhz

    def _switch(self, i, cur, f, rec: list) -> float:
        r = SwitchRecord(i, cur, f, time.perf_counter(), None)
        self.freq.set(f)
        deadline = r.requested_s + 0.5
        while time.perf_counter() < deadline:
            if abs(self.read_clock() - f) <= self.tol:
                r.settled_s = time.perf_counter()
                break
            time.sleep(0.0002)
        rec.append(r)
        return f

    def run(self, freqs: list[float], enqueue, mode: str = "sync") -> RunResult:
        if mode not in ("sync", "async"):
            raise ValueError("mode must be 'sync' or 'async'")
        avail = getattr(self.freq, "available", False)
        res = RunResult(mode, 0.0, [], getattr(self.freq, "reason", ""))
        t0 = time.perf_counter()
        cur = None
        if mode == "sync" or not avail:
            last = None
            for i, f in enumerate(freqs):
                if avail and f != cur:
                    if last is not None:
                        last.synchronize()  # the previous microbatch has finished: the switch is a gap
                    cur = self._switch(i, cur, f, res.switches)
                last = enqueue(i)
            if last is not None:
                last.synchronize()
        else:
            handles: list = [None] * len(freqs)
            ready = [threading.Event() for _ in freqs]
            err: list = []

            def worker():
                nonlocal cur
                try:
                    for i, f in enumerate(freqs):
                        if f != cur:
                            if i > 0:
                                ready[i - 1].wait()
                                handles[i - 1].synchronize()
                            cur = self._switch(i, cur, f, res.switches)
                except Exception as ex:  # pragma: no cover - surfaced below
                    err.append(ex)

            # the first microbatch's clock is set before anything runs
            if freqs:
                cur = self._switch(0, None, freqs[0], res.switches)
            th = threading.Thread(target=worker, daemon=True)
            th.start()
            for i in range(len(freqs)):
                handles[i] = enqueue(i)
                ready[i].set()
            th.join()
            if err:
                raise err[0]
            if handles:
                handles[-1].synchronize()
        res.total_s = time.perf_counter() - t0
        return res
