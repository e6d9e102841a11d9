"""Per-microbatch clock controller on a simulated clock: switch latency
measurement, switches exactly at frequency changes, sync (gap) vs async (overlapped) semantics, and
the no-clock-control path the B200 pool takes (NVML NOT_SUPPORTED)."""
import threading
import time

from paper_2601_17654_b200.freqctl import MicrobatchClockController, measure_switch_ms


class FakeClock:
    """Locked clocks take `lag_s` to settle."""

    def __init__(self, start=1965.0, lag_s=0.004, available=True):
        self.available = available
        self.reason = "fake" if available else "unavailable: NOT_SUPPORTED"
        self.mhz, self.target, self.t_set, self.lag = start, start, 0.0, lag_s
        self.sets = []

    def set(self, f):
        self.target, self.t_set = f, time.perf_counter()
        self.sets.append(f)
        return True

    def read(self):
        if time.perf_counter() - self.t_set >= self.lag:
            self.mhz = self.target
        return self.mhz

    def release(self):
        self.sets.append("reset")


class FakeWork:
    """A 'stream' executing microbatches back to back on a thread; records the clock each ran at."""

    def __init__(self, clock, dur_s=0.01):
        self.clock, self.dur = clock, dur_s
        self.lock = threading.Lock()
        self.busy_until = time.perf_counter()
        self.log = []

    def enqueue(self, i):
        done = threading.Event()
        with self.lock:
            start = max(self.busy_until, time.perf_counter())
            self.busy_until = start + self.dur

        def body():
            time.sleep(max(0.0, start - time.perf_counter()))
            self.log.append((i, self.clock.read(), time.perf_counter()))
            time.sleep(self.dur)
            done.set()

        threading.Thread(target=body, daemon=True).start()

        class H:
            def synchronize(self_inner):
                done.wait()
        return H()


def test_measure_switch_latency():
    c = FakeClock(lag_s=0.006)
    ms = measure_switch_ms(c, c.read, 1200.0)
    assert ms is not None and 5.0 <= ms < 50.0
    assert measure_switch_ms(FakeClock(available=False), c.read, 1200.0) is None


def test_sync_switches_only_on_changes_and_runs_at_target():
    c = FakeClock(lag_s=0.003)
    w = FakeWork(c)
    freqs = [1965.0, 1965.0, 1500.0, 1500.0, 1965.0]
    res = MicrobatchClockController(c, c.read).run(freqs, w.enqueue, "sync")
    assert [s.index for s in res.switches] == [0, 2, 4]
    assert all(s.latency_ms is not None and s.latency_ms >= 2.5 for s in res.switches[1:])
    ran = {i: mhz for i, mhz, _ in w.log}
    assert [ran[i] for i in range(5)] == freqs  # every microbatch ran at its assigned clock


def test_async_overlaps_switch_with_next_microbatch():
    lag = 0.02
    c1, c2 = FakeClock(lag_s=lag), FakeClock(lag_s=lag)
    freqs = [1965.0, 1500.0, 1965.0, 1500.0]
    r_sync = MicrobatchClockController(c1, c1.read).run(freqs, FakeWork(c1, 0.02).enqueue, "sync")
    r_async = MicrobatchClockController(c2, c2.read).run(freqs, FakeWork(c2, 0.02).enqueue, "async")
    assert len(r_sync.switches) == len(r_async.switches) == 4
    # sync pays every switch as a gap, async hides it under the next microbatch
    assert r_async.total_s < r_sync.total_s - 1.5 * lag


def test_no_clock_control_runs_at_current_clock():
    c = FakeClock(available=False)
    w = FakeWork(c, 0.002)
    res = MicrobatchClockController(c, c.read).run([1965.0, 1200.0, 1965.0], w.enqueue, "async")
    assert res.switches == [] and "NOT_SUPPORTED" in res.clock_control
    assert len(w.log) == 3 and c.sets == []
