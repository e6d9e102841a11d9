"""NVML frequency / energy controller (host code; pynvml).

Replaces the reference's analytic energy model (`dynamic_energy`, simgpu.py:171-178) and its
frequency knob (`ScheduleConfig.frequency_mhz`, domain.py:151) with the device's own counters:

  * energy: `nvmlDeviceGetTotalEnergyConsumption` (mJ).  The counter advances in ~100 ms steps on
    this pool's B200s (tools/box_probe.py), so an `EnergySampler` thread timestamps every step
    and the window energy is interpolated at the window's exact host start/end times;
  * clocks: `nvmlDeviceSetGpuLockedClocks` per partition when the driver permits it.  On the
    pool's boxes it returns NOT_SUPPORTED (measured), so `FrequencyController` reports
    `available == False` and the engine records the clock actually observed instead of
    pretending to have set one;
  * temperature / throttle reasons for the thermally-stable protocol (simgpu.py:289-364).
"""

from __future__ import annotations

import bisect
import threading
import time

try:
    import pynvml
except Exception:  # pragma: no cover - pynvml is in the image
    pynvml = None

_THROTTLE_NAMES = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
    0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
    0x100: "display_clock_setting",
}


class Nvml:
    _inited = False

    def __init__(self, index: int = 0):
        if pynvml is None:
            raise RuntimeError("pynvml unavailable")
        if not Nvml._inited:
            pynvml.nvmlInit()
            Nvml._inited = True
        self.index = index
        self.h = pynvml.nvmlDeviceGetHandleByIndex(index)

    def energy_mj(self) -> int:
        return pynvml.nvmlDeviceGetTotalEnergyConsumption(self.h)

    def power_w(self) -> float:
        return pynvml.nvmlDeviceGetPowerUsage(self.h) / 1000.0

    def temperature_c(self) -> float:
        return float(pynvml.nvmlDeviceGetTemperature(self.h, pynvml.NVML_TEMPERATURE_GPU))

    def sm_clock_mhz(self) -> float:
        return float(pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM))

    def max_sm_clock_mhz(self) -> float:
        return float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))

    def supported_sm_clocks(self) -> list[float]:
        mem = pynvml.nvmlDeviceGetSupportedMemoryClocks(self.h)
        return [float(f) for f in pynvml.nvmlDeviceGetSupportedGraphicsClocks(self.h, mem[0])]

    def throttle_reasons(self) -> list[str]:
        try:
            mask = pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            mask = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        return [n for bit, n in _THROTTLE_NAMES.items() if mask & bit]


class FrequencyController:
    """Per-partition locked SM clocks, if the driver allows it (always reset on release)."""

    def __init__(self, nvml: Nvml, enable: bool = True):
        self.nvml = nvml
        self.available = False
        self.reason = "disabled"
        self.current: float | None = None
        if enable:
            self._probe()

    def _probe(self) -> None:
        try:
            f = self.nvml.max_sm_clock_mhz()
            pynvml.nvmlDeviceSetGpuLockedClocks(self.nvml.h, int(f), int(f))
            pynvml.nvmlDeviceResetGpuLockedClocks(self.nvml.h)
            self.available = True
            self.reason = "nvml-locked-clocks"
        except Exception as ex:  # NVMLError_NotSupported / NoPermission on shared pools
            self.available = False
            self.reason = f"unavailable: {ex!r}"

    def set(self, mhz: float) -> bool:
        if not self.available:
            return False
        if self.current == mhz:
            return True
        pynvml.nvmlDeviceSetGpuLockedClocks(self.nvml.h, int(mhz), int(mhz))
        self.current = mhz
        return True

    def release(self) -> None:
        if self.available and self.current is not None:
            try:
                pynvml.nvmlDeviceResetGpuLockedClocks(self.nvml.h)
            finally:
                self.current = None


class EnergySampler:
    """Background poller that timestamps every step of the NVML energy counter, plus SM clock,
    power and throttle reasons, so windows can be integrated at arbitrary host times."""

    def __init__(self, nvml: Nvml, period_s: float = 0.002, aux_period_s: float = 0.05):
        self.nvml = nvml
        self.period_s = period_s
        self.aux_period_s = aux_period_s
        self._t: list[float] = []
        self._e: list[int] = []
        self.aux: list[tuple[float, float, float, tuple[str, ...]]] = []  # (t, sm_mhz, power_w, reasons)
        self._stop = threading.Event()
        self._lock = threading.Lock()
        self._thr = None

    def __enter__(self):
        self.start()
        return self

    def __exit__(self, *exc):
        self.stop()

    def start(self) -> None:
        e = self.nvml.energy_mj()
        self._t, self._e = [time.perf_counter()], [e]
        self._stop.clear()
        self._thr = threading.Thread(target=self._run, daemon=True)
        self._thr.start()

    def stop(self) -> None:
        self._stop.set()
        if self._thr:
            self._thr.join()

    def _run(self) -> None:
        last_aux = 0.0
        while not self._stop.is_set():
            now = time.perf_counter()
            e = self.nvml.energy_mj()
            with self._lock:
                if e != self._e[-1]:
                    self._t.append(now)
                    self._e.append(e)
            if now - last_aux >= self.aux_period_s:
                last_aux = now
                try:
                    self.aux.append((now, self.nvml.sm_clock_mhz(), self.nvml.power_w(),
                                     tuple(self.nvml.throttle_reasons())))
                except Exception:
                    pass
            time.sleep(self.period_s)

    def energy_at(self, t: float) -> float:
        """Counter value (mJ) interpolated linearly between the steps bracketing host time t."""
        with self._lock:
            ts, es = list(self._t), list(self._e)
        i = bisect.bisect_right(ts, t)
        if i == 0:
            return float(es[0])
        if i >= len(ts):
            return float(es[-1])
        t0, t1, e0, e1 = ts[i - 1], ts[i], es[i - 1], es[i]
        return e0 + (e1 - e0) * (t - t0) / max(t1 - t0, 1e-9)

    def window_j(self, t0: float, t1: float, settle_s: float = 0.25) -> float:
        """Energy (J) between host times t0 and t1; waits until the counter has stepped past t1."""
        deadline = time.perf_counter() + settle_s
        while time.perf_counter() < deadline:
            with self._lock:
                if self._t[-1] > t1:
                    break
            time.sleep(0.005)
        return (self.energy_at(t1) - self.energy_at(t0)) / 1000.0

    def clocks_summary(self, t0: float, t1: float) -> dict:
        rows = [a for a in self.aux if t0 <= a[0] <= t1]
        if not rows:
            return {"samples": 0}
        mhz = sorted(r[1] for r in rows)
        reasons = sorted({x for r in rows for x in r[3]} - {"gpu_idle"})
        return {"samples": len(rows), "sm_mhz": mhz[len(mhz) // 2], "power_w_max": max(r[2] for r in rows),
                "reasons": reasons}
