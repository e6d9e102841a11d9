"""Drop-in plumbing for the reference optimizer (GPU-free).

The reference resolves its hot path as module globals at call time:
  schedfront.mbo.measure                (mbo.py:30 import, called at mbo.py:291)
  schedfront.oracle.simulate_schedule   (oracle.py:24, called at :61 and :138)
  schedfront.compose.simulate_schedule  (compose.py:29, called at :223)
`patch_reference` rebinds them to this engine's callables (an Engine, an SpmdEngine, or a
ProfileTable evaluator) and returns a function that restores the originals.
"""

from __future__ import annotations

import importlib


def _mods(schedfront_module=None):
    if schedfront_module is None:
        schedfront_module = importlib.import_module("schedfront")
    base = schedfront_module.__name__
    return (importlib.import_module(base + ".mbo"), importlib.import_module(base + ".oracle"),
            importlib.import_module(base + ".compose"), importlib.import_module(base + ".domain"))


def reference_measurement_cls(schedfront_module=None):
    return _mods(schedfront_module)[3].Measurement


def patch_reference(measure=None, simulate=None, schedfront_module=None):
    mbo, oracle, compose, _ = _mods(schedfront_module)
    prev = (mbo.measure, oracle.simulate_schedule, compose.simulate_schedule)
    if measure is not None:
        mbo.measure = measure
    if simulate is not None:
        oracle.simulate_schedule = simulate
        compose.simulate_schedule = simulate

    def restore():
        mbo.measure, oracle.simulate_schedule, compose.simulate_schedule = prev

    return restore
