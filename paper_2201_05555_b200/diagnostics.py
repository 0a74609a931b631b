"""Phase timers (mirror of picrom.diagnostics.PhaseTimers, diagnostics.py:169-195).

Wall time per labelled phase with a per-step series; the reduced loop
brackets its phases exactly as the reference does (rom_basis, rom_coeff,
dmd_fit, deim_fit).  Device work is asynchronous, so a phase that ends in a
host read (every phase of the reduced step does) measures device time too.
"""

from __future__ import annotations

import time
from collections import defaultdict
from contextlib import contextmanager

import numpy as np


class PhaseTimers:
    def __init__(self, names=("fom_step", "rom_basis", "rom_coeff", "dmd_fit", "deim_fit")):
        self.names = tuple(names)
        self.totals = {k: 0.0 for k in self.names}
        self.series = {k: [] for k in self.names}
        self._current = defaultdict(float)

    @contextmanager
    def phase(self, name):
        t0 = time.perf_counter()
        try:
            yield
        finally:
            el = time.perf_counter() - t0
            self.totals[name] = self.totals.get(name, 0.0) + el
            self._current[name] += el

    def flush_step(self):
        for k in self.names:
            self.series[k].append(self._current.get(k, 0.0))
        self._current.clear()

    def series_arrays(self):
        return {k: np.asarray(v) for k, v in self.series.items()}
