"""Synchronised wall time of the pieces of reduced steps at full size (dev
tool): wraps the listed functions with cuda-synchronised timers, runs C3/C4 and
prints per-step milliseconds over the last `steps` steps.
    python tools/prof_rom_host.py C4 [steps]"""
import sys
import time
from collections import defaultdict
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2201_05555_b200 import driver, hyper, reduction, workloads as wl  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
T = defaultdict(float)
C = defaultdict(int)
state = {"on": False, "k": 0}


def wrap(mod, name, label=None):
    fn = getattr(mod, name)
    label = label or f"{mod.__name__.split('.')[-1]}.{name}"

    def w(*a, **k):
        if not state["on"]:
            return fn(*a, **k)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn(*a, **k)
        torch.cuda.synchronize()
        T[label] += time.perf_counter() - t0
        C[label] += 1
        return out
    setattr(mod, name, w)


for mod, names in ((hyper, ["_window_svd", "_orth_factor", "_tsq", "_mul", "svd", "_greedy_device", "_rows",
                            "fit_parametric_dmd", "fit_deim_device", "make_hyper_stage_device"]),
                   (hyper.DeimWindow, ["append", "eigh"]),
                   (driver, ["exact_gradients_device", "prk2_step", "orthosymplectic_residuals"]),
                   (reduction, ["basis_velocity", "retraction", "tangent_velocity", "SMatrix"]),
                   (reduction.DeviceFixedPoint, ["__call__"])):
    for nm in names:
        wrap(mod, nm)

w = wl.config(cfg)
x0, v0 = wl.generate(w)
params = np.stack([w.wavenumbers, w.alphas], axis=1)
ex = w.extra
system = driver.ParametricVlasovSystem(w.lengths, w.num_cells, w.degree, w.num_particles)
u0, z0 = reduction.complex_svd_basis(x0, v0, ex["basis_dim"], device=True)
hyper_on = cfg.upper() == "C4"
warm = (ex.get("window", 3) + 3) if hyper_on else 3
orig = driver.prk2_step


def count(*a, **k):
    state["k"] += 1
    return orig(*a, **k)


driver.prk2_step = count
orig_fit_dmd = hyper.fit_parametric_dmd


class Timers:
    def __init__(self):
        from paper_2201_05555_b200.diagnostics import PhaseTimers
        self.t = PhaseTimers()

    def phase(self, name):
        if state["k"] == warm and not state["on"]:
            state["on"] = True
        return self.t.phase(name)

    def flush_step(self):
        self.t.flush_step()

    def series_arrays(self):
        return self.t.series_arrays()


tm = Timers()
rec = driver.run_reduced(system, params, x0, v0, basis_dim=ex["basis_dim"],
                         subsample=ex.get("subsample", w.p), window=ex.get("window", 3),
                         deim_dim=ex.get("deim_dim", 8), deim_period=ex.get("deim_period", 3),
                         deim_update=ex.get("deim_update", 2), dt=w.dt,
                         t_final=(warm + steps) * w.dt, hyper_reduction=hyper_on,
                         energy_stride=10**9, record_snapshots=False, decomp_stride=10**9,
                         u0=u0, z0=z0, timers=tm)
ser = tm.series_arrays()
print(cfg, "phases ms/step:", {k: round(1e3 * float(np.mean(v[-steps:])), 2) for k, v in ser.items()})
for k in sorted(T, key=lambda k: -T[k]):
    print(f"  {1e3 * T[k] / steps:8.2f} ms/step  x{C[k] / steps:5.1f}  {k}")
