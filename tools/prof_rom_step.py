"""Steady-state per-operation wall time of one reduced PRK2 step at C3 size
(dev tool): each op is synchronised and timed after a warm-up pass, so the
caching allocator and graph/plan caches are hot."""
import sys
import time
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2201_05555_b200 import _build, driver, reduction

_build.build()
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
p, n, nx, d, dt = 128, 20, 64, 2, 0.05
rng = np.random.default_rng(0)
lengths = 2 * np.pi / rng.uniform(0.4, 0.6, p)
sysm = driver.ParametricVlasovSystem(lengths, nx, d, N)
u = torch.from_numpy(np.linalg.qr(rng.standard_normal((2 * N, n)))[0]).cuda()
z = rng.standard_normal((n, p)) * 30.0
sub = np.arange(p)
T = defaultdict(list)


def timed(name, fn, *a, **k):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn(*a, **k)
    torch.cuda.synchronize()
    T[name].append((time.perf_counter() - t0) * 1e3)
    return out


def one_step():
    g0 = timed("exact_gradients(u)", lambda: driver.exact_gradients_device(sysm, u, z, sub, harvest=False)[0])
    s0 = timed("SMatrix", reduction.SMatrix, z)
    xi1 = timed("basis_velocity(u)", reduction.basis_velocity, u, z, g0, s=s0)
    half = timed("scaled", reduction.scaled, xi1, 0.5 * dt)
    umid = timed("retraction(half)", reduction.retraction, u, half)
    g = timed("coeff_stage", driver.make_full_stage(sysm), umid)
    for _ in range(3):
        timed("g(z) [x iters]", g, z)
    gm = timed("exact_gradients(u_mid)", lambda: driver.exact_gradients_device(sysm, umid, z, sub, harvest=False)[0])
    xim = timed("basis_velocity(u_mid)", reduction.basis_velocity, umid, z, gm)
    xi2 = timed("tangent_velocity", reduction.tangent_velocity, u, half, umid, xim)
    full = timed("scaled", reduction.scaled, xi2, dt)
    timed("retraction(full)", reduction.retraction, u, full)


one_step()
T.clear()
for _ in range(3):
    one_step()
tot = 0.0
for k, v in T.items():
    per = float(np.median(v)) * (len(v) / 3)
    tot += per if "g(z)" not in k else 0
    print(f"{k:28s} {np.median(v):8.3f} ms  (x{len(v) // 3} per step)")
print(f"{'basis phase total':28s} {tot:8.3f} ms")
