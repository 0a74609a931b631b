"""Seeded synthetic inputs for the five BASELINE.json configurations (C1-C5).

The paper's benchmarks are analytic initial distributions; BASELINE.json asks
for seeded pseudo-random loading, so each instance i draws
from numpy.random.default_rng(SeedSequence(seed).spawn(p)[i]): positions by
rejection against 1 + alpha cos(k x) on [0, 2 pi / k), velocities from the
config's model.  Parameter draws use default_rng(seed) (separate stream).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

DEFAULT_SEED = 20220114


@dataclass
class Workload:
    name: str
    num_particles: int
    num_cells: int
    degree: int
    dt: float
    num_steps: int
    wavenumbers: np.ndarray      # (p,)
    alphas: np.ndarray           # (p,)
    velocity: str                # "maxwellian" | "two_stream" | "bump_on_tail"
    vparams: np.ndarray          # (p, k) model parameters per instance
    seed: int = DEFAULT_SEED
    extra: dict = field(default_factory=dict)

    @property
    def p(self):
        return len(self.alphas)

    @property
    def lengths(self):
        return 2.0 * np.pi / self.wavenumbers

    @property
    def single_mesh(self):
        return bool(np.all(self.wavenumbers == self.wavenumbers[0]))

    def describe(self):
        return {"workload": self.name, "num_particles": self.num_particles, "p": self.p,
                "num_cells": self.num_cells, "degree": self.degree, "dt": self.dt,
                "steps": self.num_steps, "seed": self.seed}


def _positions(rng, n, alpha, k):
    length = 2.0 * np.pi / k
    out = np.empty(n)
    filled = 0
    while filled < n:
        m = int((n - filled) * (1.0 + alpha) * 1.05) + 64
        u = rng.uniform(0.0, length, m)
        acc = rng.uniform(0.0, 1.0 + alpha, m) < 1.0 + alpha * np.cos(k * u)
        take = u[acc][: n - filled]
        out[filled:filled + take.size] = take
        filled += take.size
    return out


def _velocities(rng, n, model, prm):
    if model == "maxwellian":
        return rng.standard_normal(n)
    if model == "two_stream":
        v0, sigma = prm
        sign = np.where(rng.uniform(size=n) < 0.5, -1.0, 1.0)
        return sign * v0 + sigma * rng.standard_normal(n)
    if model == "bump_on_tail":
        vb, sb, frac = prm
        bump = rng.uniform(size=n) < frac
        base = rng.standard_normal(n)
        return np.where(bump, vb + sb * base, base)
    raise ValueError(model)


def generate(w: Workload, num_particles=None, instances=None, layout="np"):
    """(x0, v0): (N, p) reference layout ("np") or (p, N) device layout ("pn")."""
    n = int(num_particles or w.num_particles)
    cols = list(range(w.p)) if instances is None else list(instances)
    seqs = np.random.SeedSequence(w.seed).spawn(w.p)
    x = np.empty((len(cols), n))
    v = np.empty((len(cols), n))
    for r, j in enumerate(cols):
        rng = np.random.default_rng(seqs[j])
        x[r] = _positions(rng, n, w.alphas[j], w.wavenumbers[j])
        v[r] = _velocities(rng, n, w.velocity, w.vparams[j])
    if layout == "pn":
        return x, v
    return np.ascontiguousarray(x.T), np.ascontiguousarray(v.T)


def config(name, seed=DEFAULT_SEED):
    """BASELINE.json configs[0..4] as Workload objects (C1..C5)."""
    rng = np.random.default_rng(seed)
    name = name.upper()
    if name == "C1":    # linear Landau damping, one instance, quadratic splines
        return Workload("C1", 100_000, 64, 2, 0.05, 200, np.array([0.5]), np.array([0.01]),
                        "maxwellian", np.zeros((1, 0)), seed)
    if name == "C2":    # two-stream, 4 x 8 (alpha, v0) grid, cubic splines
        al, v0 = np.meshgrid([0.001, 0.004, 0.007, 0.01], np.linspace(2.0, 3.4, 8), indexing="ij")
        al, v0 = al.ravel(), v0.ravel()
        return Workload("C2", 250_000, 128, 3, 0.05, 500, np.full(32, 0.2), al, "two_stream",
                        np.stack([v0, np.full(32, 0.3)], axis=1), seed)
    if name in ("C3", "C4"):   # nonlinear reduced-basis Landau instances, per-instance k
        k = rng.uniform(0.4, 0.6, 128)
        al = rng.uniform(0.01, 0.1, 128)
        w = Workload(name, 1_000_000, 64, 2, 0.05, 200, k, al, "maxwellian",
                     np.zeros((128, 0)), seed)
        w.extra = {"basis_dim": 20}
        if name == "C4":
            w.extra.update(subsample=20, window=20, deim_dim=40, deim_period=3, deim_update=12)
        return w
    if name == "C5":    # large bump-on-tail, cubic splines
        al = rng.uniform(0.02, 0.06, 64)
        vb = rng.uniform(4.0, 5.0, 64)
        return Workload("C5", 4_000_000, 512, 3, 0.05, 100, np.full(64, 0.3), al, "bump_on_tail",
                        np.stack([vb, np.full(64, 0.5), np.full(64, 0.1)], axis=1), seed)
    raise ValueError(f"unknown config {name!r}")
