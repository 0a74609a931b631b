"""ORACLE (test infrastructure only): full-order PIC (Stoermer-Verlet) on CPU.

Restates /root/reference/pkg/src/picrom/fullorder.py:57-226 for degree-d
splines: ``System.field`` (fullorder.py:66-92, including the column-chunk
thread pool, bit-identical to serial), ``Stepper.step`` kick-drift-kick with the
cached end-of-step field (fullorder.py:102-134) and ``run`` (fullorder.py:
169-226) which additionally keeps the per-step charge/potential/energy history
BASELINE's parity contract is stated on.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from . import fe_bspline as fe


class System:
    """fullorder.VlasovSystem restated (fullorder.py:57-99)."""

    def __init__(self, mesh, charge, workers=1):
        self.mesh = mesh
        self.charge = charge
        self.poisson = fe.Poisson(mesh)
        self.workers = max(1, int(workers))
        self._pool = None

    def _block(self, x):
        basis, grad = fe.eval_basis_pair(self.mesh, x)
        rho = fe.deposit_charge(basis, self.charge)
        phi = self.poisson.solve(rho)
        return fe.field_at_particles(grad, phi, self.charge), phi, rho

    def field_full(self, x):
        """(E, phi, rho) -- rho is kept for the per-step parity history."""
        x = np.asarray(x, dtype=float)
        if self.workers == 1 or x.ndim == 1 or x.shape[1] < 2 * self.workers:
            return self._block(x)
        p = x.shape[1]
        bounds = np.linspace(0, p, self.workers + 1).astype(int)
        e = np.empty_like(x)
        phi = np.empty((self.mesh.num_cells, p))
        rho = np.empty((self.mesh.num_cells, p))
        if self._pool is None:
            self._pool = ThreadPoolExecutor(max_workers=self.workers)
        jobs = {self._pool.submit(self._block, x[:, a:b]): (a, b)
                for a, b in zip(bounds[:-1], bounds[1:]) if b > a}
        for job, (a, b) in jobs.items():
            e[:, a:b], phi[:, a:b], rho[:, a:b] = job.result()
        return e, phi, rho

    def field(self, x):
        e, phi, _ = self.field_full(x)
        return e, phi

    def hamiltonian(self, x, v):
        v = np.asarray(v, dtype=float)
        kinetic = 0.5 * np.einsum("i...,i...->...", v, v)
        basis, _ = fe.eval_basis_pair(self.mesh, x)
        phi = self.poisson.solve(fe.deposit_charge(basis, self.charge))
        return kinetic + fe.electric_energy(self.poisson, phi, self.charge)


class Stepper:
    """fullorder.VerletStepper restated (fullorder.py:102-134)."""

    def __init__(self, system):
        self.system = system
        self.cache_time = None
        self.cache_field = None
        self.last_potential = None
        self.last_rho = None

    def step(self, x, v, t, dt):
        if self.cache_time == t and self.cache_field is not None:
            e0 = self.cache_field
        else:
            e0, self.last_potential, self.last_rho = self.system.field_full(x)
        x1 = x + dt * (v + 0.5 * dt * e0)
        e1, phi1, rho1 = self.system.field_full(x1)
        v1 = v + 0.5 * dt * (e0 + e1)
        self.cache_time = t + dt
        self.cache_field = e1
        self.last_potential = phi1
        self.last_rho = rho1
        return x1, v1, t + dt


@dataclass
class History:
    rho: np.ndarray          # (steps+1, Nx, p)
    phi: np.ndarray          # (steps+1, Nx, p)
    electric: np.ndarray     # (steps+1, p)
    kinetic: np.ndarray      # (steps+1, p)
    x: np.ndarray
    v: np.ndarray


def run(system, x0, v0, dt, num_steps):
    """run_full_order (fullorder.py:169-226) at energy_stride = 1, no snapshots."""
    st = Stepper(system)
    x, v, t = np.array(x0, dtype=float), np.array(v0, dtype=float), 0.0
    e0, phi0, rho0 = system.field_full(x)
    st.cache_time, st.cache_field, st.last_potential, st.last_rho = t, e0, phi0, rho0
    rhos, phis, ees, kins = [], [], [], []

    def rec():
        rhos.append(np.atleast_2d(st.last_rho.T).T.copy())
        phis.append(np.atleast_2d(st.last_potential.T).T.copy())
        ees.append(np.atleast_1d(fe.electric_energy(system.poisson, st.last_potential,
                                                    system.charge)))
        kins.append(np.atleast_1d(0.5 * np.einsum("i...,i...->...", v, v)))

    rec()
    for _ in range(num_steps):
        x, v, t = st.step(x, v, t, dt)
        rec()
    return History(np.asarray(rhos), np.asarray(phis), np.asarray(ees), np.asarray(kins), x, v)
