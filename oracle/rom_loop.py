"""ORACLE (test infrastructure only): reduced-order main loop.

Restates /root/reference/pkg/src/picrom/driver.py:63-274 (exact_gradients,
make_full_stage, run_reduced) on top of oracle.manifold / oracle.dmd_deim,
extended to per-instance meshes (BASELINE C3/C4 draw a wavenumber k per
instance, hence a length L_j = 2 pi / k_j, mesh width h_j, charge weight and
particle mass per column).  With a single length the
batched reference code path is used verbatim (bit-identical at degree 1,
pinned by tests/golden/rom_p1.npz); with several lengths each column is
evaluated against its own mesh (column-independent arithmetic, so the batched
and per-column forms agree bit for bit where they overlap).
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field

import numpy as np

from . import dmd_deim as dd
from . import fe_bspline as fe
from . import manifold as mf


class ParamSystem:
    """Per-column meshes/charges; ``single`` when all columns share one length."""

    def __init__(self, lengths, num_cells, degree, num_particles):
        self.lengths = np.asarray(lengths, dtype=float).reshape(-1)
        self.num_cells, self.degree, self.num_particles = num_cells, degree, num_particles
        self._by_len = {}
        for L in np.unique(self.lengths):
            mesh = fe.Mesh(float(L), num_cells, degree)
            self._by_len[float(L)] = (mesh, fe.Charge(num_particles, float(L)), fe.Poisson(mesh))
        self.single = len(self._by_len) == 1

    def column(self, j):
        return self._by_len[float(self.lengths[j])]

    @property
    def mesh(self):
        return self.column(0)[0]

    @property
    def charge(self):
        return self.column(0)[1]

    @property
    def poisson(self):
        return self.column(0)[2]


def exact_gradients(system, u, z, cols=None):
    """(G (2N, p'), phi (Nx, p'), lam (N, p')) at the reconstructed columns U z
    (driver.py:63-76); ``cols`` names the instances of z's columns."""
    xr, vr = mf.split_reconstruct(u, z)
    cols = np.arange(z.shape[1]) if cols is None else np.asarray(cols)
    if system.single:
        mesh, charge, poisson = system.column(0)
        basis, grad = fe.eval_basis_pair(mesh, xr)
        phi = poisson.solve(fe.deposit_charge(basis, charge))
        coef = charge.charge_weight / charge.particle_mass
        g = np.concatenate([coef * grad.matvec(phi), vr], axis=0)
        return g, phi, basis.matvec(phi)
    top = np.empty_like(xr)
    lam = np.empty_like(xr)
    phi = np.empty((system.num_cells, z.shape[1]))
    for c, j in enumerate(cols):
        mesh, charge, poisson = system.column(j)
        basis, grad = fe.eval_basis_pair(mesh, xr[:, c])
        ph = poisson.solve(fe.deposit_charge(basis, charge))
        coef = charge.charge_weight / charge.particle_mass
        top[:, c] = coef * grad.matvec(ph)
        lam[:, c] = basis.matvec(ph)
        phi[:, c] = ph
    return np.concatenate([top, vr], axis=0), phi, lam


def full_stage(system):
    """Warm-up coefficient gradient U_mid^T F(U_mid z) over all columns (driver.py:79-89)."""

    def factory(u_mid):
        def g(z):
            return u_mid.T @ exact_gradients(system, u_mid, z)[0]
        return g

    return factory


def hyper_stage(system, dmd, deim, t_stage, params):
    """make_hyper_stage (hyper.py:299-332) with per-column mesh/mass."""
    if system.single:
        return dd.hyper_stage(dmd, deim, t_stage, system.mesh, system.charge.particle_mass, params)
    qw_ref = system.charge.charge_weight

    def factory(u_mid):
        half = u_mid.shape[0] // 2
        ux_d = u_mid[deim.indices, :]
        uv = u_mid[half:]
        gram_v = uv.T @ uv
        cache = {}

        def g(z):
            phi = cache.get("phi")
            if phi is None:
                dmd.ensure_coords(params)
                phi = cache["phi"] = dmd.potential(t_stage)
            xd = ux_d @ z
            out = gram_v @ z
            for j in range(z.shape[1]):
                mesh, charge, _ = system.column(j)
                w = deim.weights * (charge.charge_weight / qw_ref)
                dphi = fe.eval_basis_grad(mesh, xd[:, j]).matvec(phi[:, j])
                out[:, j] += (1.0 / charge.particle_mass) * (ux_d.T @ (dphi * w))
            return out

        return g

    return factory


def hyper_energy(system, dmd, deim, u, z, t, params):
    """hyper_hamiltonian (hyper.py:280-296) with per-column mesh / mass and the
    hyper stage's per-column weight rescaling."""
    if system.single:
        mesh, charge, _ = system.column(0)
        dmd.ensure_coords(params)
        return dd.hyper_energy(dmd, deim, u, z, t, mesh, charge.particle_mass)
    half = u.shape[0] // 2
    ux_d = u[deim.indices, :]
    uv = u[half:]
    kin = 0.5 * np.einsum("ij,ij->j", z, (uv.T @ uv) @ z)
    dmd.ensure_coords(params)
    phi = dmd.potential(t)
    xd = ux_d @ z
    qw_ref = system.charge.charge_weight
    fld = np.empty(z.shape[1])
    for j in range(z.shape[1]):
        mesh, charge, _ = system.column(j)
        lam = fe.eval_basis(mesh, xd[:, j]).matvec(phi[:, j])
        w = deim.weights * (charge.charge_weight / qw_ref)
        fld[j] = (0.5 / charge.particle_mass) * (w @ lam)
    return kin + fld


@dataclass
class RomHistory:
    u: np.ndarray
    z: np.ndarray
    energy_times: list = field(default_factory=list)
    electric: list = field(default_factory=list)
    kinetic: list = field(default_factory=list)
    ortho: list = field(default_factory=list)
    sympl: list = field(default_factory=list)
    fp_iterations: list = field(default_factory=list)
    dmd_ranks: list = field(default_factory=list)
    s_conds: list = field(default_factory=list)
    deim_indices: list = field(default_factory=list)
    sub: np.ndarray = None
    bases: list = field(default_factory=list)
    hyper_engaged: bool = False
    decomp_times: list = field(default_factory=list)
    dh_total: list = field(default_factory=list)
    dh_coeff: list = field(default_factory=list)
    dh_coeff_dd: list = field(default_factory=list)


def _energies(system, u, z):
    xr, vr = mf.split_reconstruct(u, z)
    kin = 0.5 * np.einsum("ij,ij->j", vr, vr)
    if system.single:
        mesh, charge, poisson = system.column(0)
        basis, _ = fe.eval_basis_pair(mesh, xr)
        phi = poisson.solve(fe.deposit_charge(basis, charge))
        return np.atleast_1d(fe.electric_energy(poisson, phi, charge)), kin
    ee = np.empty(z.shape[1])
    for j in range(z.shape[1]):
        mesh, charge, poisson = system.column(j)
        phi = poisson.solve(fe.deposit_charge(fe.eval_basis(mesh, xr[:, j]), charge))
        ee[j] = fe.electric_energy(poisson, phi, charge)
    return ee, kin


def run_reduced(system, params, x0, v0, *, basis_dim, subsample, window, deim_dim, deim_period,
                deim_update, dt, num_steps, svd_tol_dmd=1e-5, fp_tol=1e-9, fp_max_iter=100,
                hyper_reduction=True, energy_stride=10, snapshot_stride=None, u0=None, z0=None,
                decomp_stride=None):
    """Algorithm-2 loop (driver.py:117-274); the Hamiltonian-error
    decomposition (driver.py:229-246) at `decomp_stride` when given."""
    params = np.asarray(params, dtype=float)
    snap = max(1, int(snapshot_stride)) if snapshot_stride else max(1, num_steps // 40)
    if u0 is None:
        u, z = mf.csvd_basis(x0, v0, basis_dim)
    else:
        u, z = u0, z0
    sub = np.sort(mf.farthest_point_subset(z, subsample))
    pots = deque(maxlen=window + 1)
    lams = deque(maxlen=window + 1)
    dmd = deim = None
    counter = 0
    hist = RomHistory(u=u, z=z, sub=sub)
    fstage = full_stage(system)

    def grad_sub(u_eval, z_sub):
        return exact_gradients(system, u_eval, z_sub, sub)[0]

    def diag(tau, uu, zz):
        if tau % energy_stride == 0 or tau == num_steps:
            ee, kin = _energies(system, uu, zz)
            hist.energy_times.append(tau * dt)
            hist.electric.append(ee)
            hist.kinetic.append(kin)
        if tau % snap == 0 or tau == num_steps:
            hist.bases.append((tau * dt, uu.copy(), zz.copy()))

    o, s = mf.structure_defects(u)
    hist.ortho.append(o)
    hist.sympl.append(s)
    diag(0, u, z)
    for tau in range(1, num_steps + 1):
        t_prev = (tau - 1) * dt
        g0, phi_sub, lam_sub = exact_gradients(system, u, z[:, sub], sub)
        pots.append(phi_sub)
        lams.append(lam_sub)
        hyper_now = hyper_reduction and len(pots) == window + 1
        if hyper_now:
            hist.hyper_engaged = True
            dmd = dd.parametric_dmd(list(pots), dt, t_prev, params, sub, svd_tol=svd_tol_dmd)
            block = np.stack(lams).transpose(1, 2, 0)
            deim = dd.deim_fit(block.reshape(block.shape[0], -1), deim_dim,
                               system.charge.charge_weight, prev=deim,
                               full=(counter % deim_period == 0), n_update=deim_update)
            counter += 1
            stage = hyper_stage(system, dmd, deim, t_prev + 0.5 * dt, params)
            hist.deim_indices.append(deim.indices.copy())
            hist.dmd_ranks.append(dmd.rank)
        else:
            stage = fstage
        res = mf.prk2(u, z, dt, sub, grad_sub, g0, stage, fp_tol=fp_tol, fp_max_iter=fp_max_iter)
        u_prev, z_prev = u, z
        u, z = res.u, res.z
        if hyper_now and decomp_stride and tau % decomp_stride == 0:
            def ham(uu, zz):
                ee, kin = _energies(system, uu, zz)
                return kin + ee
            h_new, h_prev = ham(u, z), ham(u_prev, z_prev)
            hm_new, hm_prev = ham(res.u_mid, z), ham(res.u_mid, z_prev)
            hd_new = hyper_energy(system, dmd, deim, res.u_mid, z, tau * dt, params)
            hd_prev = hyper_energy(system, dmd, deim, res.u_mid, z_prev, t_prev, params)
            hist.decomp_times.append(tau * dt)
            hist.dh_total.append(float(np.linalg.norm(np.atleast_1d(h_new - h_prev))))
            hist.dh_coeff.append(float(np.linalg.norm(np.atleast_1d(hm_new - hm_prev))))
            hist.dh_coeff_dd.append(float(np.linalg.norm(np.atleast_1d(hd_new - hd_prev))))
        o, s = mf.structure_defects(u)
        hist.ortho.append(o)
        hist.sympl.append(s)
        hist.fp_iterations.append(res.fp_iterations)
        hist.s_conds.append(res.s_cond)
        diag(tau, u, z)
    hist.u, hist.z = u, z
    return hist
