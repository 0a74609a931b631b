"""Degree-2/3 oracle pinned by the reference's property tests ported to degree p.

Ports of /root/reference/pkg/tests/test_fem.py (partition of unity :59-65,
adjoint vs dense :68-79, gradient rows :82-89, batched == per-column :99-109,
translation equivariance :119-129, zero-mean solve vs pinv :132-140, gauge
:143-149, two-path Hamiltonian :152-167) and selftest.py:290-312 (force =
-grad energy by finite differences).
"""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import fe_bspline as fe

L, NX = 4.0, 16
DEG = [1, 2, 3]


@pytest.mark.parametrize("d", DEG)
@settings(max_examples=25, deadline=None)
@given(st.lists(st.floats(min_value=-10.0, max_value=10.0, allow_nan=False), min_size=1, max_size=30))
def test_partition_of_unity(d, pos):
    t = fe.eval_basis(fe.Mesh(L, NX, d), np.asarray(pos))
    np.testing.assert_allclose(t.matvec(np.ones(NX)), 1.0, atol=1e-14)
    gr = fe.eval_basis_grad(fe.Mesh(L, NX, d), np.asarray(pos))
    np.testing.assert_allclose(gr.matvec(np.ones(NX)), 0.0, atol=1e-12)


@pytest.mark.parametrize("d", DEG)
def test_adjoint_matches_dense(d):
    rng = np.random.default_rng(d)
    mesh = fe.Mesh(L, NX, d)
    for _ in range(10):
        x = rng.uniform(-L, 2 * L, 12)
        for t in (fe.eval_basis(mesh, x), fe.eval_basis_grad(mesh, x)):
            dense = t.toarray()
            w, phi = rng.standard_normal(12), rng.standard_normal(NX)
            np.testing.assert_allclose(t.matvec(phi), dense @ phi, atol=1e-12)
            np.testing.assert_allclose(t.rmatvec(w), dense.T @ w, atol=1e-12)


@pytest.mark.parametrize("d", DEG)
def test_gradient_is_derivative_of_value(d):
    rng = np.random.default_rng(10 + d)
    mesh = fe.Mesh(L, NX, d)
    x = rng.uniform(0, L, 40)
    phi = rng.standard_normal(NX)
    eps = 1e-6
    fd = (fe.eval_basis(mesh, x + eps).matvec(phi) - fe.eval_basis(mesh, x - eps).matvec(phi)) / (2 * eps)
    got = fe.eval_basis_grad(mesh, x).matvec(phi)
    if d == 1:   # P1 derivative is discontinuous at nodes; random x avoids them
        np.testing.assert_allclose(got, fd, atol=1e-5)
    else:
        np.testing.assert_allclose(got, fd, atol=1e-6)


@pytest.mark.parametrize("d", DEG)
def test_batched_equals_per_column_and_neutral(d):
    rng = np.random.default_rng(0)
    mesh = fe.Mesh(L, NX, d)
    charge = fe.Charge(200, L)
    x = rng.uniform(0, L, (200, 3))
    rho = fe.deposit_charge(fe.eval_basis(mesh, x), charge)
    np.testing.assert_allclose(rho.sum(axis=0), 0.0, atol=1e-12)
    for j in range(3):
        np.testing.assert_allclose(rho[:, j], fe.deposit_charge(fe.eval_basis(mesh, x[:, j]), charge),
                                   atol=1e-14)


@pytest.mark.parametrize("d", DEG)
def test_uniform_particles_zero_density(d):
    mesh = fe.Mesh(L, NX, d)
    charge = fe.Charge(4 * NX, L)
    x = np.arange(4 * NX) * (L / (4 * NX))
    np.testing.assert_allclose(fe.deposit_charge(fe.eval_basis(mesh, x), charge), 0.0, atol=1e-13)


@pytest.mark.parametrize("d", DEG)
def test_translation_equivariance(d):
    rng = np.random.default_rng(5)
    mesh = fe.Mesh(L, NX, d)
    x = rng.uniform(0, L, 120)
    charge = fe.Charge(120, L)
    poisson = fe.Poisson(mesh)
    rho = fe.deposit_charge(fe.eval_basis(mesh, x), charge)
    rho_s = fe.deposit_charge(fe.eval_basis(mesh, x + mesh.h), charge)
    np.testing.assert_allclose(np.roll(rho, 1), rho_s, atol=1e-12)
    np.testing.assert_allclose(np.roll(poisson.solve(rho), 1), poisson.solve(rho_s), atol=1e-12)


@pytest.mark.parametrize("d", DEG)
def test_zero_mean_solve_vs_pinv_and_gauge(d):
    rng = np.random.default_rng(1)
    mesh = fe.Mesh(L, NX, d)
    poisson = fe.Poisson(mesh)
    rho = rng.standard_normal(NX)
    phi = poisson.solve(rho)
    assert abs(phi.mean()) < 1e-13
    np.testing.assert_allclose(poisson.stiffness @ phi, rho - rho.mean(), atol=1e-10)
    ref = np.linalg.pinv(poisson.stiffness) @ (rho - rho.mean())
    np.testing.assert_allclose(phi, ref - ref.mean(), atol=1e-10)
    np.testing.assert_allclose(poisson.stiffness @ np.ones(NX), 0.0, atol=1e-12)
    charge = fe.Charge(200, L)
    e0 = fe.electric_energy(poisson, phi, charge)
    assert e0 >= 0 and fe.electric_energy(poisson, phi + 3.7, charge) == pytest.approx(e0, rel=1e-12)


@pytest.mark.parametrize("d", DEG)
def test_stiffness_is_exact_gram_of_derivatives(d):
    """L_ij = int lambda_i' lambda_j' dx by Gauss quadrature on every cell."""
    mesh = fe.Mesh(L, NX, d)
    gx, gw = np.polynomial.legendre.leggauss(8)
    dense = np.zeros((NX, NX))
    for c in range(NX):
        xs = (c + 0.5 * (gx + 1.0)) * mesh.h
        D = fe.eval_basis_grad(mesh, xs).toarray()
        dense += D.T @ (D * (0.5 * mesh.h * gw)[:, None])
    np.testing.assert_allclose(fe.stiffness_matrix(mesh), dense, atol=1e-12)


@pytest.mark.parametrize("d", DEG)
def test_hamiltonian_two_paths(d):
    mesh = fe.Mesh(L, NX, d)
    poisson = fe.Poisson(mesh)
    charge = fe.Charge(60, L)
    rng = np.random.default_rng(3)
    x, v = rng.uniform(0, L, 60), rng.standard_normal(60)
    lam = fe.eval_basis(mesh, x).toarray()
    q = lam.T @ np.full(60, charge.charge_weight)
    q = q - q.mean()
    h_ref = 0.5 * v @ v + 0.5 / charge.particle_mass * q @ np.linalg.pinv(poisson.stiffness) @ q
    assert fe.hamiltonian(x, v, poisson, charge) == pytest.approx(h_ref, rel=1e-12)


@pytest.mark.parametrize("d", DEG)
def test_force_is_minus_energy_gradient(d):
    """selftest.py:290-312 at degree d: E_k = -(1/m_p) dH_field/dx_k * ... by FD."""
    mesh = fe.Mesh(L, NX, d)
    poisson = fe.Poisson(mesh)
    n = 30
    charge = fe.Charge(n, L)
    rng = np.random.default_rng(8)
    x = rng.uniform(0, L, n)
    zero = np.zeros(n)
    b, gr = fe.eval_basis_pair(mesh, x)
    phi = poisson.solve(fe.deposit_charge(b, charge))
    e = fe.field_at_particles(gr, phi, charge)
    eps = 1e-6
    for k in range(0, n, 7):
        xp, xm = x.copy(), x.copy()
        xp[k] += eps
        xm[k] -= eps
        dh = (fe.hamiltonian(xp, zero, poisson, charge) - fe.hamiltonian(xm, zero, poisson, charge)) / (2 * eps)
        # H = sum 0.5 v^2 + E_field ; dv/dt = E = -dH/dx (unit mass per particle)
        assert e[k] == pytest.approx(-dh, rel=1e-5, abs=1e-8)
