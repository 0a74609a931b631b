"""The CPU oracle at degree 1 reproduces the reference's own outputs bit for bit.

Golden vectors: tests/golden/*.npz, produced by tests/golden/make_golden.py
running /root/reference/pkg/src/picrom.  This pins the oracle before it is
trusted as the checker for the GPU path (and for degree 2/3 by extension).
"""

import numpy as np
import pytest

from conftest import GOLDEN, REFERENCE_SRC
from oracle import fe_bspline as fe
from oracle import pic_loop


@pytest.fixture(scope="module")
def g():
    return np.load(GOLDEN / "fem_p1.npz")


def test_locate_bit_exact(g):
    mesh = fe.Mesh(float(g["length"]), int(g["nx"]), 1)
    i0, frac = fe.locate(mesh, g["x2"])
    assert i0.dtype == np.int64
    np.testing.assert_array_equal(i0, g["i0"])
    np.testing.assert_array_equal(frac, g["frac"])


def test_tables_bit_exact(g):
    mesh = fe.Mesh(float(g["length"]), int(g["nx"]), 1)
    b, gr = fe.eval_basis_pair(mesh, g["x2"])
    for got, key in ((b.w0, "w0"), (b.w1, "w1"), (gr.w0, "gw0"), (gr.w1, "gw1")):
        np.testing.assert_array_equal(got, g[key])


def test_deposit_solve_field_energy_bit_exact(g):
    L, nx = float(g["length"]), int(g["nx"])
    mesh = fe.Mesh(L, nx, 1)
    x2 = g["x2"]
    charge = fe.Charge(num_particles=x2.shape[0], length=L)
    poisson = fe.Poisson(mesh)
    np.testing.assert_array_equal(poisson.stiffness, g["stiffness"])
    b, gr = fe.eval_basis_pair(mesh, x2)
    rho = fe.deposit_charge(b, charge)
    np.testing.assert_array_equal(rho, g["rho2"])
    phi = poisson.solve(rho)
    np.testing.assert_array_equal(phi, g["phi2"])
    np.testing.assert_array_equal(fe.electric_energy(poisson, phi, charge), g["ee2"])
    np.testing.assert_array_equal(fe.field_at_particles(gr, phi, charge), g["e2"])
    np.testing.assert_array_equal(b.matvec(phi), g["lam2"])
    np.testing.assert_array_equal(b.rmatvec(g["y"]), g["rmat2"])
    rho1 = fe.deposit_charge(fe.eval_basis(mesh, g["x1"]), charge)
    np.testing.assert_array_equal(rho1, g["rho1"])
    np.testing.assert_array_equal(poisson.solve(rho1), g["phi1"])
    np.testing.assert_array_equal(fe.hamiltonian(x2, g["v2"], poisson, charge), g["ham2"])


def test_verlet_and_run_bit_exact():
    f = np.load(GOLDEN / "fullorder_p1.npz")
    L, nx = float(f["length"]), int(f["nx"])
    mesh = fe.Mesh(L, nx, 1)
    charge = fe.Charge(num_particles=f["x"].shape[0], length=L)
    sysm = pic_loop.System(mesh, charge)
    st = pic_loop.Stepper(sysm)
    x1, v1, t1 = st.step(f["x"], f["v"], 0.0, 0.1)
    x2, v2, t2 = st.step(x1, v1, t1, 0.1)
    np.testing.assert_array_equal(x1, f["x_step1"])
    np.testing.assert_array_equal(v1, f["v_step1"])
    np.testing.assert_array_equal(x2, f["x_step2"])
    np.testing.assert_array_equal(v2, f["v_step2"])
    np.testing.assert_array_equal(st.last_potential, f["phi_step2"])
    hist = pic_loop.run(sysm, f["x"], f["v"], 0.05, 20)
    np.testing.assert_array_equal(hist.electric, f["rec_energy"])
    np.testing.assert_array_equal(hist.electric + hist.kinetic, f["rec_ham"])
    np.testing.assert_array_equal(hist.phi, f["rec_pot"])
    np.testing.assert_array_equal(hist.x, f["rec_snap_x"][-1])
    np.testing.assert_array_equal(hist.v, f["rec_snap_v"][-1])


@pytest.mark.skipif(not REFERENCE_SRC.exists(), reason="reference tree absent (GPU box)")
def test_oracle_matches_live_reference_random():
    """Live cross-check on fresh random inputs (only where /root/reference exists)."""
    import sys
    sys.path.insert(0, str(REFERENCE_SRC))
    from picrom import fem as rfem
    rng = np.random.default_rng(99)
    for nx in (3, 8, 33):
        L = float(rng.uniform(1, 20))
        x = rng.uniform(-3 * L, 3 * L, size=(101, 4))
        rm, om = rfem.build_mesh(L, nx), fe.Mesh(L, nx, 1)
        rc, oc = rfem.ChargeConfig(101, L), fe.Charge(101, L)
        rb, rg = rfem.eval_basis_pair(rm, x)
        ob, og = fe.eval_basis_pair(om, x)
        np.testing.assert_array_equal(rb.i0, ob.i0)
        rrho, orho = rfem.deposit_charge(rb, rc), fe.deposit_charge(ob, oc)
        np.testing.assert_array_equal(rrho, orho)
        rphi = rfem.PoissonOperator(rm).solve(rrho)
        np.testing.assert_array_equal(rphi, fe.Poisson(om).solve(orho))
        np.testing.assert_array_equal(rfem.field_at_particles(rg, rphi, rc),
                                      fe.field_at_particles(og, rphi, oc))
