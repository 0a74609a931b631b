"""GPU parity of the FE kernels against the CPU oracle (degrees 1-3).

Tolerances (BASELINE.json north_star): integer cell indices bit-exact; charge
and potential <= 1e-12 normwise relative per evaluation.  Degree-1 field and
value gathers keep the reference's operation order and are bit-exact given the
same potential.  Also ports the reference's own FE tests
(/root/reference/pkg/tests/test_fem.py) onto the GPU API.
"""

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import fe_bspline as fe

pytestmark = pytest.mark.gpu

RTOL = 1e-12
DEG = [1, 2, 3]


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def gfem(lib_built):
    from paper_2201_05555_b200 import fem
    return fem


def _inputs(rng, n, p, L, nx):
    x = rng.uniform(-2 * L, 3 * L, size=(n, p))
    h = L / nx
    x[0, 0] = 0.0
    x[1, -1] = 5 * h
    x[2, 0] = -3 * h
    x[3, -1] = np.nextafter(7 * h, 0)
    x[4, 0] = 1e12 * h
    return x


@pytest.mark.parametrize("d", DEG)
def test_locate_and_tables(gfem, d):
    rng = np.random.default_rng(d)
    L, nx = 4.0 * np.pi, 64
    x = _inputs(rng, 5000, 5, L, nx)
    om, gm = fe.Mesh(L, nx, d), gfem.build_mesh(L, nx, d)
    ob, og = fe.eval_basis_pair(om, x)
    gb, gg = gfem.eval_basis_pair(gm, x)
    np.testing.assert_array_equal(gb.i0, ob.i0)
    for m in range(d + 1):
        if d == 1:
            np.testing.assert_array_equal(gb.weights[m], ob.w[m])
            np.testing.assert_array_equal(gg.weights[m], og.w[m])
        else:
            np.testing.assert_allclose(gb.weights[m], ob.w[m], rtol=0, atol=1e-15)
            np.testing.assert_allclose(gg.weights[m], og.w[m], rtol=0, atol=1e-15 / om.h)


def test_locate_division_is_ieee(lib_built):
    """The device x/h (Markstein correction with RN(1/h)) equals IEEE division:
    frac = s - floor(s) is exact, so bitwise-equal frac means bitwise-equal s."""
    import torch
    from paper_2201_05555_b200 import _device as dev
    from paper_2201_05555_b200 import _lib
    rng = np.random.default_rng(0)
    for L, nx in ((4 * np.pi, 64), (10 * np.pi, 128), (2 * np.pi / 0.3, 512), (1.0, 3), (7.77, 100)):
        h = L / nx
        parts = [rng.uniform(-3 * L, 3 * L, 2_000_000),
                 rng.integers(-10 * nx, 10 * nx, 200_000) * h,
                 np.nextafter(rng.integers(-10 * nx, 10 * nx, 200_000) * h, np.inf),
                 np.nextafter(rng.integers(-10 * nx, 10 * nx, 200_000) * h, -np.inf),
                 rng.uniform(-1e6, 1e6, 200_000), rng.standard_normal(200_000) * 1e-300,
                 # around the fast path's |x/h| < 2^31 - 1 limit and the +-0 / tiny edges
                 np.array([2.0**31 - 1, 2.0**31 - 1.5, 2.0**31, 2.0**31 + 7, -(2.0**31),
                           -(2.0**31) + 1, -(2.0**31) - 3, 0.5, -0.5]) * h,
                 np.array([2.0**51 - 1, 2.0**51 - 0.5, 2.0**51, 2.0**51 + 2, -(2.0**51),
                           -(2.0**51) + 1, -(2.0**51) - 2, 2.0**52 + 6, 2.0**60]) * h,
                 np.array([0.0, -0.0, 5e-324, -5e-324, 1e-280, -1e-280, 2.0**-800, 2.0**-801,
                           -(2.0**-800), 3.0 * 2.0**-801, 1e300, -1e300])]
        x = np.concatenate(parts)
        xd = torch.from_numpy(x).cuda().reshape(1, -1)
        n = x.size
        i0 = torch.empty((1, n), dtype=torch.int64, device="cuda")
        fr = torch.empty((1, n), dtype=torch.float64, device="cuda")
        st = dev.new_status()
        inst = dev.inst_rows(gfem_mesh(L, nx), gfem_charge(L), 1)
        _lib.call("picrom_locate", xd.data_ptr(), n, 1, n, inst.data_ptr(), nx, i0.data_ptr(),
                  fr.data_ptr(), n, st.data_ptr(), dev.stream_handle())
        s = x / h
        np.testing.assert_array_equal(fr.cpu().numpy()[0], s - np.floor(s))
        np.testing.assert_array_equal(i0.cpu().numpy()[0], np.floor(s).astype(np.int64) % nx)


def gfem_mesh(L, nx):
    from paper_2201_05555_b200 import fem
    return fem.build_mesh(L, nx)


def gfem_charge(L):
    from paper_2201_05555_b200 import fem
    return fem.ChargeConfig(1000, L)


def test_golden_p1_end_to_end(gfem):
    g = np.load(GOLDEN / "fem_p1.npz")
    L, nx = float(g["length"]), int(g["nx"])
    mesh = gfem.build_mesh(L, nx)
    x2 = g["x2"]
    charge = gfem.ChargeConfig(num_particles=x2.shape[0], length=L)
    poisson = gfem.PoissonOperator(mesh)
    np.testing.assert_array_equal(poisson.stiffness, g["stiffness"])
    b, gr = gfem.eval_basis_pair(mesh, x2)
    np.testing.assert_array_equal(b.i0, g["i0"])
    rho = gfem.deposit_charge(b, charge)
    assert rel(rho, g["rho2"]) <= RTOL
    phi = poisson.solve(g["rho2"])
    assert rel(phi, g["phi2"]) <= RTOL
    # teacher-forced gathers are bit-exact at degree 1 (reference operation order)
    np.testing.assert_array_equal(gfem.field_at_particles(gr, g["phi2"], charge), g["e2"])
    np.testing.assert_array_equal(b.matvec(g["phi2"]), g["lam2"])
    assert rel(gfem.electric_energy(poisson, g["phi2"], charge), g["ee2"]) <= RTOL
    assert rel(b.rmatvec(g["y"]), g["rmat2"]) <= RTOL
    assert rel(gfem.hamiltonian(x2, g["v2"], poisson, charge), g["ham2"]) <= RTOL


@pytest.mark.parametrize("d", DEG)
@pytest.mark.parametrize("n,p,nx", [(3000, 4, 16), (250_000, 2, 128), (40_000, 3, 512)])
def test_deposit_solve_field_vs_oracle(gfem, d, n, p, nx):
    rng = np.random.default_rng(n + d)
    L = 10.0 * np.pi
    x = rng.uniform(0, L, size=(n, p))
    om, gm = fe.Mesh(L, nx, d), gfem.build_mesh(L, nx, d)
    oc, gc = fe.Charge(n, L), gfem.ChargeConfig(n, L)
    ob, og = fe.eval_basis_pair(om, x)
    orho = fe.deposit_charge(ob, oc)
    gb, gg = gfem.eval_basis_pair(gm, x)
    grho = gfem.deposit_charge(gb, gc)
    # normwise on rho and, stricter, against the particle term qw*Lambda^T 1
    assert rel(grho, orho) <= RTOL
    assert np.linalg.norm(grho - orho) / (abs(oc.charge_weight) * n / nx * np.sqrt(nx * p)) < 1e-14
    op, gp = fe.Poisson(om), gfem.PoissonOperator(gm)
    ophi = op.solve(orho)
    gphi = gp.solve(orho)                    # teacher-forced: same rho
    assert rel(gphi, ophi) <= RTOL
    assert rel(gp.solve(grho), ophi) <= RTOL
    assert rel(gfem.electric_energy(gp, ophi, gc), fe.electric_energy(op, ophi, oc)) <= RTOL
    oe = fe.field_at_particles(og, ophi, oc)
    ge = gfem.field_at_particles(gg, ophi, gc)
    if d == 1:
        np.testing.assert_array_equal(ge, oe)
    else:
        assert rel(ge, oe) <= 1e-13
    assert rel(gb.matvec(ophi), ob.matvec(ophi)) <= 1e-14


@pytest.mark.parametrize("d", DEG)
def test_reference_fem_properties_on_gpu(gfem, d):
    """test_fem.py:59-149 properties, through the GPU API."""
    L, nx = 4.0, 8 if d == 1 else 16
    mesh = gfem.build_mesh(L, nx, d)
    rng = np.random.default_rng(7)
    x = rng.uniform(-10, 10, 30)
    np.testing.assert_allclose(gfem.eval_basis(mesh, x).matvec(np.ones(nx)), 1.0, atol=1e-14)
    t = gfem.eval_basis(mesh, x[:12])
    dense = t.toarray()
    w, phi = rng.standard_normal(12), rng.standard_normal(nx)
    np.testing.assert_allclose(t.matvec(phi), dense @ phi, atol=1e-13)
    np.testing.assert_allclose(t.rmatvec(w), dense.T @ w, atol=1e-13)
    charge = gfem.ChargeConfig(4 * nx, L)
    xu = np.arange(4 * nx) * (L / (4 * nx))
    np.testing.assert_allclose(gfem.deposit_charge(gfem.eval_basis(mesh, xu), charge), 0.0, atol=1e-13)
    poisson = gfem.PoissonOperator(mesh)
    rho = rng.standard_normal(nx)
    ph = poisson.solve(rho)
    assert abs(ph.mean()) < 1e-13
    np.testing.assert_allclose(poisson.stiffness @ ph, rho - rho.mean(), atol=1e-10)
    x120 = rng.uniform(0, L, 120)
    c120 = gfem.ChargeConfig(120, L)
    r0 = gfem.deposit_charge(gfem.eval_basis(mesh, x120), c120)
    r1 = gfem.deposit_charge(gfem.eval_basis(mesh, x120 + mesh.h), c120)
    np.testing.assert_allclose(np.roll(r0, 1), r1, atol=1e-12)
    e0 = gfem.electric_energy(poisson, ph, charge)
    assert e0 >= 0 and gfem.electric_energy(poisson, ph + 3.7, charge) == pytest.approx(e0, rel=1e-12)


def test_nonfinite_position_raises_with_index(gfem):
    from paper_2201_05555_b200.errors import EvaluationError
    mesh = gfem.build_mesh(4.0, 8)
    x = np.zeros((5, 2))
    x[3, 1] = np.nan
    x[4, 0] = np.inf
    with pytest.raises(EvaluationError) as err:
        gfem.eval_basis(mesh, x)
    assert err.value.index == (3, 1)


def test_deposit_is_deterministic(gfem):
    rng = np.random.default_rng(3)
    mesh = gfem.build_mesh(10.0, 128, 3)
    x = rng.uniform(0, 10.0, size=(300_000, 3))
    c = gfem.ChargeConfig(300_000, 10.0)
    r1 = gfem.deposit_charge(gfem.eval_basis(mesh, x), c)
    r2 = gfem.deposit_charge(gfem.eval_basis(mesh, x), c)
    np.testing.assert_array_equal(r1, r2)


def test_torch_inputs_stay_on_device(gfem):
    import torch
    mesh = gfem.build_mesh(4.0, 16, 2)
    x = torch.rand(1000, 3, dtype=torch.float64, device="cuda") * 4.0
    c = gfem.ChargeConfig(1000, 4.0)
    rho = gfem.deposit_charge(gfem.eval_basis(mesh, x), c)
    assert isinstance(rho, torch.Tensor) and rho.is_cuda and rho.shape == (16, 3)
    ref = fe.deposit_charge(fe.eval_basis(fe.Mesh(4.0, 16, 2), x.cpu().numpy()), fe.Charge(1000, 4.0))
    assert rel(rho.cpu().numpy(), ref) <= RTOL
