"""GPU reduced-basis path vs the reference golden runs and the CPU oracle.

* building blocks (basis_velocity / retraction / tangent_velocity / residuals)
  against the reference's own outputs (tests/golden/rom_p1.npz);
* exact_gradients and the warm-up stage vs the oracle at degrees 1-3, single
  mesh and per-instance meshes (BASELINE C3/C4), 1e-12;
* run_reduced (no hyper-reduction) vs the reference golden run (degree 1) and
  vs the oracle with per-instance meshes (degree 2);
* DEIM: greedy indices bit-exact given the oracle's basis, DMD extrapolation,
  DEIM-sampled stage gradient, and a short hyper-reduced run.
"""

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import dmd_deim as odd
from oracle import fe_bspline as ofe
from oracle import manifold as omf
from oracle import rom_loop as orl

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def m(lib_built):
    from paper_2201_05555_b200 import driver, fem, fullorder, hyper, reduction
    return type("M", (), dict(driver=driver, fem=fem, fullorder=fullorder, hyper=hyper,
                              red=reduction))


@pytest.fixture(scope="module")
def g():
    return np.load(GOLDEN / "rom_p1.npz")


def test_building_blocks_vs_reference(m, g):
    u, z = g["bb_u"], g["bb_z"]
    xi = m.red.basis_velocity(u, z, g["bb_g"])
    assert rel(xi, g["bb_xi"]) <= 1e-12
    r = m.red.retraction(u, 0.1 * g["bb_xi"])
    assert rel(r, g["bb_r"]) <= 1e-13
    t = m.red.tangent_velocity(u, 0.1 * g["bb_xi"], g["bb_r"], g["bb_xe"])
    assert rel(t, g["bb_tan"]) <= 1e-12
    o, s = m.red.orthosymplectic_residuals(g["bb_r"])
    oo, os_ = omf.structure_defects(g["bb_r"])
    assert abs(o - oo) < 1e-14 and abs(s - os_) < 1e-14
    np.testing.assert_array_equal(m.red.SMatrix(z).matrix, g["bb_s"])
    np.testing.assert_array_equal(m.red.select_parameter_subset(z, 5), g["bb_sub"])


def _setup(m, d, per_instance, n=3000, p=6, nx=32, nb=4, seed=0):
    rng = np.random.default_rng(seed)
    ks = rng.uniform(0.4, 0.6, p) if per_instance else np.full(p, 0.5)
    lengths = 2 * np.pi / ks
    x0 = np.stack([rng.uniform(0, L, n) for L in lengths], axis=1)
    v0 = rng.standard_normal((n, p))
    u, z = omf.csvd_basis(x0, v0, nb)
    osys = orl.ParamSystem(lengths, nx, d, n)
    gsys = m.driver.ParametricVlasovSystem(lengths, nx, d, n)
    return u, z, osys, gsys, x0, v0, lengths


@pytest.mark.parametrize("d", [1, 2, 3])
@pytest.mark.parametrize("per_instance", [False, True])
def test_exact_gradients_vs_oracle(m, d, per_instance):
    u, z, osys, gsys, *_ = _setup(m, d, per_instance)
    og, ophi, olam = orl.exact_gradients(osys, u, z)
    gg, gphi, glam = m.driver.exact_gradients(gsys, u, z)
    assert rel(gphi, ophi) <= 1e-12
    assert rel(gg, og) <= 1e-12
    assert rel(glam, olam) <= 1e-12
    # warm-up stage g(z) = U^T F(U z)
    o_stage = orl.full_stage(osys)(u)(z)
    import torch
    g_stage = m.driver.make_full_stage(gsys)(torch.from_numpy(u).cuda())(z)
    assert rel(g_stage, o_stage) <= 1e-12


@pytest.mark.parametrize("p", [20, 33, 70, 130])
def test_exact_gradients_column_tilings(m, p):
    """The F-evaluation kernels pick their CTA shape from the column count: 4-warp
    / 32-column CTAs for p' <= 32 (the hyper-reduced subsample), 16-warp deposit
    and 8-warp gather CTAs above, with partly filled and multiple column tiles;
    full and ragged row tiles (N not a multiple of 64)."""
    u, z, osys, gsys, *_ = _setup(m, 2, True, n=2500, p=p, nx=32, nb=8, seed=p)
    og, ophi, olam = orl.exact_gradients(osys, u, z)
    gg, gphi, glam = m.driver.exact_gradients(gsys, u, z)
    assert rel(gphi, ophi) <= 1e-12
    assert rel(gg, og) <= 1e-12
    assert rel(glam, olam) <= 1e-12


def test_reduced_run_no_hyper_vs_reference(m, g):
    L, nx = float(g["length"]), int(g["nx"])
    mesh = m.fem.build_mesh(L, nx)
    sysm = m.fullorder.VlasovSystem(mesh, m.fem.ChargeConfig(g["a_x0"].shape[0], L))
    rec = m.driver.run_reduced(sysm, g["a_params"], g["a_x0"], g["a_v0"], basis_dim=4, subsample=4,
                               window=3, deim_dim=8, deim_period=3, deim_update=2, dt=0.02,
                               t_final=0.1, hyper_reduction=False, snapshot_stride=5,
                               energy_stride=1, decomp_stride=10**9)
    u, z = rec.bases[-1]
    np.testing.assert_allclose(u.cpu().numpy(), g["nohyper_u"], atol=1e-12)
    np.testing.assert_allclose(z, g["nohyper_z"], atol=1e-12)
    assert np.max(np.abs(rec.electric_energy - g["nohyper_ee"]) / np.abs(g["nohyper_ee"])) <= 1e-9
    np.testing.assert_array_equal(rec.fp_iterations, g["nohyper_fp"])


def test_reduced_run_per_instance_vs_oracle(m):
    """C3-like: per-instance wavenumbers, quadratic splines, no hyper-reduction."""
    u, z, osys, gsys, x0, v0, lengths = _setup(m, 2, True, n=4000, p=8, nx=32, nb=4, seed=3)
    params = np.stack([2 * np.pi / lengths, np.linspace(0.01, 0.1, 8)], axis=1)
    kw = dict(basis_dim=4, subsample=8, window=3, deim_dim=8, deim_period=3, deim_update=2,
              dt=0.05)
    h = orl.run_reduced(osys, params, x0, v0, num_steps=6, hyper_reduction=False,
                        energy_stride=1, **kw)
    rec = m.driver.run_reduced(gsys, params, x0, v0, t_final=0.3, hyper_reduction=False,
                               energy_stride=1, decomp_stride=10**9, **kw)
    u_g, z_g = rec.bases[-1]
    assert rel(u_g.cpu().numpy(), h.u) <= 1e-11
    assert rel(z_g, h.z) <= 1e-11
    ee_o = np.asarray(h.electric)
    assert np.max(np.abs(rec.electric_energy - ee_o) / np.abs(ee_o)) <= 1e-9
    np.testing.assert_array_equal(rec.fp_iterations, np.asarray(h.fp_iterations))


def test_deim_greedy_bit_exact_given_basis(m):
    rng = np.random.default_rng(11)
    psi = np.linalg.qr(rng.standard_normal((20000, 12)))[0]
    want = odd.greedy_indices(psi)
    got = m.hyper.deim_greedy(psi)
    np.testing.assert_array_equal(got, want)
    keep = {0: int(want[0]), 3: int(want[3]), 7: int(want[7])}
    np.testing.assert_array_equal(m.hyper.deim_greedy(psi, keep=dict(keep)),
                                  odd.greedy_indices(psi, keep=dict(keep)))


def test_deim_fit_well_separated_window_matches_lapack_svd(m):
    """fit_deim on a window with separated singular values (decay 10^-0.1 per
    index over 6 decades, the shape of C4's harvested window): indices equal and
    weights within 1e-12 of the oracle's direct LAPACK SVD (hyper.py:262-276)."""
    rng = np.random.default_rng(21)
    rows, cols, dim = 6000, 60, 12
    left = np.linalg.qr(rng.standard_normal((rows, cols)))[0]
    right = np.linalg.qr(rng.standard_normal((cols, cols)))[0]
    samples = (left * np.logspace(0, -6, cols)) @ right.T
    ch = m.fem.ChargeConfig(rows, 2 * np.pi)
    want = odd.deim_fit(samples, dim, ch.charge_weight)
    dm = m.hyper.fit_deim(samples, dim, ch)
    np.testing.assert_array_equal(dm.indices, want.indices)
    np.testing.assert_allclose(dm.weights, want.weights, rtol=1e-12, atol=1e-13 * np.abs(want.weights).max())
    s = np.linalg.svd(dm.psi.cpu().numpy().T @ want.psi, compute_uv=False)
    assert np.min(s) > 1 - 1e-12


def test_deim_fit_and_golden(m, g):
    ch = m.fem.ChargeConfig(80, 2 * np.pi)
    dm = m.hyper.fit_deim(g["de_samples"], 10, ch)
    np.testing.assert_array_equal(dm.indices, g["de_idx"])
    # this golden window is 4 modes + white noise: sigma_10 / sigma_11 = 1.01, so the
    # 10-dimensional subspace (and the weights, a function of span(Psi) only) is
    # ill-conditioned -- any SVD's answer moves by ~eps / gap; the well-separated
    # case below holds 1e-12
    np.testing.assert_allclose(dm.weights, g["de_w"], rtol=1e-8, atol=1e-12)
    # span agreement with the reference basis (principal angles)
    s = np.linalg.svd(dm.psi.cpu().numpy().T @ g["de_psi"], compute_uv=False)
    assert np.min(s) > 1 - 1e-10


def test_dmd_device_extrapolation_matches_host(m, g):
    model = m.hyper.fit_parametric_dmd(list(g["dmd_win"]), 0.05, 0.4, g["dmd_prm"],
                                       np.array([1, 3, 5]))
    model.ensure_coords(g["dmd_prm"])
    np.testing.assert_array_equal(model.eigenvalues, g["dmd_eigs"])
    host = model.potential(0.45)
    assert rel(host, g["dmd_phi"]) <= 1e-14
    devv = model.potential_device(0.45).cpu().numpy().T
    assert rel(devv, g["dmd_phi"]) <= 1e-13


def test_hyper_stage_vs_oracle(m):
    u, z, osys, gsys, x0, v0, lengths = _setup(m, 2, True, n=3000, p=6, nx=32, nb=4, seed=5)
    rng = np.random.default_rng(1)
    idx = rng.choice(3000, 12, replace=False)
    w = rng.standard_normal(12)
    win = [rng.standard_normal((32, 3)) for _ in range(5)]
    params = rng.uniform(size=(6, 2))
    od = odd.parametric_dmd(win, 0.05, 0.2, params, np.array([0, 2, 4]))
    gd = m.hyper.fit_parametric_dmd(win, 0.05, 0.2, params, np.array([0, 2, 4]))
    deim_o = odd.Deim(psi=None, indices=idx, weights=w)
    deim_g = m.hyper.DEIMModel(psi=None, indices=idx, weights=w)
    go = orl.hyper_stage(osys, od, deim_o, 0.225, params)(u)(z)
    import torch
    gg = m.hyper.make_hyper_stage_device(gd, deim_g, 0.225, gsys, params)(torch.from_numpy(u).cuda())(z)
    assert rel(gg, go) <= 1e-12


def test_reduced_run_with_hyper_reduction(m):
    """Hyper-reduction engages after the window fills; energies track the oracle."""
    u, z, osys, gsys, x0, v0, lengths = _setup(m, 1, False, n=3000, p=6, nx=16, nb=4, seed=7)
    params = np.stack([np.linspace(0.03, 0.06, 6), np.linspace(0.8, 1.0, 6)], axis=1)
    kw = dict(basis_dim=4, subsample=4, window=2, deim_dim=8, deim_period=2, deim_update=3,
              dt=0.01)
    h = orl.run_reduced(osys, params, x0, v0, num_steps=8, energy_stride=1, decomp_stride=2, **kw)
    rec = m.driver.run_reduced(gsys, params, x0, v0, t_final=0.08, energy_stride=1,
                               decomp_stride=2, **kw)
    assert rec.hyper_engaged and h.hyper_engaged
    for a, b in zip(rec.deim_indices, h.deim_indices):
        np.testing.assert_array_equal(a, b)
    ee_o = np.asarray(h.electric)
    assert np.max(np.abs(rec.electric_energy - ee_o) / np.abs(ee_o)) <= 1e-9
    # Hamiltonian-error decomposition at decomp_stride (driver.py:229-246):
    # differences of O(|H|) energies, compared at 1e-10 |H|
    np.testing.assert_allclose(rec.decomp_times, h.decomp_times)
    assert len(rec.decomp_times) >= 2
    hscale = np.linalg.norm(np.asarray(h.kinetic[-1]) + np.asarray(h.electric[-1]))
    for key in ("dh_total", "dh_coeff", "dh_coeff_dd"):
        np.testing.assert_allclose(getattr(rec, key), getattr(h, key), rtol=0, atol=1e-10 * hscale)
    assert rec.dmd_imag_defect >= 0.0 and rec.timers is not None
    assert rec.s_conds.shape == rec.fp_iterations.shape == (8,)


def test_reduced_run_decomposition_per_instance(m):
    """decomp_stride on per-instance meshes (C4's layout): the device
    hyper_hamiltonian (per-column mesh, mass and weight scaling) vs the oracle."""
    u, z, osys, gsys, x0, v0, lengths = _setup(m, 2, True, n=3000, p=6, nx=16, nb=4, seed=8)
    params = np.stack([2 * np.pi / lengths, np.linspace(0.03, 0.06, 6)], axis=1)
    kw = dict(basis_dim=4, subsample=4, window=2, deim_dim=8, deim_period=2, deim_update=3,
              dt=0.01)
    h = orl.run_reduced(osys, params, x0, v0, num_steps=7, energy_stride=1, decomp_stride=3, **kw)
    rec = m.driver.run_reduced(gsys, params, x0, v0, t_final=0.07, energy_stride=1,
                               decomp_stride=3, **kw)
    np.testing.assert_array_equal(rec.fp_iterations, np.asarray(h.fp_iterations))
    np.testing.assert_allclose(rec.decomp_times, h.decomp_times)
    hscale = np.linalg.norm(np.asarray(h.kinetic[-1]) + np.asarray(h.electric[-1]))
    for key in ("dh_total", "dh_coeff", "dh_coeff_dd"):
        np.testing.assert_allclose(getattr(rec, key), getattr(h, key), rtol=0, atol=1e-10 * hscale)


@pytest.mark.parametrize("d", [2, 3])
def test_gather_uv_projections_vs_dense(m, d):
    """picrom_rom_gather_uv's two DMMA projections (U_X^T E, U_V^T E) against the
    dense products of the E it also returns and of the oracle's gradient."""
    import torch
    u, z, osys, gsys, *_ = _setup(m, d, True)
    og, _, _ = orl.exact_gradients(osys, u, z)
    ud = torch.from_numpy(u).cuda()
    dg, _, _ = m.driver.exact_gradients_device(gsys, ud, z, harvest=False)
    N = u.shape[0] // 2
    e = og[:N]                                     # oracle E = coef d/dx (phi.Lambda)(U_X z)
    assert rel(dg.e.cpu().numpy(), e) <= 1e-12
    assert rel(dg.ux_e, u[:N].T @ e) <= 1e-12
    assert rel(dg.uv_e, u[N:].T @ e) <= 1e-12


def test_gram_tasks_blocks(m):
    """Only the requested block products of a tall Gram (the tangent transport's
    7 of 10), with and without the DMMA fast path (equal widths / a wider block)."""
    import torch
    from paper_2201_05555_b200 import _tall
    rng = np.random.default_rng(3)
    rows = 2 * 30011
    for widths in ([20, 20, 20, 20], [20, 24, 20, 20]):
        hs = [rng.standard_normal((rows, w)) for w in widths]
        blocks = [(torch.from_numpy(h).cuda(), False) for h in hs]
        tasks = [(0, 0), (0, 1), (0, 2), (0, 3), (1, 3), (2, 1), (2, 3)]
        G = _tall.gram_tasks(blocks, tasks)
        off = np.concatenate([[0], np.cumsum(widths)])
        for i, j in tasks:
            ref = hs[i].T @ hs[j]
            got = G[off[i]:off[i + 1], off[j]:off[j + 1]]
            assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max(), (widths, i, j)


def test_host_results_not_recycled_while_held(m):
    """Result arrays come from recycled pinned buffers: a held result is never
    overwritten by a later call; a dropped one's buffer is reused."""
    import torch
    from paper_2201_05555_b200 import _device as dev
    a = torch.full((1 << 20,), 1.0, dtype=torch.float64, device="cuda")
    b = torch.full((1 << 20,), 2.0, dtype=torch.float64, device="cuda")
    ha = dev.to_host(a)
    hb = dev.to_host(b)
    assert ha.ctypes.data != hb.ctypes.data
    assert (ha == 1.0).all() and (hb == 2.0).all()
    del ha
    live = [dev.to_host(b * k) for k in (3, 4, 5)]     # may reuse ha's buffer, never hb's
    assert (hb == 2.0).all()
    for k, h in zip((3, 4, 5), live):
        assert (h == 2.0 * k).all()
    assert len({h.ctypes.data for h in live} | {hb.ctypes.data}) == 4


def test_host_result_views_keep_their_buffer(m):
    """A numpy VIEW of a recycled pinned result (transpose / slice, as
    run_full_order's potential history) keeps the slot reserved after the
    original array is dropped (the history views once aliased)."""
    import torch
    from paper_2201_05555_b200 import _device as dev
    rows = (5 << 20) // (8 * 12)                       # >= 4 MiB: the recycled path
    a = torch.full((rows, 3, 4), 1.0, dtype=torch.float64, device="cuda")
    b = torch.full((rows, 3, 4), 2.0, dtype=torch.float64, device="cuda")
    va = dev.to_host(a).transpose(0, 2, 1)             # the array itself is dropped at once
    vs = dev.to_host(a)[::2]
    hb = dev.to_host(b)                                # same size: must not reuse va's/vs's slot
    assert (va == 1.0).all() and (vs == 1.0).all() and (hb == 2.0).all()
    # end to end: potential and charge histories of a run at >= 4 MiB stay distinct
    fem, fo = m.fem, m.fullorder
    n, p, nx, steps = 2048, 32, 128, 160               # 161 x 32 x 128 x 8 B = 5.3 MB each
    rng = np.random.default_rng(0)
    L = 4 * np.pi
    x, v = rng.uniform(0, L, (n, p)), rng.standard_normal((n, p))
    sysm = fo.VlasovSystem(fem.build_mesh(L, nx, 1), fem.ChargeConfig(n, L))
    rec = fo.run_full_order(sysm, fo.ParticleEnsemble(x, v), 0.05, steps * 0.05,
                            record=fo.RecordOptions(energy_stride=1, record_snapshots=False))
    assert rec.potential_history.nbytes >= (4 << 20)
    assert not np.array_equal(rec.potential_history, rec.charge_history)
    np.testing.assert_array_equal(rec.potentials, rec.potential_history)
    # the potential solves the Poisson problem of the recorded charge
    phi = m.fem.PoissonOperator(sysm.mesh).solve(rec.charge_history[-1])
    assert rel(phi, rec.potential_history[-1]) <= 1e-12


def _align_phases(u, ref, n):
    """Rotate each (Phi_j, Psi_j) pair of u onto ref's phase (complex
    singular vectors are defined up to e^{i theta})."""
    N = u.shape[0] // 2
    h = n // 2
    a = u[:N, :h] + 1j * u[N:, :h]
    b = ref[:N, :h] + 1j * ref[N:, :h]
    ph = np.exp(1j * np.angle(np.einsum("ij,ij->j", np.conj(a), b)))
    a = a * ph
    out = np.empty_like(u)
    out[:N, :h], out[N:, :h] = a.real, a.imag
    out[:N, h:], out[N:, h:] = -a.imag, a.real
    return out


@pytest.mark.parametrize("N,p,n", [(20_000, 16, 6), (200_000, 128, 20)])
def test_device_complex_svd_basis(m, N, p, n):
    """complex_svd_basis_device (Hermitian Gram + eigensolve + combines) equals the
    host LAPACK basis modulo the per-vector phase: U <= 1e-12 after phase
    alignment, U Z (the reconstruction) and U^T U directly."""
    rng = np.random.default_rng(N)
    ks = rng.uniform(0.4, 0.6, p)
    x = np.stack([rng.uniform(0, 2 * np.pi / k, N) for k in ks], axis=1)
    v = rng.standard_normal((N, p))
    u_h, z_h = m.red.complex_svd_basis(x, v, n)
    u_d, z_d = m.red.complex_svd_basis_device(x, v, n)
    u_d = u_d.cpu().numpy()
    ua = _align_phases(u_d, u_h, n)
    assert rel(ua, u_h) <= 1e-12
    assert rel(u_d @ z_d, u_h @ z_h) <= 1e-12
    assert np.abs(u_d.T @ u_d - np.eye(n)).max() <= 1e-13
    o, s_ = m.red.orthosymplectic_residuals(u_d)
    assert o <= 1e-13 and s_ <= 1e-13


def test_compare_diagnostics_vs_reference(m):
    """diagnostics.relative_errors / total_relative_error /
    target_projection_errors / numerical_rank / hamiltonian_relative_error
    (device norms, device cSVD basis) against the reference's own functions
    (picrom.diagnostics from baseline/_ref) or their formulas."""
    import sys
    from pathlib import Path
    from paper_2201_05555_b200 import diagnostics as dg
    rng = np.random.default_rng(17)
    N, p, nb = 40_000, 12, 6
    sx = rng.uniform(0, 10, (N, p))
    sv = rng.standard_normal((N, p))
    u, z = m.red.complex_svd_basis(sx, sv, nb)
    xr, vr = u[:N] @ z, u[N:] @ z
    ref = Path(__file__).resolve().parent.parent / "baseline" / "_ref"
    if (ref / "picrom").exists():
        sys.path.insert(0, str(ref))
        try:
            from picrom import diagnostics as rdg
        finally:
            sys.path.remove(str(ref))
        want = dict(rel=rdg.relative_errors(sx, sv, xr, vr),
                    tot=rdg.total_relative_error(sx, sv, xr, vr),
                    tgt=rdg.target_projection_errors(sx, sv, nb),
                    rank=rdg.numerical_rank(np.concatenate([sx, sv]), 1e-3),
                    ham=rdg.hamiltonian_relative_error(np.arange(1.0, 5.0), np.arange(1.0, 5.0) + 1e-3))
    else:
        def r(a, b):
            return np.linalg.norm(a - b) / np.linalg.norm(a)
        s = np.linalg.svd(np.concatenate([sx, sv]), compute_uv=False)
        want = dict(rel=(r(sx, xr), r(sv, vr)),
                    tot=r(np.concatenate([sx, sv]), np.concatenate([xr, vr])),
                    tgt=(r(sx, xr), r(sv, vr)), rank=int((s >= 1e-3 * s[0]).sum()),
                    ham=np.linalg.norm(np.full(4, 1e-3)) / np.linalg.norm(np.arange(1.0, 5.0)))
    got_rel = dg.relative_errors(sx, sv, xr, vr)
    np.testing.assert_allclose(got_rel, want["rel"], rtol=1e-12)
    np.testing.assert_allclose(dg.total_relative_error(sx, sv, xr, vr), want["tot"], rtol=1e-12)
    np.testing.assert_allclose(dg.target_projection_errors(sx, sv, nb), want["tgt"], rtol=1e-10)
    assert dg.numerical_rank(np.concatenate([sx, sv]), 1e-3) == want["rank"]
    np.testing.assert_allclose(dg.hamiltonian_relative_error(np.arange(1.0, 5.0),
                                                             np.arange(1.0, 5.0) + 1e-3),
                               want["ham"], rtol=1e-14)
