"""Parity at BASELINE.json's own configurations (C1-C5), at their stated sizes.

Inputs are the seeded workloads (paper_2201_05555_b200.workloads, SURVEY.md
§8(d)), regenerated bit for bit here.  Tolerances are north_star's:
* teacher-forced (the SAME positions fed to the GPU and the CPU oracle) charge
  and potential <= 1e-12 per step (normwise), charge also <= 1e-14 against the
  norm of its particle term;
* free-running electric-energy history <= 1e-9 (max relative over the run).

C1 (100k x 1, quadratic, 200 steps) runs the oracle live.  C2 (8 M particles,
cubic, 500 steps) compares with tests/golden/config_C2.npz (the oracle's run,
tests/golden/make_config_golden.py) and is teacher-forced live at 5 sampled
steps.  C5 (256 M particles) is teacher-forced live at full size at steps 0, 1
and 3, plus a 100-step free run at N = 40k with C5's p, Nx and distribution.
The reduced configurations (C3/C4) follow below the FOM ones.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
from conftest import GOLDEN
from oracle import fe_bspline as fe
from oracle import pic_loop

pytestmark = pytest.mark.gpu

CORES = max(1, len(os.sched_getaffinity(0)))


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def mods(lib_built):
    from paper_2201_05555_b200 import fem, fullorder
    from paper_2201_05555_b200 import workloads as wl
    return fem, fullorder, wl


def oracle_rho_phi(w, x_pn, cols=None):
    """Oracle deposit + solve (fem.py:203-244 restated) of (p, N) positions,
    one column per task over the host cores: (rho (Nx, p), phi (Nx, p))."""
    p = x_pn.shape[0]
    cols = range(p) if cols is None else cols
    n = x_pn.shape[1]

    def one(j):
        L = float(w.lengths[j])
        mesh = fe.Mesh(L, w.num_cells, w.degree)
        rho = fe.deposit_charge(fe.eval_basis(mesh, x_pn[j]), fe.Charge(n, L))
        return rho, fe.Poisson(mesh).solve(rho)

    with ThreadPoolExecutor(max_workers=CORES) as pool:
        out = list(pool.map(one, cols))
    return np.stack([o[0] for o in out], axis=1), np.stack([o[1] for o in out], axis=1)


def check_teacher_forced(w, run, k, x_pn, tag, report=None):
    """GPU rho_k / phi_k of the run vs the oracle's on the run's own x_k."""
    rho_o, phi_o = oracle_rho_phi(w, x_pn)
    rho_g = run.rho_hist[k].cpu().numpy().T
    phi_g = run.phi_hist[k].cpu().numpy().T
    bgh = np.array([1.0 * (L / w.num_cells) for L in w.lengths])[None, :]
    e_rho, e_phi = rel(rho_g, rho_o), rel(phi_g, phi_o)
    e_part = np.linalg.norm(rho_g - rho_o) / np.linalg.norm(rho_o - bgh)
    assert e_rho <= 1e-12, (tag, k, e_rho)
    assert e_phi <= 1e-12, (tag, k, e_phi)
    assert e_part <= 1e-14, (tag, k, e_part)
    if report:
        report(step=k, teacher_forced_rho=e_rho, teacher_forced_phi=e_phi, rho_vs_particle_term=e_part)
    return e_rho, e_phi


def _gpu_run(mods, w, x_pn, v_pn, steps):
    import torch
    fem, fo, _ = mods
    L = float(w.lengths[0])
    n = x_pn.shape[1]
    sysm = fo.VlasovSystem(fem.build_mesh(L, w.num_cells, w.degree), fem.ChargeConfig(n, L))
    run = fo.PicRun(sysm, torch.from_numpy(x_pn).cuda(), torch.from_numpy(v_pn).cuda(), w.dt,
                    steps)
    run.init_field()
    return sysm, run


def test_c1_full_size_free_run(mods, parity_report):
    """C1 at its size: 100k particles, quadratic, 200 steps; oracle live."""
    fem, fo, wl = mods
    w = wl.config("C1")
    x, v = wl.generate(w)
    L = float(w.lengths[0])
    osys = pic_loop.System(fe.Mesh(L, w.num_cells, w.degree), fe.Charge(x.shape[0], L))
    hist = pic_loop.run(osys, x, v, w.dt, w.num_steps)
    gsys = fo.VlasovSystem(fem.build_mesh(L, w.num_cells, w.degree),
                           fem.ChargeConfig(x.shape[0], L))
    rec = fo.run_full_order(gsys, fo.ParticleEnsemble(x.copy(), v.copy(), 0.0), w.dt,
                            w.num_steps * w.dt,
                            record=fo.RecordOptions(energy_stride=1, record_snapshots=False))
    ee = np.max(np.abs(rec.electric_history - hist.electric) / np.abs(hist.electric))
    kin = np.max(np.abs(rec.kinetic_history - hist.kinetic) / np.abs(hist.kinetic))
    assert rec.electric_energy.shape == (w.num_steps + 1, 1)
    assert ee <= 1e-9 and kin <= 1e-9, (ee, kin)
    # free-running charge / potential along the whole run
    worst_rho = max(rel(rec.charge_history[k], hist.rho[k]) for k in range(w.num_steps + 1))
    worst_phi = max(rel(rec.potential_history[k], hist.phi[k]) for k in range(w.num_steps + 1))
    assert worst_rho <= 1e-10 and worst_phi <= 1e-10, (worst_rho, worst_phi)
    parity_report(free_energy=ee, free_kinetic=kin, free_rho_worst=worst_rho, free_phi_worst=worst_phi)
    # teacher-forced at sampled steps of the GPU's own trajectory
    xp, vp = wl.generate(w, layout="pn")
    _, run = _gpu_run(mods, w, xp, vp, w.num_steps)
    check_teacher_forced(w, run, 0, xp, "C1", parity_report)
    done = 0
    for k in (1, 50, 200):
        run.advance(k - done)
        done = k
        check_teacher_forced(w, run, k, run.x.cpu().numpy(), "C1", parity_report)


def test_c2_full_size_500_steps(mods, parity_report):
    """C2 at its size (32 x 250k, cubic two-stream, 500 steps): free-running
    energy history vs the oracle's run (fixture), teacher-forced charge and
    potential at 5 sampled steps (oracle live on the GPU's positions)."""
    fem, fo, wl = mods
    f = np.load(GOLDEN / "config_C2.npz")
    w = wl.config("C2")
    xp, vp = wl.generate(w, layout="pn")
    _, run = _gpu_run(mods, w, xp, vp, w.num_steps)
    check_teacher_forced(w, run, 0, xp, "C2", parity_report)
    done = 0
    samples = [int(k) for k in f["sample_steps"]]
    free = {}
    for k in samples:
        run.advance(k - done)
        done = k
        check_teacher_forced(w, run, k, run.x.cpu().numpy(), "C2", parity_report)
    run.finish_kinetic()
    run.check()
    ee_g = run.ee_hist.cpu().numpy()
    kin_g = run.kin_hist.cpu().numpy()
    ee = np.max(np.abs(ee_g - f["electric"]) / np.abs(f["electric"]))
    kin = np.max(np.abs(kin_g - f["kinetic"]) / np.abs(f["kinetic"]))
    assert ee <= 1e-9, ee
    assert kin <= 1e-9, kin
    # free-running charge / potential at the sampled steps (the two-stream
    # instability amplifies per-particle rounding; bounded well inside 1e-9)
    for i, k in enumerate(samples):
        free[k] = (rel(run.rho_hist[k].cpu().numpy().T, f["rho"][i]),
                   rel(run.phi_hist[k].cpu().numpy().T, f["phi"][i]))
        assert max(free[k]) <= 1e-9, (k, free[k])
    # the first particles' final state, against the oracle's full-step values
    xo = run.x.cpu().numpy()[:, :64].T
    assert rel(xo, f["x_final_rows"]) <= 1e-9
    parity_report(free_energy=ee, free_kinetic=kin, free_rho_worst=max(v[0] for v in free.values()),
                  free_phi_worst=max(v[1] for v in free.values()), x_final=rel(xo, f["x_final_rows"]))


def test_c5_full_size_teacher_forced(mods, parity_report):
    """C5 at its size (64 x 4M = 256M particles, Nx = 512, cubic): charge and
    potential at steps 0, 1 and 3 vs the oracle on the same positions."""
    fem, fo, wl = mods
    w = wl.config("C5")
    xp, vp = wl.generate(w, layout="pn")
    _, run = _gpu_run(mods, w, xp, vp, 3)
    del vp
    check_teacher_forced(w, run, 0, xp, "C5", parity_report)
    del xp
    run.advance(1)
    check_teacher_forced(w, run, 1, run.x.cpu().numpy(), "C5", parity_report)
    run.advance(2)
    run.check()
    check_teacher_forced(w, run, 3, run.x.cpu().numpy(), "C5", parity_report)


def test_c5_reduced_n_free_run(mods, parity_report):
    """C5's p = 64, Nx = 512, cubic bump-on-tail at N = 40k per instance,
    100 steps free-running: energy history <= 1e-9 vs the oracle (live)."""
    fem, fo, wl = mods
    w = wl.config("C5")
    n = 40_000
    x, v = wl.generate(w, num_particles=n)
    L = float(w.lengths[0])
    osys = pic_loop.System(fe.Mesh(L, w.num_cells, w.degree), fe.Charge(n, L), workers=CORES)
    hist = pic_loop.run(osys, x, v, w.dt, w.num_steps)
    gsys = fo.VlasovSystem(fem.build_mesh(L, w.num_cells, w.degree), fem.ChargeConfig(n, L))
    rec = fo.run_full_order(gsys, fo.ParticleEnsemble(x, v, 0.0), w.dt, w.num_steps * w.dt,
                            record=fo.RecordOptions(energy_stride=1, record_snapshots=False))
    ee = np.max(np.abs(rec.electric_history - hist.electric) / np.abs(hist.electric))
    kin = np.max(np.abs(rec.kinetic_history - hist.kinetic) / np.abs(hist.kinetic))
    assert ee <= 1e-9 and kin <= 1e-9, (ee, kin)
    parity_report(free_energy=ee, free_kinetic=kin, rho_step1=rel(rec.charge_history[1], hist.rho[1]))
    assert rel(rec.charge_history[1], hist.rho[1]) <= 1e-12
    assert rel(rec.potential_history[1], hist.phi[1]) <= 1e-12


# ------------------------------------------------------------------ C3 / C4

@pytest.fixture(scope="module")
def rom(lib_built):
    from paper_2201_05555_b200 import driver, hyper, reduction
    from paper_2201_05555_b200 import workloads as wl
    return driver, reduction, hyper, wl


def _rom_inputs(wl, name, n=None):
    w = wl.config(name)
    x0, v0 = wl.generate(w, num_particles=n)
    params = np.stack([w.wavenumbers, w.alphas], axis=1)
    return w, x0, v0, params


def test_c3_full_scale_teacher_forced(rom, parity_report):
    """C3 at its size (N = 1e6, p = 128, n = 20, quadratic, per-instance k):
    F(U Z) (charge -> potential -> gradient, the DEIM harvest Lambda phi), the
    warm-up stage U^T F(U z) and the manifold maps (basis velocity, both
    retractions, tangent transport) on the SAME (U, Z) for GPU and oracle, at
    the initial basis and after two GPU steps; <= 1e-12 normwise."""
    import torch
    from oracle import manifold as omf
    from oracle import rom_loop as orl
    driver, red, _, wl = rom
    w, x0, v0, params = _rom_inputs(wl, "C3")
    N, nb = w.num_particles, w.extra["basis_dim"]
    u0, z0 = red.complex_svd_basis(x0, v0, nb)
    osys = orl.ParamSystem(w.lengths, w.num_cells, w.degree, N)
    gsys = driver.ParametricVlasovSystem(w.lengths, w.num_cells, w.degree, N)
    rec = driver.run_reduced(gsys, params, x0, v0, basis_dim=nb, subsample=w.p, window=3,
                             deim_dim=8, deim_period=3, deim_update=2, dt=w.dt, t_final=2 * w.dt,
                             hyper_reduction=False, energy_stride=10**9, snapshot_stride=2,
                             decomp_stride=10**9, u0=u0, z0=z0)
    del x0, v0
    u2, z2 = rec.bases[-1]
    dt = w.dt
    for tag, u, z in (("step0", u0, z0), ("step2", u2.cpu().numpy(), z2)):
        ud = torch.from_numpy(u).cuda()
        og, ophi, olam = orl.exact_gradients(osys, u, z)
        gg, gphi, glam = driver.exact_gradients(gsys, ud, z)
        errs = dict(phi=rel(gphi.cpu().numpy(), ophi), grad=rel(gg.cpu().numpy(), og),
                    lam=rel(glam.cpu().numpy(), olam))
        assert errs["phi"] <= 1e-12 and errs["grad"] <= 1e-12 and errs["lam"] <= 1e-12, (tag, errs)
        del gg, glam, olam
        stage = driver.make_full_stage(gsys)(ud)(z)
        errs["stage"] = rel(stage, u.T @ og)
        assert errs["stage"] <= 1e-12, tag
        # manifold maps: GPU basis velocity from its own implicit device gradient
        dg, _, _ = driver.exact_gradients_device(gsys, ud, z, harvest=False)
        xi_o = omf.velocity_of_basis(u, z, og)
        xi_g = red.basis_velocity(ud, z, dg)
        errs["basis_velocity"] = rel(xi_g.cpu().numpy(), xi_o)
        assert errs["basis_velocity"] <= 1e-12, tag
        del og, dg, xi_g
        r_o = omf.cayley_retract(u, 0.5 * dt * xi_o)
        r_g = red.retraction(ud, red.scaled(torch.from_numpy(xi_o).cuda(), 0.5 * dt))
        errs["retraction"] = rel(r_g.cpu().numpy(), r_o)
        assert errs["retraction"] <= 1e-12, tag
        x_eval = xi_o[::-1].copy()                     # any tangent-sized operand
        t_o = omf.transport_back(u, 0.5 * dt * xi_o, r_o, x_eval)
        t_g = red.tangent_velocity(ud, red.scaled(torch.from_numpy(xi_o).cuda(), 0.5 * dt),
                                   torch.from_numpy(r_o).cuda(), torch.from_numpy(x_eval).cuda())
        errs["tangent"] = rel(t_g.cpu().numpy(), t_o)
        assert errs["tangent"] <= 1e-12, tag
        o_o, s_o = omf.structure_defects(r_o)
        o_g, s_g = red.orthosymplectic_residuals(r_g)
        assert abs(o_g - o_o) <= 1e-13 and abs(s_g - s_o) <= 1e-13, tag
        parity_report(at=tag, **errs)


def _rom_free_run(rom, name, report=None):
    from oracle import manifold as omf
    driver, red, _, wl = rom
    f = np.load(GOLDEN / f"config_{name}.npz")
    n = int(f["num_particles"])
    w, x0, v0, params = _rom_inputs(wl, name[:2], n)
    ex = w.extra
    nb = ex["basis_dim"]
    u0, z0 = red.complex_svd_basis(x0, v0, nb)
    # the box's LAPACK reproduces the fixture's initial basis (same seeded data)
    assert rel(z0, f["z0"]) <= 1e-12
    assert rel(u0[f["rows"]], f["u0_rows"]) <= 1e-12
    gsys = driver.ParametricVlasovSystem(w.lengths, w.num_cells, w.degree, n)
    steps, es = int(f["steps"]), int(f["energy_stride"])
    rec = driver.run_reduced(
        gsys, params, x0, v0, basis_dim=nb, subsample=ex.get("subsample", w.p),
        window=ex.get("window", 3), deim_dim=ex.get("deim_dim", 8),
        deim_period=ex.get("deim_period", 3), deim_update=ex.get("deim_update", 2), dt=w.dt,
        t_final=steps * w.dt, hyper_reduction=name.startswith("C4"), energy_stride=es,
        snapshot_stride=steps, decomp_stride=10**9, u0=u0, z0=z0)
    np.testing.assert_array_equal(np.sort(omf.farthest_point_subset(z0, ex.get("subsample", w.p))),
                                  f["sub"])
    np.testing.assert_array_equal(rec.fp_iterations, f["fp_iterations"])
    ee = np.max(np.abs(rec.electric_energy - f["electric"]) / np.abs(f["electric"]))
    ham_o = f["kinetic"] + f["electric"]
    ham = np.max(np.abs(rec.hamiltonian - ham_o) / np.abs(ham_o))
    assert ee <= 1e-9 and ham <= 1e-9, (ee, ham)
    u, z = rec.bases[-1]
    assert rel(z, f["z_final"]) <= 1e-9
    assert rel(u.cpu().numpy()[f["rows"]], f["u_final_rows"]) <= 1e-9
    np.testing.assert_allclose(rec.ortho_residuals, f["ortho"], atol=1e-13)
    if report:
        report(free_energy=ee, free_hamiltonian=ham, z_final=rel(z, f["z_final"]),
               u_final_rows=rel(u.cpu().numpy()[f["rows"]], f["u_final_rows"]),
               fp_iterations_mean=float(np.mean(rec.fp_iterations)))
    return rec, f


def test_c3_reduced_n_free_run(rom, parity_report):
    """C3's p = 128, n = 20, quadratic, per-instance k, 200 steps at N = 5e4:
    fixed-point counts equal, energies <= 1e-9 vs the oracle's run (fixture)."""
    _rom_free_run(rom, "C3r", parity_report)


def _recording(monkeypatch, module, name, sink, wrap=None):
    orig = getattr(module, name)

    def rec(*a, **k):
        r = orig(*a, **k)
        sink.append(wrap(a, k, r) if wrap else r)
        return r

    monkeypatch.setattr(module, name, rec)


def test_c4_reduced_n_warmup_fit_and_failure(rom, monkeypatch, parity_report):
    """C4 (p* = 20, T = 20, d = 40) at N = 5e4.  The reference algorithm's
    hyper-reduced fixed point does not converge at this particle count (the
    oracle's run ends in StepFailure at the first hyper step, step 21; at
    N = 1e6 it converges, see the full-scale test below).  Parity: the 20
    warm-up steps (fixed-point counts equal, state and energies <= 1e-9), the
    first DEIM fit's indices bit-exact, and the same StepFailureError with the
    same iteration count and residual trace."""
    from paper_2201_05555_b200.errors import StepFailureError
    driver, red, hyp, wl = rom
    f = np.load(GOLDEN / "config_C4r.npz")
    n = int(f["num_particles"])
    w, x0, v0, params = _rom_inputs(wl, "C4", n)
    ex = w.extra
    u0, z0 = red.complex_svd_basis(x0, v0, ex["basis_dim"])
    assert rel(z0, f["z0"]) <= 1e-12
    gsys = driver.ParametricVlasovSystem(w.lengths, w.num_cells, w.degree, n)
    steps, fits = [], []
    _recording(monkeypatch, driver, "prk2_step", steps)
    _recording(monkeypatch, hyp, "fit_deim_device", fits)
    with pytest.raises(StepFailureError) as err:
        driver.run_reduced(gsys, params, x0, v0, basis_dim=ex["basis_dim"],
                           subsample=ex["subsample"], window=ex["window"], deim_dim=ex["deim_dim"],
                           deim_period=ex["deim_period"], deim_update=ex["deim_update"], dt=w.dt,
                           t_final=(ex["window"] + 1) * w.dt, hyper_reduction=True,
                           energy_stride=10**9, snapshot_stride=10**9, decomp_stride=10**9,
                           u0=u0, z0=z0)
    np.testing.assert_array_equal([r.fp_iterations for r in steps], f["fp_iterations"])
    last = steps[-1]
    assert rel(last.z, f["z_warm"]) <= 1e-9
    assert rel(last.u.cpu().numpy()[f["rows"]], f["u_warm_rows"]) <= 1e-9
    ee, kin = driver._diag_energies(gsys, last.u, last.z)
    assert np.max(np.abs(ee - f["electric_warm"]) / np.abs(f["electric_warm"])) <= 1e-9
    assert np.max(np.abs(kin - f["kinetic_warm"]) / np.abs(f["kinetic_warm"])) <= 1e-9
    np.testing.assert_array_equal(fits[0].indices, f["deim_indices"])
    assert rel(fits[0].weights, f["deim_weights"]) <= 1e-10
    assert err.value.iterations == int(f["fail_iterations"]) == 100
    trace, want = np.asarray(err.value.residual_trace), f["fail_trace"]
    assert np.max(np.abs(trace[:6] - want[:6]) / want[:6]) <= 1e-6
    assert trace[-1] > 1e-9 and want[-1] > 1e-9
    parity_report(z_warm=rel(last.z, f["z_warm"]), deim_weights=rel(fits[0].weights, f["deim_weights"]),
                  trace6=float(np.max(np.abs(trace[:6] - want[:6]) / want[:6])),
                  fp_warm=[int(r.fp_iterations) for r in steps], last_update=float(trace[-1]))


def test_c4_full_scale_first_hyper_step_teacher_forced(rom, monkeypatch, parity_report):
    """C4 at its size (N = 1e6, p = 128, p* = 20, T = 20, d = 40): run the GPU
    model to its first hyper-reduced step (21) and give the oracle the SAME
    inputs of that step -- the potential window, the DEIM sample window, U and
    Z.  DMD eigenvalues equal, DEIM indices bit-exact, DEIM weights and the
    step's Z to tolerance, equal fixed-point iteration counts."""
    from oracle import dmd_deim as odd
    from oracle import manifold as omf
    from oracle import rom_loop as orl
    driver, red, hyp, wl = rom
    w, x0, v0, params = _rom_inputs(wl, "C4")
    ex = w.extra
    N = w.num_particles
    u0, z0 = red.complex_svd_basis(x0, v0, ex["basis_dim"])
    gsys = driver.ParametricVlasovSystem(w.lengths, w.num_cells, w.degree, N)
    dmd_in, deim_in, prk_in = [], [], []

    def cap_dmd(a, k, r):
        return ([np.array(b) for b in a[0]], a[2], r)

    def cap_deim(a, k, r):
        cols = [c.cpu().numpy() for c in a[0].columns()]      # ring order, oldest first
        return (cols, r)

    def cap_prk(a, k, r):
        return (a[0].cpu().numpy(), np.array(a[1]), r) if len(prk_in) == ex["window"] else None

    _recording(monkeypatch, hyp, "fit_parametric_dmd", dmd_in, cap_dmd)
    _recording(monkeypatch, hyp, "fit_deim_device", deim_in, cap_deim)
    _recording(monkeypatch, driver, "prk2_step", prk_in, cap_prk)
    driver.run_reduced(gsys, params, x0, v0, basis_dim=ex["basis_dim"], subsample=ex["subsample"],
                       window=ex["window"], deim_dim=ex["deim_dim"],
                       deim_period=ex["deim_period"], deim_update=ex["deim_update"], dt=w.dt,
                       t_final=(ex["window"] + 1) * w.dt, hyper_reduction=True,
                       energy_stride=10**9, snapshot_stride=10**9, decomp_stride=10**9,
                       u0=u0, z0=z0)
    del x0, v0
    win, t_prev, g_dmd = dmd_in[0]
    cols, g_deim = deim_in[0]
    u, z, g_res = prk_in[-1]
    osys = orl.ParamSystem(w.lengths, w.num_cells, w.degree, N)
    sub = np.sort(omf.farthest_point_subset(z0, ex["subsample"]))
    o_dmd = odd.parametric_dmd(win, w.dt, t_prev, params, sub)
    np.testing.assert_allclose(np.sort_complex(g_dmd.eigenvalues), np.sort_complex(o_dmd.eigenvalues),
                               rtol=1e-10)
    block = np.stack(cols).transpose(1, 2, 0)               # the reference's column order
    del cols
    o_deim = odd.deim_fit(block.reshape(block.shape[0], -1), ex["deim_dim"],
                          osys.charge.charge_weight)
    del block
    np.testing.assert_array_equal(g_deim.indices, o_deim.indices)
    assert rel(g_deim.weights, o_deim.weights) <= 1e-10
    grad_sub = lambda uu, zs: orl.exact_gradients(osys, uu, zs, sub)[0]  # noqa: E731
    o_res = omf.prk2(u, z, w.dt, sub, grad_sub, grad_sub(u, z[:, sub]),
                     orl.hyper_stage(osys, o_dmd, o_deim, t_prev + 0.5 * w.dt, params))
    assert g_res.fp_iterations == o_res.fp_iterations
    assert rel(g_res.z, o_res.z) <= 1e-9
    assert rel(g_res.u.cpu().numpy(), o_res.u) <= 1e-9
    parity_report(deim_weights=rel(g_deim.weights, o_deim.weights), z=rel(g_res.z, o_res.z),
                  u=rel(g_res.u.cpu().numpy(), o_res.u), fp_iterations=int(g_res.fp_iterations))
