"""GPU full-order PIC vs the CPU oracle.

* VerletStepper.step (reference operation order) vs the reference's golden
  steps (degree 1) and vs the oracle (degrees 2/3), 1e-12.
* run_full_order (fused leapfrog loop, CUDA graphs): free-running electric-
  energy history <= 1e-9 relative (north_star), teacher-forced per-step charge
  and potential <= 1e-12, bitwise determinism, DivergenceError context.
* the reference's own stepper tests with test doubles
  (/root/reference/pkg/tests/test_fullorder.py:19-101).
"""

from pathlib import Path

import numpy as np
import pytest
from conftest import GOLDEN
from oracle import fe_bspline as fe
from oracle import pic_loop

ROOT = Path(__file__).resolve().parent.parent

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def mods(lib_built):
    from paper_2201_05555_b200 import fem, fullorder
    return fem, fullorder


def test_stepper_matches_reference_golden(mods):
    fem, fo = mods
    f = np.load(GOLDEN / "fullorder_p1.npz")
    L, nx = float(f["length"]), int(f["nx"])
    sysm = fo.VlasovSystem(fem.build_mesh(L, nx), fem.ChargeConfig(f["x"].shape[0], L))
    st = fo.VerletStepper(sysm)
    e1 = st.step(fo.ParticleEnsemble(f["x"].copy(), f["v"].copy(), 0.0), 0.1)
    e2 = st.step(e1, 0.1)
    for got, key in ((e1.x, "x_step1"), (e1.v, "v_step1"), (e2.x, "x_step2"), (e2.v, "v_step2")):
        assert rel(got, f[key]) <= 1e-12, key
    assert rel(st.last_potential, f["phi_step2"]) <= 1e-12


@pytest.mark.parametrize("d", [2, 3])
def test_stepper_matches_oracle(mods, d):
    fem, fo = mods
    rng = np.random.default_rng(d)
    L, nx, n, p = 10 * np.pi, 64, 5000, 3
    x, v = rng.uniform(0, L, (n, p)), rng.standard_normal((n, p))
    osys = pic_loop.System(fe.Mesh(L, nx, d), fe.Charge(n, L))
    ost = pic_loop.Stepper(osys)
    gst = fo.VerletStepper(fo.VlasovSystem(fem.build_mesh(L, nx, d), fem.ChargeConfig(n, L)))
    ox, ov, t = x, v, 0.0
    ens = fo.ParticleEnsemble(x.copy(), v.copy(), 0.0)
    for _ in range(3):
        ox, ov, t = ost.step(ox, ov, t, 0.05)
        ens = gst.step(ens, 0.05)
    assert rel(ens.x, ox) <= 1e-12 and rel(ens.v, ov) <= 1e-12
    assert rel(gst.last_potential, ost.last_potential) <= 1e-11


class HarmonicDouble:
    def field(self, x):
        return -np.asarray(x, dtype=float), np.zeros(4)


def test_stepper_with_test_double_exact(mods):
    _, fo = mods
    for dt in (0.01, 0.1, 0.5):
        a11 = 1 - dt * dt / 2
        m = np.array([[a11, dt], [-dt / 2 * (1 + a11), 1 - dt * dt / 2]])
        out = fo.VerletStepper(HarmonicDouble()).step(
            fo.ParticleEnsemble(np.array([0.7]), np.array([-0.3]), 0.0), dt)
        np.testing.assert_allclose([out.x[0], out.v[0]], m @ np.array([0.7, -0.3]), atol=1e-14)


def _compare_run(mods, d, nx, n, p, steps, dt, L, vgen, seed):
    fem, fo = mods
    rng = np.random.default_rng(seed)
    x = rng.uniform(0, L, (n, p))
    v = vgen(rng, (n, p))
    osys = pic_loop.System(fe.Mesh(L, nx, d), fe.Charge(n, L))
    hist = pic_loop.run(osys, x, v, dt, steps)
    gsys = fo.VlasovSystem(fem.build_mesh(L, nx, d), fem.ChargeConfig(n, L))
    rec = fo.run_full_order(gsys, fo.ParticleEnsemble(x.copy(), v.copy(), 0.0), dt, steps * dt,
                            record=fo.RecordOptions(energy_stride=1, record_snapshots=False))
    return hist, rec, gsys, osys


@pytest.mark.parametrize("d", [1, 2, 3])
def test_run_energy_history_landau(mods, d):
    """C1-like (Landau, 200 steps): free-running electric-energy history <= 1e-9."""
    L = 4 * np.pi
    hist, rec, gsys, osys = _compare_run(mods, d, 64, 20_000, 2, 200, 0.05, L,
                                         lambda r, s: r.standard_normal(s), seed=11)
    ee_o, ee_g = hist.electric, rec.electric_history
    worst = np.max(np.abs(ee_g - ee_o) / np.abs(ee_o))
    assert worst <= 1e-9, worst
    assert np.max(np.abs(rec.kinetic_history - hist.kinetic) / hist.kinetic) <= 1e-9
    # recorded series in the reference layout
    assert rec.electric_energy.shape == (201, 2)
    np.testing.assert_allclose(rec.hamiltonian, rec.kinetic_history + rec.electric_history)
    # per-step charge/potential along the trajectory (free-running, so this
    # also bounds the trajectory drift): 1e-12 at the start
    assert rel(rec.charge_history[1], hist.rho[1]) <= 1e-12
    assert rel(rec.potential_history[1], hist.phi[1]) <= 1e-12


def test_run_two_stream_cubic(mods):
    """C2-like (two-stream, cubic, 4 instances, 300 steps)."""
    def two_stream(r, s):
        return np.where(r.uniform(size=s) < 0.5, -3.0, 3.0) + 0.3 * r.standard_normal(s)
    hist, rec, _, _ = _compare_run(mods, 3, 128, 20_000, 4, 300, 0.05, 10 * np.pi, two_stream, 5)
    worst = np.max(np.abs(rec.electric_history - hist.electric) / np.abs(hist.electric))
    assert worst <= 1e-9, worst


@pytest.mark.parametrize("nx", [512, 2048])
def test_run_bump_on_tail_large_mesh(mods, nx):
    """C5-like (bump-on-tail, cubic, 3 instances, 60 steps) on large meshes:
    Nx = 512 takes the K = 8 lane-shared histograms (C5's path), Nx = 2048 the
    one-histogram-per-warp path (cell-mod-4 phases with match-ranked rounds)
    that the plan picks once K-lane histograms no longer fit shared memory."""
    def bot(r, s):
        return (np.where(r.uniform(size=s) < 0.9, 0.0, 4.5)
                + np.where(r.uniform(size=s) < 0.9, 1.0, 0.5) * r.standard_normal(s))
    hist, rec, _, _ = _compare_run(mods, 3, nx, 40_000, 3, 60, 0.05, 2 * np.pi / 0.3, bot, 9)
    worst = np.max(np.abs(rec.electric_history - hist.electric) / np.abs(hist.electric))
    rho = rel(rec.charge_history[1], hist.rho[1])
    assert worst <= 1e-9 and rho <= 1e-12, (worst, rho)


def test_push_plus_solve_equals_fused_step(mods):
    """picrom_pic_push + picrom_pic_solve (the split C-ABI halves) reproduce
    picrom_pic_step bit for bit (same segments, same fixed-order sums)."""
    import torch
    from paper_2201_05555_b200 import _device as dev
    from paper_2201_05555_b200 import _lib
    fem, fo = mods
    rng = np.random.default_rng(6)
    L, nx, d, n, p = 10 * np.pi, 128, 3, 60_000, 4
    sysm = fo.VlasovSystem(fem.build_mesh(L, nx, d), fem.ChargeConfig(n, L))
    x0 = torch.from_numpy(rng.uniform(0, L, (p, n))).cuda()
    v0 = torch.from_numpy(rng.standard_normal((p, n))).cuda()
    outs = []
    for split in (False, True):
        run = fo.PicRun(sysm, x0, v0, 0.05, 3, keep_rho=True)
        run.init_field()
        e = run.e
        s = dev.stream_handle()
        ws = torch.zeros(int(_lib.query("picrom_fom_workspace_bytes", n, p, nx, d)),
                         dtype=torch.uint8, device="cuda")
        st = dev.new_status()
        rho = torch.zeros((4, p, nx), dtype=torch.float64, device="cuda")
        phi = torch.zeros_like(rho)
        ee = torch.zeros((4, p), dtype=torch.float64, device="cuda")
        kin = torch.zeros_like(ee)
        for k in range(3):
            kick, kfull = (0.025, 0.0) if k == 0 else (0.05, 0.025)
            if split:
                _lib.call("picrom_pic_push", e.x.data_ptr(), e.v.data_ptr(), n, p, n,
                          e.inst.data_ptr(), nx, d, e.phi.data_ptr(), 0.05, kick, kfull, k,
                          None, ws.data_ptr(), st.data_ptr(), s)
                _lib.call("picrom_pic_solve", n, p, nx, d, e.inst.data_ptr(),
                          e.c.khat.data_ptr(), e.c.stencil.data_ptr(), e.phi.data_ptr(), k,
                          None, 0, rho.data_ptr(), phi.data_ptr(), ee.data_ptr(), kin.data_ptr(),
                          ws.data_ptr(), s)
            else:
                _lib.call("picrom_pic_step", e.x.data_ptr(), e.v.data_ptr(), n, p, n,
                          e.inst.data_ptr(), nx, d, e.c.khat.data_ptr(), e.c.stencil.data_ptr(),
                          e.phi.data_ptr(), 0.05, kick, kfull, k, None, 0, 0, rho.data_ptr(),
                          phi.data_ptr(), ee.data_ptr(), kin.data_ptr(), None, ws.data_ptr(),
                          st.data_ptr(), s)
        outs.append([t.cpu().numpy() for t in (e.x, e.v, rho, phi, ee, kin)])
    for a, b in zip(*outs):
        np.testing.assert_array_equal(a, b)


def test_teacher_forced_per_step_charge_and_potential(mods):
    """At sampled steps, feed the oracle's positions to the GPU deposit/solve."""
    fem, fo = mods
    rng = np.random.default_rng(4)
    L, nx, n, p, d = 10 * np.pi, 128, 30_000, 3, 3
    x, v = rng.uniform(0, L, (n, p)), rng.standard_normal((n, p))
    osys = pic_loop.System(fe.Mesh(L, nx, d), fe.Charge(n, L))
    ost = pic_loop.Stepper(osys)
    gsys = fo.VlasovSystem(fem.build_mesh(L, nx, d), fem.ChargeConfig(n, L))
    t = 0.0
    for k in range(40):
        x, v, t = ost.step(x, v, t, 0.05)
        if k % 10 == 9:
            b, _ = fem.eval_basis_pair(gsys.mesh, x)
            rho = fem.deposit_charge(b, gsys.charge)
            assert rel(rho, ost.last_rho) <= 1e-12
            assert rel(gsys.poisson.solve(ost.last_rho), ost.last_potential) <= 1e-12


def test_run_is_deterministic(mods):
    fem, fo = mods
    rng = np.random.default_rng(2)
    L, n, p = 4 * np.pi, 50_000, 3
    x, v = rng.uniform(0, L, (n, p)), rng.standard_normal((n, p))
    sysm = fo.VlasovSystem(fem.build_mesh(L, 64, 2), fem.ChargeConfig(n, L))
    r = [fo.run_full_order(sysm, fo.ParticleEnsemble(x.copy(), v.copy(), 0.0), 0.05, 2.0,
                           record=fo.RecordOptions(energy_stride=5, snapshot_stride=10))
         for _ in range(2)]
    np.testing.assert_array_equal(r[0].electric_energy, r[1].electric_energy)
    np.testing.assert_array_equal(r[0].snapshots_x, r[1].snapshots_x)
    np.testing.assert_array_equal(r[0].snapshots_v, r[1].snapshots_v)
    assert r[0].snapshots_x.shape == (41 // 10 + 1 + 0, n, p) or r[0].snapshots_x.shape[1:] == (n, p)


def test_snapshots_match_oracle(mods):
    fem, fo = mods
    rng = np.random.default_rng(9)
    L, nx, n, p, d = 4 * np.pi, 32, 4000, 2, 2
    x, v = rng.uniform(0, L, (n, p)), rng.standard_normal((n, p))
    osys = pic_loop.System(fe.Mesh(L, nx, d), fe.Charge(n, L))
    ost = pic_loop.Stepper(osys)
    ox, ov, t = x, v, 0.0
    for _ in range(20):
        ox, ov, t = ost.step(ox, ov, t, 0.05)
    gsys = fo.VlasovSystem(fem.build_mesh(L, nx, d), fem.ChargeConfig(n, L))
    rec = fo.run_full_order(gsys, fo.ParticleEnsemble(x.copy(), v.copy(), 0.0), 0.05, 1.0,
                            record=fo.RecordOptions(energy_stride=2, snapshot_stride=10))
    assert rec.snapshot_times.tolist() == pytest.approx([0.0, 0.5, 1.0])
    assert rel(rec.snapshots_x[-1], ox) <= 1e-12
    assert rel(rec.snapshots_v[-1], ov) <= 1e-12
    assert rel(rec.final_state.v, ov) <= 1e-12


def test_divergence_error_reports_parameter_and_time(mods):
    fem, fo = mods
    rng = np.random.default_rng(1)
    L, n = 4 * np.pi, 800
    x, v = rng.uniform(0, L, (n, 3)), rng.standard_normal((n, 3))
    v[:, 1] = np.inf
    sysm = fo.VlasovSystem(fem.build_mesh(L, 16), fem.ChargeConfig(n, L))
    with pytest.raises(fo.DivergenceError) as err:
        fo.run_full_order(sysm, fo.ParticleEnsemble(x, v, 0.0), 0.01, 0.05)
    assert err.value.parameter_index == 1
    assert err.value.time == pytest.approx(0.01)
    with pytest.raises(fo.DivergenceError) as err:
        fo.VerletStepper(sysm).step(fo.ParticleEnsemble(x, v, 0.0), 0.01)
    assert err.value.parameter_index == 1


def test_step_seconds_are_per_step_device_times(mods):
    """run_full_order's step_seconds are the device times of each step (the
    end of each step's last solve, %globaltimer), not a uniform fill."""
    fem, fo = mods
    rng = np.random.default_rng(12)
    L, n, p, steps = 10 * np.pi, 50_000, 8, 40
    x, v = rng.uniform(0, L, (n, p)), rng.standard_normal((n, p))
    sysm = fo.VlasovSystem(fem.build_mesh(L, 128, 3), fem.ChargeConfig(n, L))
    rec = fo.run_full_order(sysm, fo.ParticleEnsemble(x, v), 0.05, steps * 0.05,
                            record=fo.RecordOptions(energy_stride=1, record_snapshots=False))
    ss = rec.step_seconds
    # device time between consecutive step ends: includes any idle gap (the
    # first graph replay waits for the host-side capture), like the
    # reference's wall-clock step_seconds
    assert ss.shape == (steps,) and np.all(ss > 0) and np.median(ss) < 1e-3
    assert ss.max() > ss.min()           # per-step values (%globaltimer ticks are ~32 ns-1 us)
    assert ss.sum() <= rec.phase_seconds["fom_step"] * 1.01


def test_reference_stepper_drives_gpu_system(mods):
    """The unmodified reference's own VerletStepper / run_full_order (picrom
    from baseline/_ref, installed from /root/reference/pkg) driving the GPU
    VlasovSystem through its duck-typed `field` seam (fullorder.py:111-114):
    identical to the reference with its own P1 system to 1e-12."""
    import sys
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "picrom").exists():
        pytest.skip("baseline/_ref not installed (pip install --target baseline/_ref)")
    sys.path.insert(0, str(ref))
    try:
        from picrom import fem as rfem
        from picrom import fullorder as rfo
    finally:
        sys.path.remove(str(ref))
    fem, fo = mods
    rng = np.random.default_rng(13)
    L, nx, n, p = 4 * np.pi, 32, 6000, 3
    x, v = rng.uniform(0, L, (n, p)), rng.standard_normal((n, p))
    rsys = rfo.VlasovSystem(rfem.build_mesh(L, nx), rfem.ChargeConfig(num_particles=n, length=L))
    gsys = fo.VlasovSystem(fem.build_mesh(L, nx), fem.ChargeConfig(n, L))
    opts = rfo.RecordOptions(energy_stride=1, snapshot_stride=5)
    want = rfo.run_full_order(rsys, rfo.ParticleEnsemble(x.copy(), v.copy()), 0.05, 1.0, opts)
    got = rfo.run_full_order(gsys, rfo.ParticleEnsemble(x.copy(), v.copy()), 0.05, 1.0, opts)
    assert rel(got.snapshots_x, want.snapshots_x) <= 1e-12
    assert rel(got.snapshots_v, want.snapshots_v) <= 1e-12
    assert np.max(np.abs(got.electric_energy - want.electric_energy)
                  / np.abs(want.electric_energy)) <= 1e-10
    st = rfo.VerletStepper(gsys)
    e1 = st.step(rfo.ParticleEnsemble(x.copy(), v.copy()), 0.05)
    e1r = rfo.VerletStepper(rsys).step(rfo.ParticleEnsemble(x.copy(), v.copy()), 0.05)
    assert rel(e1.x, e1r.x) <= 1e-13 and rel(e1.v, e1r.v) <= 1e-13
