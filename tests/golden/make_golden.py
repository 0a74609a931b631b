"""Generate golden vectors by running the REFERENCE package (picrom) itself.

Run in the build container, where /root/reference exists:
    python tests/golden/make_golden.py
The fixtures (*.npz) are committed; nothing on the GPU box reads /root/reference.
They pin the CPU oracle (oracle/) at degree 1, where oracle and reference must
agree bit for bit (the oracle generalises the reference to degree 2/3).
Inputs are seeded; every reference call used is named next to its output key.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def main():
    sys.path.insert(0, str(REF))
    from picrom import fem, fullorder  # noqa: E402

    rng = np.random.default_rng(1234)
    length, nx = 4.0 * np.pi, 16
    mesh = fem.build_mesh(length, nx)
    n, p = 257, 3
    x2 = rng.uniform(-length, 2 * length, size=(n, p))
    x2[0, 0] = 0.0                 # on a node
    x2[1, 1] = mesh.h * 5          # on a node (right-cell convention)
    x2[2, 2] = -mesh.h * 3         # negative on node
    x1 = rng.uniform(0, length, size=n)
    charge = fem.ChargeConfig(num_particles=n, length=length)
    poisson = fem.PoissonOperator(mesh)
    out = {"length": length, "nx": nx, "x2": x2, "x1": x1}
    i0, frac = fem._locate(mesh, x2)                          # fem.py:108-116
    out["i0"], out["frac"] = i0, frac
    b2, g2 = fem.eval_basis_pair(mesh, x2)                    # fem.py:193-200
    out["w0"], out["w1"], out["gw0"], out["gw1"] = b2.w0, b2.w1, g2.w0, g2.w1
    rho2 = fem.deposit_charge(b2, charge)                     # fem.py:203-215
    out["rho2"] = rho2
    phi2 = poisson.solve(rho2)                                # fem.py:239-244
    out["phi2"] = phi2
    out["ee2"] = fem.electric_energy(poisson, phi2, charge)   # fem.py:247-251
    out["e2"] = fem.field_at_particles(g2, phi2, charge)      # fem.py:254-256
    out["lam2"] = b2.matvec(phi2)                             # fem.py:138-149
    y = rng.standard_normal((n, p))
    out["y"] = y
    out["rmat2"] = b2.rmatvec(y)                              # fem.py:151-166
    b1 = fem.eval_basis(mesh, x1)
    out["rho1"] = fem.deposit_charge(b1, charge)
    out["phi1"] = poisson.solve(out["rho1"])
    v2 = rng.standard_normal((n, p))
    out["v2"] = v2
    out["ham2"] = fem.hamiltonian(x2, v2, poisson, charge)    # fem.py:259-268
    out["stiffness"] = poisson.stiffness
    np.savez_compressed(OUT / "fem_p1.npz", **out)

    # fullorder: Verlet steps (fullorder.py:122-134) and a recorded run (169-226)
    n, p = 400, 2
    charge = fem.ChargeConfig(num_particles=n, length=length)
    system = fullorder.VlasovSystem(mesh, charge)
    xs = rng.uniform(0, length, size=(n, p))
    vs = rng.standard_normal((n, p))
    ens = fullorder.ParticleEnsemble(xs.copy(), vs.copy(), 0.0)
    st = fullorder.VerletStepper(system)
    e1 = st.step(ens, 0.1)
    e2 = st.step(e1, 0.1)
    rec = fullorder.run_full_order(system, fullorder.ParticleEnsemble(xs.copy(), vs.copy(), 0.0),
                                   0.05, 1.0,
                                   record=fullorder.RecordOptions(energy_stride=1,
                                                                  snapshot_stride=5))
    np.savez_compressed(
        OUT / "fullorder_p1.npz", length=length, nx=nx, x=xs, v=vs,
        x_step1=e1.x, v_step1=e1.v, x_step2=e2.x, v_step2=e2.v, phi_step2=st.last_potential,
        rec_energy=rec.electric_energy, rec_ham=rec.hamiltonian, rec_pot=rec.potentials,
        rec_snap_x=rec.snapshots_x, rec_snap_v=rec.snapshots_v, rec_snap_t=rec.snapshot_times)
    rom_golden()
    print("wrote", sorted(p.name for p in OUT.glob("*.npz")))


def rom_golden():
    """driver.run_reduced (driver.py:117-274) no-hyper and hyper, plus the
    reduction/hyper building blocks, on the reference's tiny test problem
    (pkg/tests/test_driver.py:102-110)."""
    from picrom import driver, fem, fullorder, hyper, reduction
    from picrom.sampling import BENCHMARKS, build_initial_ensemble, sample_parameters

    bench = BENCHMARKS["weak_landau"]
    out = {}
    for tag, npart, ncell, npar in (("a", 240, 16, 6), ("b", 200, 16, 5)):
        params = sample_parameters(bench.alpha_range, bench.sigma_range, npar)
        x0, v0 = build_initial_ensemble(bench, params, npart)
        out[f"{tag}_params"], out[f"{tag}_x0"], out[f"{tag}_v0"] = params, x0, v0
    out["length"], out["nx"] = bench.length, 16

    def system(tag):
        mesh = fem.build_mesh(bench.length, 16)
        return fullorder.VlasovSystem(mesh, fem.ChargeConfig(out[f"{tag}_x0"].shape[0], bench.length))

    # no hyper-reduction (test_driver.py:112-119)
    rec = driver.run_reduced(system("a"), out["a_params"], out["a_x0"], out["a_v0"], basis_dim=4,
                             subsample=4, window=3, deim_dim=8, deim_period=3, deim_update=2,
                             dt=0.02, t_final=0.1, hyper_reduction=False, snapshot_stride=5,
                             energy_stride=1, decomp_stride=10**9)
    out["nohyper_u"], out["nohyper_z"] = rec.bases[-1]
    out["nohyper_ee"], out["nohyper_ham"] = rec.electric_energy, rec.hamiltonian
    out["nohyper_fp"], out["nohyper_ortho"] = rec.fp_iterations, rec.ortho_residuals
    # hyper-reduced (test_driver.py:143-153)
    rec = driver.run_reduced(system("b"), out["b_params"], out["b_x0"], out["b_v0"], basis_dim=4,
                             subsample=4, window=2, deim_dim=12, deim_period=2, deim_update=4,
                             dt=0.01, t_final=0.12, snapshot_stride=4, energy_stride=1,
                             decomp_stride=10**9)
    assert rec.hyper_engaged
    out["hyper_u"], out["hyper_z"] = rec.bases[-1]
    out["hyper_ee"], out["hyper_fp"] = rec.electric_energy, rec.fp_iterations
    out["hyper_ranks"] = rec.dmd_ranks

    # building blocks on random data
    rng = np.random.default_rng(77)
    big, n, p = 50, 6, 9
    xs, vs = rng.standard_normal((big, p)), rng.standard_normal((big, p))
    u, z = reduction.complex_svd_basis(xs, vs, n)
    g = rng.standard_normal((2 * big, p))
    xi = reduction.basis_velocity(u, z, g)
    r = reduction.retraction(u, 0.1 * xi)
    xe = reduction.basis_velocity(r, z, rng.standard_normal((2 * big, p)))
    out.update(bb_x=xs, bb_v=vs, bb_u=u, bb_z=z, bb_g=g, bb_xi=xi, bb_r=r, bb_xe=xe,
               bb_tan=reduction.tangent_velocity(u, 0.1 * xi, r, xe),
               bb_s=reduction.SMatrix(z).matrix,
               bb_sub=reduction.select_parameter_subset(z, 5))
    samples = rng.standard_normal((80, 4)) @ rng.standard_normal((4, 30)) + 1e-3 * rng.standard_normal((80, 30))
    ch = fem.ChargeConfig(80, 2 * np.pi)
    dm = hyper.fit_deim(samples, 10, ch)
    samples2 = samples + 1e-2 * rng.standard_normal((80, 30))
    dm2 = hyper.fit_deim(samples2, 10, ch, prev=dm, full=False, n_update=3)
    out.update(de_samples=samples, de_samples2=samples2, de_psi=dm.psi, de_idx=dm.indices,
               de_w=dm.weights, de_idx2=dm2.indices, de_w2=dm2.weights)
    snaps = [rng.standard_normal(12)]
    a = np.linalg.qr(rng.standard_normal((12, 12)))[0] * 0.98
    for _ in range(8):
        snaps.append(a @ snaps[-1])
    win = [np.stack([s_, 1.1 * s_, 0.9 * s_], axis=1) for s_ in snaps]
    prm = rng.uniform(size=(7, 2))
    model = hyper.fit_parametric_dmd(win, 0.05, 0.4, prm, np.array([1, 3, 5]))
    model.ensure_coords(prm)
    out.update(dmd_prm=prm, dmd_win=np.stack(win), dmd_eigs=model.eigenvalues,
               dmd_phi=model.potential(0.45))
    np.savez_compressed(OUT / "rom_p1.npz", **out)


if __name__ == "__main__":
    main()
