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
    print("wrote", sorted(p.name for p in OUT.glob("*.npz")))


if __name__ == "__main__":
    main()
