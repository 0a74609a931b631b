"""Config-scale parity fixtures: the CPU oracle (oracle/) run on BASELINE.json's
own workloads (paper_2201_05555_b200.workloads, seeded), too slow to repeat
inside the GPU test budget.  Run in the build container:

    python tests/golden/make_config_golden.py C2        # full C2: 8 M particles, 500 steps
    python tests/golden/make_config_golden.py C3r       # C3 reduced run, N = 5e4, 200 steps
    python tests/golden/make_config_golden.py C4r       # C4 at N = 5e4: warm-up, first DEIM fit, failure

Each writes tests/golden/config_<name>.npz with small arrays only (energy
histories, charge/potential at sampled steps, fixed-point counts, DEIM
indices, final Z, sampled rows of U).  The inputs are regenerated bit for bit
on the GPU box from the same seeds (workloads.generate is pure numpy), so
tests/test_config_parity_gpu.py compares the GPU path against these files.
The oracle is test infrastructure; pinned to the reference at degree 1
(tests/golden/make_golden.py), property-pinned at degrees 2/3.
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
OUT = Path(__file__).resolve().parent

# sampled steps of the C2 run whose charge/potential are stored
C2_SAMPLE_STEPS = (1, 100, 250, 400, 500)
# reduced runs: N, steps, energy stride, U rows stored
ROM_N, ROM_STEPS, ROM_ESTRIDE = 50_000, 200, 5
ROM_ROWS = np.r_[0:16, 24_990:25_006, 49_984:50_016, 50_000:50_016, 99_984:100_000]


def make_c2():
    import os
    from oracle import fe_bspline as fe
    from oracle import pic_loop
    from paper_2201_05555_b200 import workloads as wl
    w = wl.config("C2")
    x, v = wl.generate(w)
    n, p = x.shape
    L = float(w.lengths[0])
    cores = len(os.sched_getaffinity(0))
    sysm = pic_loop.System(fe.Mesh(L, w.num_cells, w.degree), fe.Charge(n, L), workers=cores)
    t0 = time.time()
    st = pic_loop.Stepper(sysm)
    t = 0.0
    e0, phi0, rho0 = sysm.field_full(x)
    st.cache_time, st.cache_field, st.last_potential, st.last_rho = t, e0, phi0, rho0
    ees = [fe.electric_energy(sysm.poisson, phi0, sysm.charge)]
    kins = [0.5 * np.einsum("ij,ij->j", v, v)]
    rho_s, phi_s = {}, {}
    for k in range(1, w.num_steps + 1):
        x, v, t = st.step(x, v, t, w.dt)
        ees.append(fe.electric_energy(sysm.poisson, st.last_potential, sysm.charge))
        kins.append(0.5 * np.einsum("ij,ij->j", v, v))
        if k in C2_SAMPLE_STEPS:
            rho_s[k], phi_s[k] = st.last_rho.copy(), st.last_potential.copy()
        if k % 50 == 0:
            print(f"C2 step {k} {time.time() - t0:.0f}s", flush=True)
    np.savez_compressed(
        OUT / "config_C2.npz", electric=np.asarray(ees), kinetic=np.asarray(kins),
        sample_steps=np.asarray(C2_SAMPLE_STEPS),
        rho=np.stack([rho_s[k] for k in C2_SAMPLE_STEPS]),
        phi=np.stack([phi_s[k] for k in C2_SAMPLE_STEPS]),
        x_final_rows=x[:64], v_final_rows=v[:64], seed=w.seed,
        seconds=time.time() - t0)


def make_rom(name):
    from oracle import manifold as mf
    from oracle import rom_loop as orl
    from paper_2201_05555_b200 import workloads as wl
    cfg = name[:2]
    w = wl.config(cfg)
    x0, v0 = wl.generate(w, num_particles=ROM_N)
    params = np.stack([w.wavenumbers, w.alphas], axis=1)
    ex = w.extra
    nb = ex["basis_dim"]
    hyper = cfg == "C4"
    osys = orl.ParamSystem(w.lengths, w.num_cells, w.degree, ROM_N)
    t0 = time.time()
    u0, z0 = mf.csvd_basis(x0, v0, nb)
    h = orl.run_reduced(osys, params, x0, v0, basis_dim=nb, subsample=ex.get("subsample", w.p),
                        window=ex.get("window", 3), deim_dim=ex.get("deim_dim", 8),
                        deim_period=ex.get("deim_period", 3), deim_update=ex.get("deim_update", 2),
                        dt=w.dt, num_steps=ROM_STEPS, hyper_reduction=hyper,
                        energy_stride=ROM_ESTRIDE, snapshot_stride=10**9, u0=u0, z0=z0)
    extra = {}
    if hyper:
        extra["deim_indices"] = np.asarray(h.deim_indices, dtype=np.int64)
        extra["dmd_ranks"] = np.asarray(h.dmd_ranks, dtype=np.int64)
    np.savez_compressed(
        OUT / f"config_{name}.npz", num_particles=ROM_N, steps=ROM_STEPS,
        energy_stride=ROM_ESTRIDE, energy_times=np.asarray(h.energy_times),
        electric=np.asarray(h.electric), kinetic=np.asarray(h.kinetic),
        fp_iterations=np.asarray(h.fp_iterations, dtype=np.int64),
        ortho=np.asarray(h.ortho), sympl=np.asarray(h.sympl), s_conds=np.asarray(h.s_conds),
        sub=np.asarray(h.sub, dtype=np.int64), z0=z0, u0_rows=u0[ROM_ROWS], rows=ROM_ROWS,
        z_final=h.z, u_final_rows=h.u[ROM_ROWS], seed=w.seed, seconds=time.time() - t0,
        **extra)
    print(f"{name}: {time.time() - t0:.0f}s, fp {np.mean(h.fp_iterations):.2f}", flush=True)


def make_c4r():
    """C4 at N = 5e4: the reference algorithm's hyper-reduced fixed point does
    not converge at this particle count (it does at N = 1e6, see the
    full-scale teacher-forced test), so the fixture records the 20 warm-up
    steps, the first DEIM fit at step 21 and the StepFailure it ends in."""
    from oracle import dmd_deim as odd
    from oracle import manifold as mf
    from oracle import rom_loop as orl
    from paper_2201_05555_b200 import workloads as wl
    w = wl.config("C4")
    x0, v0 = wl.generate(w, num_particles=ROM_N)
    params = np.stack([w.wavenumbers, w.alphas], axis=1)
    ex = w.extra
    osys = orl.ParamSystem(w.lengths, w.num_cells, w.degree, ROM_N)
    t0 = time.time()
    u0, z0 = mf.csvd_basis(x0, v0, ex["basis_dim"])
    steps, fits = [], []
    prk2, deim_fit = mf.prk2, odd.deim_fit

    def rec_prk2(*a, **k):
        r = prk2(*a, **k)
        steps.append(r)
        return r

    def rec_fit(*a, **k):
        d = deim_fit(*a, **k)
        fits.append(d)
        return d

    mf.prk2, odd.deim_fit = rec_prk2, rec_fit
    try:
        orl.run_reduced(osys, params, x0, v0, basis_dim=ex["basis_dim"], subsample=ex["subsample"],
                        window=ex["window"], deim_dim=ex["deim_dim"], deim_period=ex["deim_period"],
                        deim_update=ex["deim_update"], dt=w.dt, num_steps=ex["window"] + 1,
                        hyper_reduction=True, energy_stride=10**9, snapshot_stride=10**9,
                        u0=u0, z0=z0)
        raise SystemExit("expected the hyper-reduced fixed point to fail at N = 5e4")
    except mf.StepFailure as err:
        failure = err
    finally:
        mf.prk2, odd.deim_fit = prk2, deim_fit
    last = steps[-1]
    ee, kin = orl._energies(osys, last.u, last.z)
    np.savez_compressed(
        OUT / "config_C4r.npz", num_particles=ROM_N, warm_steps=len(steps),
        fp_iterations=np.asarray([r.fp_iterations for r in steps], dtype=np.int64),
        z_warm=last.z, u_warm_rows=last.u[ROM_ROWS], rows=ROM_ROWS, electric_warm=ee,
        kinetic_warm=kin, deim_indices=np.asarray(fits[0].indices, dtype=np.int64),
        deim_weights=np.asarray(fits[0].weights), fail_iterations=failure.iterations,
        fail_trace=np.asarray(failure.residual_trace), z0=z0, u0_rows=u0[ROM_ROWS],
        seed=w.seed, seconds=time.time() - t0)
    print(f"C4r: {time.time() - t0:.0f}s, warm fp {[r.fp_iterations for r in steps]}, "
          f"fail trace {failure.residual_trace[:3]} ... {failure.residual_trace[-1]:.3e}", flush=True)


def main():
    for name in sys.argv[1:] or ["C2", "C3r", "C4r"]:
        if name == "C2":
            make_c2()
        elif name == "C3r":
            make_rom(name)
        elif name == "C4r":
            make_c4r()
        else:
            raise SystemExit(f"unknown fixture {name}")


if __name__ == "__main__":
    main()
