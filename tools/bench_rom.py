#!/usr/bin/env python
"""Reduced-model benchmark (BASELINE C3 / C4) on one B200.

    python tools/bench_rom.py --config C3 [--n 1000000] [--steps 5] [--warmup 2]
    python tools/bench_rom.py --config C4 [--n 1000000] [--steps 5]

A step is one `driver.run_reduced` time step (the PRK2 step with its exact
subsample gradients, the fixed-point stage and, in C4, the DMD/DEIM fits),
timed by the reference's PhaseTimers phases (rom_basis + rom_coeff + dmd_fit +
deim_fit, i.e. excluding the reconstruct-based diagnostics, driver.py:160-173).
pushes/s = N * p / (seconds per step).  Roofline per SURVEY.md §8(d):
B_alg = [2 (E_p + E_*) + 22] N n 8 bytes, F_alg = (E_p p + E_* p*) 4 n N + 36 N n^2 flops.

e2e: the whole public call `driver.run_reduced(..., u0, z0)` from host numpy
U0 (2N x n) and Z0 (n x p), with the final (U, Z) recorded back to host
(record_snapshots at the last step), timed over warm-up + timed steps.
cpu_baseline: the oracle port's reduced step (oracle/rom_loop.py, the
reference algorithm restated for per-instance meshes) at a bounded sample
(same p, n, Nx, degree; N reduced), pushes/s = N p / step seconds.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

FP64_PEAK_TF = 37.2     # measured DMMA peak on this pool's B200 (DFMA: 36.4; cuBLAS DGEMM: 35.5)


def cpu_reduced_rate(config, n=20_000, steps=1):
    """Oracle reduced step on the host cores at N = n (C3: no hyper-reduction).
    C4's hyper-reduced fixed point does not converge below N ~ 1e6 in the
    reference algorithm (tests/golden/config_C4r.npz), so C4 reports None."""
    if config.upper() != "C3":
        return None
    from oracle import manifold as mf
    from oracle import rom_loop as orl
    from paper_2201_05555_b200 import workloads as wl
    w = wl.config(config)
    x0, v0 = wl.generate(w, num_particles=n)
    params = np.stack([w.wavenumbers, w.alphas], axis=1)
    nb = w.extra["basis_dim"]
    osys = orl.ParamSystem(w.lengths, w.num_cells, w.degree, n)
    u0, z0 = mf.csvd_basis(x0, v0, nb)
    t0 = time.perf_counter()
    orl.run_reduced(osys, params, x0, v0, basis_dim=nb, subsample=w.p, window=3, deim_dim=8,
                    deim_period=3, deim_update=2, dt=w.dt, num_steps=steps, hyper_reduction=False,
                    energy_stride=10**9, snapshot_stride=10**9, u0=u0, z0=z0)
    el = (time.perf_counter() - t0) / steps
    cores = len(os.sched_getaffinity(0))
    return {"value": n * w.p / el, "unit": "pushes/s", "cores": cores, "kind": "port",
            "sample": f"{config} reduced step at N = {n} (p = {w.p}, n = {nb}, Nx = {w.num_cells}, "
                      f"degree {w.degree}), {steps} PRK2 step(s) of the numpy oracle port "
                      f"(oracle/rom_loop.py), {el:.1f} s/step"}


def measure(config="C3", n=0, steps=5, warmup=2, e2e=True, cpu=True):
    """Run the reduced model on one GPU and return the bench dict (see module doc)."""
    import torch
    from paper_2201_05555_b200 import _build, driver, workloads as wl
    from paper_2201_05555_b200.diagnostics import PhaseTimers
    _build.build()
    w = wl.config(config)
    n = n or w.num_particles
    t0 = time.perf_counter()
    x0, v0 = wl.generate(w, num_particles=n)
    gen_s = time.perf_counter() - t0
    p = w.p
    params = np.stack([w.wavenumbers, w.alphas], axis=1)
    system = driver.ParametricVlasovSystem(w.lengths, w.num_cells, w.degree, n)
    hyper = config.upper() == "C4"
    ex = w.extra
    nb = ex["basis_dim"]
    sub = ex.get("subsample", p)
    window = ex.get("window", 3)
    total = warmup + steps + (window + 1 if hyper else 0)
    timers = PhaseTimers()
    t0 = time.perf_counter()
    from paper_2201_05555_b200.reduction import complex_svd_basis
    u0, z0 = complex_svd_basis(x0, v0, nb)
    init_s = time.perf_counter() - t0
    from paper_2201_05555_b200.reduction import complex_svd_basis_device
    complex_svd_basis_device(x0[:1000], v0[:1000], nb)          # warm the kernels
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    complex_svd_basis_device(x0, v0, nb)
    torch.cuda.synchronize()
    init_dev_s = time.perf_counter() - t0
    kw = dict(basis_dim=nb, subsample=sub, window=window, deim_dim=ex.get("deim_dim", 8),
              deim_period=ex.get("deim_period", 3), deim_update=ex.get("deim_update", 2), dt=w.dt,
              t_final=total * w.dt, hyper_reduction=hyper, energy_stride=10**9,
              decomp_stride=10**9)
    u0d = torch.from_numpy(u0).to("cuda")
    torch.cuda.synchronize()
    rec = driver.run_reduced(system, params, x0, v0, record_snapshots=False, timers=timers,
                             u0=u0d, z0=z0, **kw)
    ser = timers.series_arrays()
    per_step = sum(ser[k] for k in ("rom_basis", "rom_coeff", "dmd_fit", "deim_fit"))
    timed = per_step[-steps:]
    fp = rec.fp_iterations[-steps:]
    t_step = float(np.mean(timed))
    value = n * p / t_step
    e_star = 2 if hyper else 0
    e_p = 0.0 if hyper else float(np.mean(fp)) + 2
    bytes_alg = (2 * (e_p + e_star) + 22) * n * nb * 8
    flops_alg = (e_p * p + e_star * sub) * 4 * nb * n + 36 * n * nb * nb
    peaks = (json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
             if (ROOT / "MEASURED_PEAKS.json").exists() else {"hbm_gbs": 6650.0})
    out = {
        "metric": "particle-pushes/s (Np x p per reduced step) fp64 on 1 B200",
        "config": config, "value": value, "unit": "pushes/s", "num_particles": n, "p": p,
        "basis_dim": nb, "subsample": sub, "hyper": hyper, "ms_per_step": 1e3 * t_step,
        "fp_iterations_mean": float(np.mean(fp)),
        "phase_ms": {k: 1e3 * float(np.mean(ser[k][-steps:])) for k in ser},
        "roofline": {"bound": "fp64", "achieved": flops_alg / t_step / 1e12, "peak": FP64_PEAK_TF,
                     "unit": "TFLOP/s", "frac": flops_alg / t_step / 1e12 / FP64_PEAK_TF,
                     "flops_alg_per_step": flops_alg, "bytes_alg_per_step": bytes_alg,
                     "hbm_frac_of_alg_bytes": bytes_alg / t_step / 1e9 / peaks["hbm_gbs"],
                     "peak_source": "DMMA m8n8k4 microbenchmark, profiles/r01b/fp64_peak.log"},
        "timing": "host wall clock per PRK2 step (PhaseTimers rom_basis+rom_coeff"
                  + ("+dmd_fit+deim_fit" if hyper else "") + "), the step's n x n LAPACK algebra "
                  "and fixed-point convergence checks included; mean of the last "
                  f"{steps} of {total} steps",
        "dmd_ranks": rec.dmd_ranks[-steps:].tolist(),
        "ortho_residual_last": float(rec.ortho_residuals[-1]),
        "generation_s": gen_s, "init_csvd_s": init_s,
        "init_csvd_device_s": init_dev_s,
        "init_note": "initial basis: host LAPACK complex SVD (reference path, used for the run) vs "
                     "reduction.complex_svd_basis_device (Hermitian Gram on the GPU, same basis up to "
                     "a phase per singular vector; host (N, p) arrays uploaded inside the timing)",
    }
    if e2e:
        del u0d
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rec2 = driver.run_reduced(system, params, x0, v0, record_snapshots=True,
                                  snapshot_stride=total, u0=u0, z0=z0, **kw)
        u_last, z_last = rec2.bases[-1]
        u_host = u_last.cpu().numpy()
        e2e_s = time.perf_counter() - t0
        out["e2e"] = {"value": n * p * total / e2e_s, "unit": "pushes/s",
                      "h2d_bytes_per_step": (u0.nbytes + z0.nbytes) / total,
                      "d2h_bytes_per_step": (u_host.nbytes + np.asarray(z_last).nbytes) / total,
                      "call": f"driver.run_reduced({total} steps) from host numpy U0, Z0; final "
                              "(U, Z) back to host", "seconds": e2e_s}
    if cpu:
        out["cpu_baseline"] = cpu_reduced_rate(config)
        if out["cpu_baseline"] is None:
            out["cpu_baseline_note"] = ("the reference algorithm's hyper-reduced fixed point does "
                                        "not converge below N ~ 1e6 (tests/golden/config_C4r.npz), "
                                        "so no bounded CPU sample of a C4 hyper step exists")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    print(json.dumps(measure(args.config, args.n, args.steps, args.warmup, cpu=not args.no_cpu)),
          flush=True)


if __name__ == "__main__":
    main()
