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
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def measure(config="C3", n=0, steps=5, warmup=2):
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
    u0, z0 = complex_svd_basis(x0, v0, nb, device=True)
    init_s = time.perf_counter() - t0
    torch.cuda.synchronize()
    rec = driver.run_reduced(
        system, params, x0, v0, basis_dim=nb, subsample=sub, window=window,
        deim_dim=ex.get("deim_dim", 8), deim_period=ex.get("deim_period", 3),
        deim_update=ex.get("deim_update", 2), dt=w.dt, t_final=total * w.dt,
        hyper_reduction=hyper, energy_stride=10**9, record_snapshots=False,
        decomp_stride=10**9, timers=timers, u0=u0, z0=z0)
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
    return {
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
        "timing": "host wall clock per PRK2 step (PhaseTimers rom_basis+rom_coeff), "
                  "the step's n x n LAPACK algebra and fixed-point convergence checks included",
        "dmd_ranks": rec.dmd_ranks[-steps:].tolist(),
        "ortho_residual_last": float(rec.ortho_residuals[-1]),
        "generation_s": gen_s, "init_csvd_s": init_s,
    }


FP64_PEAK_TF = 37.2     # measured DMMA peak on this pool's B200 (DFMA: 36.4; cuBLAS DGEMM: 35.5)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    args = ap.parse_args()
    print(json.dumps(measure(args.config, args.n, args.steps, args.warmup)), flush=True)


if __name__ == "__main__":
    main()
