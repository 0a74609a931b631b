"""Kernel-time table of reduced steps (dev tool): torch.profiler (CUPTI) over
the last `steps` steps of a C3/C4 run at full size; prints device time per
kernel name per step and the library (cuBLAS/cuSOLVER) share.
    python tools/prof_rom_kernels.py C4 [steps]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2201_05555_b200 import driver, reduction, workloads as wl  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = wl.config(cfg)
x0, v0 = wl.generate(w)
params = np.stack([w.wavenumbers, w.alphas], axis=1)
ex = w.extra
system = driver.ParametricVlasovSystem(w.lengths, w.num_cells, w.degree, w.num_particles)
u0, z0 = reduction.complex_svd_basis(x0, v0, ex["basis_dim"], device=True)
hyper = cfg.upper() == "C4"
warm = (ex.get("window", 3) + 3) if hyper else 3
total = warm + steps
state = {"k": 0, "prof": None}
orig = driver.prk2_step


def hooked(*a, **k):
    state["k"] += 1
    if state["k"] == warm + 1:
        torch.cuda.synchronize()
        state["prof"] = torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA])
        state["prof"].__enter__()
    return orig(*a, **k)


driver.prk2_step = hooked
rec = driver.run_reduced(system, params, x0, v0, basis_dim=ex["basis_dim"],
                         subsample=ex.get("subsample", w.p), window=ex.get("window", 3),
                         deim_dim=ex.get("deim_dim", 8), deim_period=ex.get("deim_period", 3),
                         deim_update=ex.get("deim_update", 2), dt=w.dt, t_final=total * w.dt,
                         hyper_reduction=hyper, energy_stride=10**9, record_snapshots=False,
                         decomp_stride=10**9, u0=u0, z0=z0)
torch.cuda.synchronize()
state["prof"].__exit__(None, None, None)
ev = state["prof"].key_averages()
rows = [(e.key, e.device_time_total / 1e3 / steps, e.count / steps) for e in ev if e.device_time_total > 0]
rows.sort(key=lambda r: -r[1])
tot = sum(r[1] for r in rows)
lib = sum(r[1] for r in rows if any(t in r[0].lower() for t in ("gemm", "cublas", "cusolver", "syevd",
                                                                   "potrf", "cutlass", "sm90", "sm100")))
print(f"{cfg}: device ms per step {tot:.2f} (library kernels {lib:.2f}), fp iterations "
      f"{rec.fp_iterations[-steps:].tolist()}")
for name, ms, cnt in rows[:30]:
    print(f"  {ms:8.3f} ms  x{cnt:6.1f}  {name[:110]}")
