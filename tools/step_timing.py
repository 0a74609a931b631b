"""Fused PIC step timing over (N, p, nx, degree) shapes (dev tool; select the
library with PICROM_LIB).  Back-to-back steps between L2 flushes, CUDA events:
    python tools/step_timing.py [steps [groups,... [shape indices,...]]]
Prints one line per shape: G pushes/s and the fraction of MEASURED_PEAKS hbm."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2201_05555_b200 import fem, fullorder  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
group_opts = [int(g) for g in sys.argv[2].split(",")] if len(sys.argv) > 2 else [None]
peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
    if (ROOT / "MEASURED_PEAKS.json").exists() else 6450.0
shapes = [(250_000, 32, 128, 3), (250_000, 32, 512, 3), (4_000_000, 64, 512, 3),
          (4_000_000, 64, 128, 3), (1_000_000, 8, 64, 2), (250_000, 32, 64, 1)]
if len(sys.argv) > 3:
    shapes = [shapes[int(i)] for i in sys.argv[3].split(",")]
flush = torch.empty(512 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
for (n, p, nx, d) in shapes:
  for groups in group_opts:
    L = 10 * np.pi
    rng = np.random.default_rng(0)
    x = torch.from_numpy(rng.uniform(0, L, (p, n))).cuda()
    v = torch.from_numpy(np.where(rng.uniform(size=(p, n)) < 0.5, -3.0, 3.0)
                         + 0.3 * rng.standard_normal((p, n))).cuda()
    sysm = fullorder.VlasovSystem(fem.build_mesh(L, nx, d), fem.ChargeConfig(n, L))
    run = fullorder.PicRun(sysm, x, v, 0.05, 3 * steps + 10, keep_rho=False, groups=groups)
    run.init_field()
    run.advance(3)
    e = run.e
    res = []
    for rep in range(3):
        flush.zero_()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        e.launch_block(steps)
        ev1.record()
        torch.cuda.synchronize()
        res.append(ev0.elapsed_time(ev1) / steps)
    run.check()
    ms = min(res)
    gps = n * p / (ms / 1e3) / 1e9
    print(f"N={n} p={p} nx={nx} d={d} groups={e.groups}: {ms * 1e3:.1f} us/step  {gps:.1f} G pushes/s  "
          f"{32 * gps / peak:.3f} of HBM", flush=True)
    del run, x, v, sysm
    torch.cuda.empty_cache()
