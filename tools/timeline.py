"""Per-CTA timeline of the fused PIC step (dev tool; needs the
-DPICROM_EXP_TIMELINE library variant via PICROM_LIB):
    PICROM_LIB=.../libpicrom_tl.so python tools/timeline.py [groups] [N p nx d]
Prints, per step, percentiles (us from the step's first CTA entry) of CTA entry,
prologue end, streaming end, fold end, ticket, and the solve-tail ends."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2201_05555_b200 import _lib, fem, fullorder  # noqa: E402

groups = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n, p, nx, d = (int(a) for a in sys.argv[2:6]) if len(sys.argv) > 5 else (250_000, 32, 128, 3)
lib = _lib.load()
fn = lib.picrom_debug_timeline
fn.argtypes = [C.c_void_p, C.c_int, C.c_int]
L = 10 * np.pi
rng = np.random.default_rng(0)
x = torch.from_numpy(rng.uniform(0, L, (p, n))).cuda()
v = torch.from_numpy(np.where(rng.uniform(size=(p, n)) < 0.5, -3.0, 3.0)
                     + 0.3 * rng.standard_normal((p, n))).cuda()
sysm = fullorder.VlasovSystem(fem.build_mesh(L, nx, d), fem.ChargeConfig(n, L))
run = fullorder.PicRun(sysm, x, v, 0.05, 40, keep_rho=False, groups=groups)
run.init_field()
run.advance(4)
torch.cuda.synchronize()
assert fn(None, 0, 1) == 0
steps = 6
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
run.e.launch_block(steps)
ev1.record()
torch.cuda.synchronize()
print(f"groups={run.e.groups}: {ev0.elapsed_time(ev1) / steps * 1e3:.1f} us/step (events)")
buf = np.zeros((16384, 8), dtype=np.uint64)
assert fn(buf.ctypes.data, 16384, 0) == 0
rows = buf[buf[:, 2] > 0].astype(np.float64)
t_all0 = rows[:, 2].min()
names = ["entry", "prologue", "stream_end", "fold", "ticket", "solve_end"]
for stp in sorted(set(rows[:, 0].astype(int))):
    r = rows[rows[:, 0] == stp]
    t0 = r[:, 2].min()
    out = []
    for k, nm in zip(range(2, 8), names):
        col = r[:, k]
        col = col[col > 0]
        if len(col) == 0:
            continue
        q = np.percentile((col - t0) / 1e3, [0, 50, 90, 100])
        out.append(f"{nm} {q[0]:.1f}/{q[1]:.1f}/{q[2]:.1f}/{q[3]:.1f}")
    print(f"step {stp} (+{(t0 - t_all0) / 1e3:.1f} us, {len(r)} CTAs): " + " | ".join(out))

if hasattr(lib, "picrom_debug_timestamps"):
    ts = np.zeros(16, dtype=np.uint64)
    lib.picrom_debug_timestamps.argtypes = [C.c_void_p]
    lib.picrom_debug_timestamps(ts.ctypes.data)
    t = ts.astype(np.float64)
    labels = {3: "solve start", 4: "assembly+khat sync", 5: "mean rho", 6: "circulant+phi sync",
              7: "phi/energy terms", 8: "energy reduce"}
    print("instance 0 solve tail (us since solve start):",
          ", ".join(f"{labels[k]} {(t[k] - t[3]) / 1e3:.2f}" for k in range(4, 9) if t[k] > 0))
