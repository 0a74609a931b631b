"""Timing experiment (dev tool, needs the PICROM_EXP_TIMING variant): globaltimer
stamps through the C2 step kernel's last-CTA solve tail for instance 0."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2201_05555_b200 import _device as dev, _lib, fem, fullorder, workloads as wl  # noqa

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
w = wl.config(cfg)
xh, vh = wl.generate(w, layout="pn")
p, n = xh.shape
L = float(w.lengths[0])
sysm = fullorder.VlasovSystem(fem.build_mesh(L, w.num_cells, w.degree), fem.ChargeConfig(n, L))
run = fullorder.PicRun(sysm, torch.from_numpy(xh).cuda(), torch.from_numpy(vh).cuda(), w.dt, 40)
run.init_field()
run.advance(1)
e = run.e
lib = _lib.load()
f = lib.picrom_debug_timestamps
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
rows = []
for it in range(12):
    flush.zero_()
    torch.cuda.synchronize()
    _lib.call("picrom_pic_step", e.x.data_ptr(), e.v.data_ptr(), n, p, n, e.inst.data_ptr(), e.nx,
              e.degree, e.c.khat.data_ptr(), e.c.stencil.data_ptr(), e.phi.data_ptr(), e.dt, e.dt,
              0.5 * e.dt, 0, e.counter.data_ptr(), e.ring, e.r_rho.data_ptr(), e.r_phi.data_ptr(),
              e.r_ee.data_ptr(), e.r_kin.data_ptr(), e.ws.data_ptr(), e.status.data_ptr(),
              dev.stream_handle())
    torch.cuda.synchronize()
    ts = (C.c_ulonglong * 16)()
    f(ts)
    t = np.array(ts[:9], dtype=np.int64)
    rows.append(t - t[0])
r = np.median(np.array(rows[2:]), axis=0)
names = ["start", "loop end (inst0 last seg)", "fold end", "ticket won", "rho assembled",
         "mean rho", "circulant+partition", "phi mean+writes", "energy"]
for k, nm in enumerate(names):
    print(f"{nm:28s} {r[k] / 1e3:8.2f} us")
