"""Phase timing of fullorder.run_full_order with host (pinned) inputs (dev tool)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_2201_05555_b200 import _device as dev, fem, fullorder, workloads as wl

w = wl.config(sys.argv[1] if len(sys.argv) > 1 else "C2")
steps = int(sys.argv[2]) if len(sys.argv) > 2 else w.num_steps
xh, vh = wl.generate(w, layout="pn")
p, n = xh.shape
L = float(w.lengths[0])
sysm = fullorder.VlasovSystem(fem.build_mesh(L, w.num_cells, w.degree), fem.ChargeConfig(n, L))
xn = torch.from_numpy(np.ascontiguousarray(xh.T)).pin_memory()
vn = torch.from_numpy(np.ascontiguousarray(vh.T)).pin_memory()
T = {}
def tic(k):
    torch.cuda.synchronize(); T[k] = time.perf_counter()
for rep in range(2):
    tic("start")
    xd, meta = dev.to_device(xn); vd, _ = dev.to_device(vn)
    tic("upload")
    run = fullorder.PicRun(sysm, xd, vd, w.dt, steps)
    tic("alloc")
    run.init_field(); run.advance(steps)
    tic("steps")
    vf = run.finish_kinetic()
    tic("finish")
    xo = dev.from_device(run.x, meta); vo = dev.from_device(vf, meta)
    tic("download_state")
    ee = run.ee_hist.cpu().numpy(); ph = run.phi_hist.cpu().numpy(); rh = run.rho_hist.cpu().numpy()
    tic("download_hist")
    ks = list(T)
    print(rep, {ks[i]: round(T[ks[i]] - T[ks[i-1]], 4) for i in range(1, len(ks))})
t0 = time.perf_counter()
rec = fullorder.run_full_order(sysm, fullorder.ParticleEnsemble(xn, vn, 0.0), w.dt, steps * w.dt,
                               record=fullorder.RecordOptions(energy_stride=1, record_snapshots=False))
print("run_full_order", time.perf_counter() - t0)
