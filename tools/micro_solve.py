"""Standalone timing of the per-instance Poisson solve (dev tool):
picrom_poisson at C2 shape (p=32, Nx=128, cubic), graph-replayed to remove
launch overhead."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2201_05555_b200 import _build, _lib, fem
from paper_2201_05555_b200 import _device as dev

_build.build()
p = int(sys.argv[1]) if len(sys.argv) > 1 else 32
nx = int(sys.argv[2]) if len(sys.argv) > 2 else 128
d = 3
mesh = fem.build_mesh(2 * 3.141592653589793 / 0.2, nx, degree=d)
c = dev.MeshConstants(nx, d)
inst = dev.inst_rows(mesh, fem.ChargeConfig(250000, mesh.length), p)
rho = torch.randn((p, nx), dtype=torch.float64, device="cuda")
phi = torch.empty_like(rho)
ee = torch.empty(p, dtype=torch.float64, device="cuda")
s = torch.cuda.Stream()
reps = 50


def launch():
    _lib.call("picrom_poisson", rho.data_ptr(), p, nx, d, inst.data_ptr(), c.khat.data_ptr(),
              c.stencil.data_ptr(), phi.data_ptr(), ee.data_ptr(), s.cuda_stream)


with torch.cuda.stream(s):
    launch()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            launch()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(10):
        g.replay()
    e1.record(s)
    torch.cuda.synchronize()
print(f"poisson p={p} nx={nx}: {e0.elapsed_time(e1) / (10 * reps) * 1e3:.2f} us per launch (graph)")
