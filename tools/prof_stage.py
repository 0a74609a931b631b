"""cProfile of the reduced-step host path at C3 size (dev tool)."""
import cProfile, pstats, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2201_05555_b200 import _build, driver, reduction
_build.build()
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
p, n, nx, d = 128, 20, 64, 2
rng = np.random.default_rng(0)
lengths = 2 * np.pi / rng.uniform(0.4, 0.6, p)
sysm = driver.ParametricVlasovSystem(lengths, nx, d, N)
u = torch.from_numpy(np.linalg.qr(rng.standard_normal((2 * N, n)))[0]).cuda()
z = rng.standard_normal((n, p)) * 30.0
g = driver.make_full_stage(sysm)(u)
g(z); torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
t = time.perf_counter()
for _ in range(5): g(z)
torch.cuda.synchronize()
print("g(z) ms", (time.perf_counter() - t) / 5 * 1e3)
sub = np.arange(p)
gs = driver.exact_gradients_device(sysm, u, z, sub, harvest=False)[0]
torch.cuda.synchronize()
t = time.perf_counter()
xi = reduction.basis_velocity(u, z, gs)
torch.cuda.synchronize(); print("basis_velocity ms", (time.perf_counter() - t) * 1e3)
t = time.perf_counter()
r = reduction.retraction(u, xi)
torch.cuda.synchronize(); print("retraction ms", (time.perf_counter() - t) * 1e3)
t = time.perf_counter()
tv = reduction.tangent_velocity(u, xi, r, xi)
torch.cuda.synchronize(); print("tangent ms", (time.perf_counter() - t) * 1e3)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
