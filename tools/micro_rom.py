"""Per-kernel timing of the reduced-basis F-evaluation and manifold kernels at
C3 size (dev tool): rom_field, rom_gather, paired_gram, combine."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2201_05555_b200 import _build, _tall, driver
from paper_2201_05555_b200 import _device as dev
from paper_2201_05555_b200 import _lib

_build.build()
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
p, n, nx, d = 128, 20, 64, 2
rng = np.random.default_rng(0)
lengths = 2 * np.pi / rng.uniform(0.4, 0.6, p)
sysm = driver.ParametricVlasovSystem(lengths, nx, d, N)
u = torch.from_numpy(np.linalg.qr(rng.standard_normal((2 * N, n)))[0]).cuda()
z = rng.standard_normal((n, p)) * 30.0


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(reps):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / reps


cols = driver._Cols(None, p)
zd = torch.from_numpy(z).cuda()
inst = sysm._inst
phi = torch.empty((p, nx), dtype=torch.float64, device="cuda")
ws = driver._rom_ws(N, p, n, nx)
st = dev.new_status()
c = sysm.poisson.constants
s = dev.stream_handle()


def field():
    _lib.call("picrom_rom_field", u.data_ptr(), N, n, zd.data_ptr(), p, p, None, inst.data_ptr(),
              nx, d, c.khat.data_ptr(), c.stencil.data_ptr(), phi.data_ptr(), None, None,
              ws.data_ptr(), st.data_ptr(), None, s)


gout = torch.empty((n, p), dtype=torch.float64, device="cuda")
e = torch.empty((N, p), dtype=torch.float64, device="cuda")


def gather():
    _lib.call("picrom_rom_gather", u.data_ptr(), N, n, zd.data_ptr(), p, p, None, inst.data_ptr(),
              nx, d, phi.data_ptr(), 0, gout.data_ptr(), p, None, None, 0, ws.data_ptr(),
              st.data_ptr(), None, s)


def gather_e():
    _lib.call("picrom_rom_gather", u.data_ptr(), N, n, zd.data_ptr(), p, p, None, inst.data_ptr(),
              nx, d, phi.data_ptr(), 0, None, 0, None, e.data_ptr(), p, ws.data_ptr(),
              st.data_ptr(), None, s)


xi = torch.randn_like(u)


def gram2():
    _tall.gram([(u, False), (xi, False)])


def comb():
    _tall.combine([(u, np.eye(n), False), (xi, np.eye(n), False)])


def full_stage():
    g = driver.make_full_stage(sysm)(u)
    g(z)


res = {}
for name, fn in [("rom_field", field), ("rom_gather(project)", gather), ("rom_gather(E out)", gather_e),
                 ("gram[U,xi]", gram2), ("combine 2 terms", comb)]:
    res[name] = timeit(fn)
t0 = time.perf_counter()
g = driver.make_full_stage(sysm)(u)
for _ in range(5):
    g(z)
torch.cuda.synchronize()
res["full_stage g(z) host-incl"] = (time.perf_counter() - t0) / 5 * 1e3
for k, v in res.items():
    print(f"{k:28s} {v:9.3f} ms")
