"""DEIM fit cost at C4 size (dev tool): a window of T+1 = 21 blocks of N x p*
(N = 1e6, p* = 20), d = 40 -- sliding Gram append, windowed SVD, greedy, weights."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2201_05555_b200 import hyper  # noqa: E402
from paper_2201_05555_b200.fem import ChargeConfig  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
T, ps, d = 21, 20, 40
g = torch.Generator(device="cuda").manual_seed(0)
basis = torch.randn((N, 30), dtype=torch.float64, device="cuda", generator=g)
win = hyper.DeimWindow(T)


def block(i):
    mix = torch.randn((30, ps), dtype=torch.float64, device="cuda", generator=g)
    return basis @ mix + 1e-6 * torch.randn((N, ps), dtype=torch.float64, device="cuda", generator=g)


for i in range(T):
    win.append(block(i))


def timed(name, fn, *a, **k):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn(*a, **k)
    torch.cuda.synchronize()
    print(f"{name:28s} {1e3 * (time.perf_counter() - t0):9.2f} ms", flush=True)
    return out


from collections import defaultdict  # noqa: E402
TOT = defaultdict(float)
CNT = defaultdict(int)


def wrap(name):
    fn = getattr(hyper, name)

    def w(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn(*a, **k)
        torch.cuda.synchronize()
        TOT[name] += time.perf_counter() - t0
        CNT[name] += 1
        return out
    setattr(hyper, name, w)


for nm in ("_greedy_device", "_rows", "_orthonormalize", "_tsq"):
    wrap(nm)
_gram0 = hyper._tall.gram


def gram_t(blocks):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = _gram0(blocks)
    TOT["_tall.gram"] += time.perf_counter() - t0
    CNT["_tall.gram"] += 1
    return out


hyper._tall.gram = gram_t
_eigh0 = np.linalg.eigh


def eigh_t(a):
    t0 = time.perf_counter()
    out = _eigh0(a)
    TOT["np.eigh"] += time.perf_counter() - t0
    CNT["np.eigh"] += 1
    return out


hyper.np.linalg.eigh = eigh_t
_comb0 = hyper._tall.combine


def comb_t(*a, **k):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = _comb0(*a, **k)
    torch.cuda.synchronize()
    TOT["_tall.combine"] += time.perf_counter() - t0
    CNT["_tall.combine"] += 1
    return out


hyper._tall.combine = comb_t
charge = ChargeConfig(N, 4 * np.pi)
for rep in range(2):
    timed("window append (x1)", win.append, block(T + rep))
    psi, de = timed("window svd", hyper._window_svd, win, d)
    idx = timed("deim greedy (full)", hyper.deim_greedy, psi)
    timed("fit_deim_device (full)", hyper.fit_deim_device, win, d, charge)

for k in sorted(TOT, key=lambda k: -TOT[k]):
    print(f"  {k:20s} {1e3 * TOT[k] / 2:9.2f} ms per rep   calls/rep {CNT[k] / 2:.0f}")
