"""Piece timing of hyper._window_svd at C4 size (dev tool): eigh of the window
Gram, the W @ V / W^T Q tall products, CholeskyQR2, the Rayleigh-Ritz SVD."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2201_05555_b200 import hyper  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
T, ps, d = 21, 20, 40
g = torch.Generator(device="cuda").manual_seed(0)
basis = torch.randn((N, 60), dtype=torch.float64, device="cuda", generator=g)
scale = torch.logspace(0, -8, 60, dtype=torch.float64, device="cuda")
win = hyper.DeimWindow(T)
for i in range(T):
    mix = torch.randn((60, ps), dtype=torch.float64, device="cuda", generator=g)
    win.append((basis * scale) @ mix + 1e-12 * torch.randn((N, ps), dtype=torch.float64, device="cuda", generator=g))
W, G = win.matrix()


def t(name, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    print(f"{name:34s} {1e3 * (time.perf_counter() - t0) / reps:8.2f} ms", flush=True)
    return out


Gd = torch.from_numpy(np.ascontiguousarray(G)).cuda()
t("eigh 420 (cuSOLVER via torch)", lambda: torch.linalg.eigh(Gd))
t("eigh 420 (host LAPACK)", lambda: np.linalg.eigh(G))
V = torch.randn((W.shape[1], 48), dtype=torch.float64, device="cuda")
Q = torch.linalg.qr(torch.randn((N, 48), dtype=torch.float64, device="cuda"))[0]
Vh = V.cpu().numpy()
t("W @ V (torch, cuBLAS)", lambda: W @ V)
t("W @ V (_mul, picrom_combine)", lambda: hyper._mul(W, Vh))
t("W^T Q (_tsq, picrom_tall_atb)", lambda: hyper._tsq(W, Q))
t("W^T Q (torch matmul, cuBLAS)", lambda: (W.T @ Q).cpu())
t("new block^T W (_tsq 20 x 420)", lambda: hyper._tsq(W[:, :ps], W))
t("Q^T Q (_tsq)", lambda: hyper._tsq(Q, Q))
t("orthonormalize (CholQR2)", lambda: hyper._orthonormalize(Q))
t("window append", lambda: win.append(W[:, :ps].clone()), reps=1)
t("_window_svd total", lambda: hyper._window_svd(win, d), reps=2)

# piece timing inside _window_svd (each helper wrapped, device-synchronised)
import collections
acc = collections.defaultdict(lambda: [0.0, 0])


def wrap(mod, name, label=None):
    fn = getattr(mod, name)

    def inner(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn(*a, **k)
        torch.cuda.synchronize()
        key = label or name
        if name == "_tsq":
            key = f"_tsq {a[0].shape[1]}x{a[1].shape[1]}"
        if name == "_mul":
            key = f"_mul {a[0].shape[1]}->{a[1].shape[1]}"
        acc[key][0] += time.perf_counter() - t0
        acc[key][1] += 1
        return out
    setattr(mod, name, inner)


import scipy.linalg  # noqa: E402
wrap(hyper, "_tsq")
wrap(hyper, "_mul")
wrap(hyper, "svd", "host svd (Rayleigh-Ritz)")
wrap(hyper.DeimWindow, "eigh", "window.eigh")
wrap(np.linalg, "cholesky", "host cholesky")
wrap(np.linalg, "inv", "host inv")
reps = 3
t0 = time.perf_counter()
for _ in range(reps):
    hyper._window_svd(win, d)
torch.cuda.synchronize()
tot = (time.perf_counter() - t0) / reps
print(f"_window_svd instrumented total {1e3 * tot:.2f} ms")
for k, (s, c) in sorted(acc.items(), key=lambda kv: -kv[1][0]):
    print(f"  {k:30s} {1e3 * s / reps:8.2f} ms  x {c / reps:.1f}")
