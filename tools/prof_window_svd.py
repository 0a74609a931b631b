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
t("W @ V (torch)", lambda: W @ V)
t("W^T Q (_tsq, bmm split-K)", lambda: hyper._tsq(W, Q))
t("W^T Q (torch matmul)", lambda: (W.T @ Q).cpu())
t("Q^T Q (_tsq)", lambda: hyper._tsq(Q, Q))
t("orthonormalize (CholQR2)", lambda: hyper._orthonormalize(Q))
t("window append", lambda: win.append(W[:, :ps].clone()), reps=1)
t("_window_svd total", lambda: hyper._window_svd(win, d), reps=2)
