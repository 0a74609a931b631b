"""Compare-mode diagnostics and phase timers -- mirror of picrom.diagnostics.

* relative_errors / total_relative_error / target_projection_errors /
  numerical_rank / hamiltonian_relative_error (diagnostics.py:44-86): the
  N-sized work on the device -- Frobenius norms by picrom_diff_sumsq, the
  reduced reconstruction U Z by picrom_combine, the local complex-SVD basis of
  the target errors by reduction.complex_svd_basis_device (the projection is
  invariant to the basis' per-vector phase), singular values for the rank
  count from the device Gram (eigenvalues; tolerances below 1e-7 relative are
  handed to an exact SVD on the host, where the Gram's squared conditioning
  would blur the count).
* PhaseTimers (diagnostics.py:169-195): wall time per labelled phase with a
  per-step series; the reduced loop brackets its phases exactly as the
  reference does (rom_basis, rom_coeff, dmd_fit, deim_fit).  Device work is
  asynchronous, so a phase that ends in a host read (every phase of the
  reduced step does) measures device time too.
"""

from __future__ import annotations

import time
from collections import defaultdict
from contextlib import contextmanager

import numpy as np
import torch

from .errors import ConfigurationError

__all__ = ["relative_errors", "total_relative_error", "target_projection_errors",
           "numerical_rank", "hamiltonian_relative_error", "PhaseTimers"]


def _dev(a):
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to("cuda")


_WS = {}


def _sumsq(a, b=None):
    """(||a - b||^2, ||a||^2) of two equally shaped arrays on the device."""
    from . import _device as dev
    from . import _lib
    ad = _dev(a)
    bd = _dev(b) if b is not None else None
    if bd is not None and tuple(bd.shape) != tuple(ad.shape):
        raise ConfigurationError("snapshot shapes do not match")
    key = torch.cuda.current_device()
    ws = _WS.get(key)
    if ws is None:
        ws = _WS[key] = torch.empty(8 * 1024 * 2, dtype=torch.float64, device="cuda")
    out = torch.empty(2, dtype=torch.float64, device="cuda")
    _lib.call("picrom_diff_sumsq", ad.data_ptr(), dev.ptr(bd), ad.numel(), out.data_ptr(),
              ws.data_ptr(), dev.stream_handle())
    d, q = out.cpu().numpy()
    return float(d), float(q)


def _rel(ref, approx):
    d, q = _sumsq(ref, approx)
    if q == 0.0:
        raise ConfigurationError("relative error undefined for a zero reference")
    return float(np.sqrt(d) / np.sqrt(q))


def relative_errors(sx, sv, xr, vr):
    """Componentwise Frobenius relative errors of a reduced snapshot (diagnostics.py:50-54)."""
    if tuple(np.shape(sx)) != tuple(np.shape(xr)) or tuple(np.shape(sv)) != tuple(np.shape(vr)):
        raise ConfigurationError("snapshot shapes do not match")
    return _rel(sx, xr), _rel(sv, vr)


def total_relative_error(sx, sv, xr, vr):
    """Relative error of the stacked phase-space snapshot (diagnostics.py:57-61)."""
    dx, qx = _sumsq(sx, xr)
    dv, qv = _sumsq(sv, vr)
    if qx + qv == 0.0:
        raise ConfigurationError("relative error undefined for a zero reference")
    return float(np.sqrt(dx + dv) / np.sqrt(qx + qv))


def target_projection_errors(sx, sv, n):
    """Errors after projecting the snapshot onto its own local cSVD basis of
    dimension n (diagnostics.py:64-70)."""
    from .reduction import complex_svd_basis_device, reconstruct
    sxd = _dev(sx)
    svd_ = _dev(sv)
    if sxd.dim() == 1:
        sxd, svd_ = sxd.reshape(-1, 1), svd_.reshape(-1, 1)
    u, z = complex_svd_basis_device(sxd, svd_, n)
    xr, vr = reconstruct(u, z)
    return _rel(sxd, xr), _rel(svd_, vr)


def numerical_rank(a, tol):
    """Number of singular values within tol of the largest (diagnostics.py:73-82)."""
    from . import _tall
    if not 0.0 < tol < 1.0:
        raise ConfigurationError(f"rank tolerance must be in (0, 1), got {tol}")
    if tol < 1e-7 or min(np.shape(a)) > 256:
        a = a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
        if not np.any(a):
            return 0
        s = np.linalg.svd(a, compute_uv=False)
        return int((s >= tol * s[0]).sum())
    ad = _dev(a)
    if ad.dim() == 1:
        ad = ad.reshape(-1, 1)
    if ad.shape[0] < ad.shape[1]:
        ad = ad.t().contiguous()
    lam = np.linalg.eigvalsh(_tall.gram([(ad, False)]))
    if lam[-1] <= 0.0:
        return 0
    s = np.sqrt(np.clip(lam, 0.0, None))
    return int((s >= tol * s[-1]).sum())


def hamiltonian_relative_error(h_ref, h_approx):
    """2-norm relative error over the per-parameter Hamiltonian vector (diagnostics.py:85-86)."""
    h_ref = np.atleast_1d(np.asarray(h_ref, dtype=float))
    h_approx = np.atleast_1d(np.asarray(h_approx, dtype=float))
    denom = np.linalg.norm(h_ref)
    if denom == 0.0:
        raise ConfigurationError("relative error undefined for a zero reference")
    return float(np.linalg.norm(h_ref - h_approx) / denom)


class PhaseTimers:
    def __init__(self, names=("fom_step", "rom_basis", "rom_coeff", "dmd_fit", "deim_fit")):
        self.names = tuple(names)
        self.totals = {k: 0.0 for k in self.names}
        self.series = {k: [] for k in self.names}
        self._current = defaultdict(float)

    @contextmanager
    def phase(self, name):
        t0 = time.perf_counter()
        try:
            yield
        finally:
            el = time.perf_counter() - t0
            self.totals[name] = self.totals.get(name, 0.0) + el
            self._current[name] += el

    def flush_step(self):
        for k in self.names:
            self.series[k].append(self._current.get(k, 0.0))
        self._current.clear()

    def series_arrays(self):
        return {k: np.asarray(v) for k, v in self.series.items()}
