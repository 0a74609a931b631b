"""Device plumbing: layout conversion, per-mesh constants, workspaces, status.

Reference-facing calls take the reference's layouts -- particle arrays (N,) or
(N, p) row-major, grid arrays (Nx,) or (Nx, p) -- as numpy arrays or torch
tensors, and return the same kind.  On the device everything is instance-major
(p, N) / (p, Nx) float64 (include/picrom_b200.h), converted by the library's
transpose kernel, never by torch compute.
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass
from fractions import Fraction
from functools import lru_cache

import numpy as np
import torch

from . import _lib
from .errors import ConfigurationError, EvaluationError

ULL_MAX = (1 << 64) - 1
INST_STRIDE = 8


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2201_05555_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    _lib.load()


def stream_handle():
    return torch.cuda.current_stream().cuda_stream


def ptr(t):
    return None if t is None else t.data_ptr()


# ------------------------------------------------------------------ layouts

@dataclass(frozen=True)
class Meta:
    """How to hand a (p, rows) device array back to the caller."""

    kind: str          # "numpy" | "torch"
    ndim: int          # 1 -> (rows,), 2 -> (rows, p)
    device: object = None


def to_device(a):
    """numpy/torch (rows,) or (rows, p) -> contiguous cuda float64 (p, rows), Meta."""
    require_cuda()
    if isinstance(a, torch.Tensor):
        meta = Meta("torch", a.dim(), a.device)
        t = a.detach().to(device="cuda", dtype=torch.float64)
    else:
        arr = np.asarray(a, dtype=np.float64)
        meta = Meta("numpy", arr.ndim)
        t = torch.from_numpy(np.ascontiguousarray(arr)).to("cuda", non_blocking=False)
    if t.dim() == 0:
        t = t.reshape(1)
        meta = Meta(meta.kind, 1, meta.device)
    if t.dim() == 1:
        t = t.contiguous()
        if isinstance(a, torch.Tensor) and t.data_ptr() == a.data_ptr():
            t = t.clone()           # never alias the caller's array (tables are lazy)
        return t.reshape(1, -1), meta
    if t.dim() != 2:
        raise ConfigurationError("particle/grid arrays must be 1-D or 2-D")
    t = t.contiguous()
    rows, p = t.shape
    if p == 1:
        return t.reshape(1, rows).clone(), meta
    out = torch.empty((p, rows), dtype=torch.float64, device="cuda")
    _lib.call("picrom_transpose", t.data_ptr(), rows, p, out.data_ptr(), stream_handle())
    return out, meta


_STAGE = {}
_POOL = None
_PINNED = []                 # [pinned tensor, weakref of the owner of the array handed out | None]
_PINNED_CAP = 6 << 30        # bytes of result buffers kept pinned (C5 state: 2 x 2.05 GB)


class _PinnedResult:
    """Owner of one pinned slot handed out as a numpy array.

    ``np.asarray(owner)`` makes an array whose ``.base`` is this object, and every
    numpy view derived from it (transpose, slice, reshape) collapses its base to
    the same object -- so the slot stays reserved while ANY view is alive, not
    just the array first handed out."""

    def __init__(self, buf, shape, typestr):
        self.buf = buf
        self.__array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                    "data": (buf.data_ptr(), False), "version": 3}


def _slot_free(slot):
    return slot[1] is None or slot[1]() is None


def _free_pinned(numel, dtype):
    # best fit: the smallest idle slot that holds the result, so repeated
    # calls with the same result sizes settle on one slot per result
    fits = [s for s in _PINNED if s[0].dtype == dtype and s[0].numel() >= numel and _slot_free(s)]
    if fits:
        return min(fits, key=lambda s: s[0].numel())
    held = sum(b.numel() * b.element_size() for b, _ in _PINNED)
    if held + numel * 8 > _PINNED_CAP:
        # release idle slots (largest first) before giving up on the pool
        for slot in sorted([s for s in _PINNED if _slot_free(s)], key=lambda s: -s[0].numel()):
            _PINNED.remove(slot)
            held -= slot[0].numel() * slot[0].element_size()
            if held + numel * 8 <= _PINNED_CAP:
                break
        if held + numel * 8 > _PINNED_CAP:
            return None
    slot = [torch.empty(numel, dtype=dtype, pin_memory=True), None]
    _PINNED.append(slot)
    return slot


def to_host(t):
    """Device tensor -> host numpy array.

    Result buffers are pinned host memory recycled across calls: a buffer is
    reused only once the array handed out from it AND every view of that array
    have been dropped (weak reference to a per-result owner object, see
    _PinnedResult), so a result is never overwritten while the caller holds any
    part of it.  Pinning fresh memory costs ~26 ms per 64 MB and a pageable D2H
    ~30 ms, against ~1.3 ms for the D2H into a recycled pinned buffer.  The pool
    is capped (_PINNED_CAP; idle slots are released to make room); beyond it the
    copy goes through one pinned staging buffer and a multi-threaded copy into
    new pageable memory (~10 ms per 64 MB)."""
    global _POOL
    t = t.contiguous()
    nbytes = t.numel() * t.element_size()
    if nbytes < (4 << 20):
        return t.cpu().numpy()
    slot = _free_pinned(t.numel(), t.dtype)
    if slot is not None:
        view = slot[0][:t.numel()]
        view.copy_(t.reshape(-1))
        owner = _PinnedResult(view, t.shape, view.numpy().dtype.str)
        slot[1] = weakref.ref(owner)
        out = np.asarray(owner)
        assert out.base is owner
        return out
    stage = _STAGE.get(t.dtype)
    if stage is None or stage.numel() < t.numel():
        stage = _STAGE[t.dtype] = torch.empty(t.numel(), dtype=t.dtype, pin_memory=True)
    src = stage[:t.numel()]
    src.copy_(t.reshape(-1))
    out = np.empty(t.numel(), dtype=src.numpy().dtype)
    if _POOL is None:
        import os
        from concurrent.futures import ThreadPoolExecutor
        _POOL = ThreadPoolExecutor(max_workers=max(1, min(16, len(os.sched_getaffinity(0)))))
    sv = src.numpy()
    k = _POOL._max_workers
    edges = np.linspace(0, t.numel(), k + 1).astype(np.int64)
    list(_POOL.map(lambda i: np.copyto(out[edges[i]:edges[i + 1]], sv[edges[i]:edges[i + 1]]),
                   range(k)))
    return out.reshape(tuple(t.shape))


def from_device(t_pn, meta, dtype=torch.float64):
    """(p, rows) device array -> the caller's kind/shape, reference layout."""
    p, rows = t_pn.shape
    if meta.ndim == 1:
        out = t_pn.reshape(rows).clone()
    elif p == 1:
        out = t_pn.reshape(rows, 1).clone()
    else:
        out = torch.empty((rows, p), dtype=t_pn.dtype, device="cuda")
        name = "picrom_transpose_i64" if t_pn.dtype == torch.int64 else "picrom_transpose"
        _lib.call(name, t_pn.data_ptr(), p, rows, out.data_ptr(), stream_handle())
    if meta.kind == "numpy" or (meta.device is not None and not str(meta.device).startswith("cuda")):
        host = to_host(out)
        return host if meta.kind == "numpy" else torch.from_numpy(host)
    return out


def per_instance(v_p, meta):
    """(p,) device vector -> scalar for 1-D callers, (p,) otherwise."""
    if meta.kind == "numpy":
        arr = v_p.cpu().numpy()
        return arr[0] if meta.ndim == 1 else arr
    return v_p[0] if meta.ndim == 1 else v_p


# ------------------------------------------------------------ mesh constants

def stencil_rationals(degree):
    """a_k = int N_d'(t) N_d'(t+k) dt (k = 0..d): L_{i,i+-k} = a_k / h."""
    from .splines import stiffness_stencil
    return stiffness_stencil(degree)


@lru_cache(maxsize=64)
def _khat_unit(num_cells, degree):
    """First column of (A + 11^T/Nx)^{-1}, A = h*L the unit-mesh circulant stencil.

    Evaluated in extended precision from the circulant eigenvalues
    lambda_k = a_0 + 2 sum_m a_m cos(2 pi k m / Nx) (lambda_0 -> 1 from the
    rank-one term), so the device solve phi = h * khat (*) b is accurate to a
    few ulp independently of the stiffness condition number.
    """
    a = stencil_rationals(degree)
    nx = num_cells
    ld = np.longdouble
    two_pi = ld(8) * np.arctan(ld(1))
    k = np.arange(nx)
    lam = np.full(nx, ld(a[0].numerator) / ld(a[0].denominator), dtype=ld)
    for m in range(1, degree + 1):
        am = ld(a[m].numerator) / ld(a[m].denominator)
        lam += ld(2) * am * np.cos(two_pi * ((k * m) % nx).astype(ld) / ld(nx))
    lam[0] = ld(1)
    inv = ld(1) / lam
    # khat[r] = (1/nx) sum_k cos(2 pi k r / nx) / lambda_k, angle reduced exactly mod nx
    ang = two_pi * (np.outer(k, k) % nx).astype(ld) / ld(nx)
    col = (np.cos(ang) * inv[None, :]).sum(axis=1) / ld(nx)
    return np.asarray(col, dtype=np.float64)


class MeshConstants:
    """Device copies of khat (Nx,) and the stiffness stencil (d+1,)."""

    def __init__(self, num_cells, degree):
        self.num_cells = num_cells
        self.degree = degree
        self.khat = torch.from_numpy(_khat_unit(num_cells, degree)).to("cuda")
        st = [float(c) for c in stencil_rationals(degree)]
        self.stencil = torch.tensor(st, dtype=torch.float64, device="cuda")


_CONST_CACHE = {}


def mesh_constants(num_cells, degree):
    key = (int(num_cells), int(degree), torch.cuda.current_device())
    c = _CONST_CACHE.get(key)
    if c is None:
        c = _CONST_CACHE[key] = MeshConstants(int(num_cells), int(degree))
    return c


def inst_rows_host(lengths, num_cells, charges):
    """(p, 8) float64 host table of per-instance constants (fem.py:54-98)."""
    rows = []
    for length, ch in zip(lengths, charges):
        h = length / num_cells
        qw = ch.charge_weight
        mp = ch.particle_mass
        rows.append([h, 1.0 / h, qw, ch.background * h, -(qw / mp), qw / mp, 0.5 / mp, length])
    return np.asarray(rows, dtype=np.float64).reshape(-1, INST_STRIDE)


_INST_CACHE = {}


def inst_rows(mesh, charge, p):
    """Device per-instance table for one mesh/charge replicated over p columns."""
    key = (mesh, charge, int(p), torch.cuda.current_device())
    t = _INST_CACHE.get(key)
    if t is None:
        host = inst_rows_host([mesh.length] * p, mesh.num_cells, [charge] * p)
        t = _INST_CACHE[key] = torch.from_numpy(host).to("cuda")
    return t


# ---------------------------------------------------------------- workspace

_WS = {}


def workspace(n, p, nx, degree):
    nbytes = int(_lib.query("picrom_fom_workspace_bytes", int(n), int(p), int(nx), int(degree)))
    key = (torch.cuda.current_device(), torch.cuda.current_stream().cuda_stream)
    buf = _WS.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = _WS[key] = torch.zeros(max(nbytes, 1 << 20), dtype=torch.uint8, device="cuda")
    return buf


def new_status():
    return torch.full((2,), -1, dtype=torch.int64, device="cuda")


def decode_status(status, p):
    """None, or (step, row, col) of the first non-finite position."""
    v = int(status[0].item()) & ULL_MAX
    if v == ULL_MAX:
        return None
    step = v >> 40
    lin = v & ((1 << 40) - 1)
    return step, lin // p, lin % p


def raise_if_bad(status, p, ndim):
    bad = decode_status(status, p)
    if bad is None:
        return
    _, row, col = bad
    index = (row,) if ndim == 1 else (row, col)
    raise EvaluationError(f"non-finite particle position at index {index}", index=index)
