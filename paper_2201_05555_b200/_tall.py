"""Tall-skinny primitives over device matrices (the two kernels every manifold
operation of the reduced basis is built from).

* ``gram(blocks)``    -> W^T W on the host (numpy), W = column concatenation of
                         tall device blocks, optionally J-applied (picrom_paired_gram)
* ``gram_tasks``      -> only the listed block products of that Gram (picrom_gram_tasks)
* ``combine(terms)``  -> sum_t op_t(B_t) @ M_t on the device (picrom_combine)

Tall blocks are row-major float64 CUDA tensors with a common row count; the
small matrices live on the host and are shipped per call.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _device as dev
from . import _lib
from .errors import ConfigurationError

_WS = {}

# set by parallel.row_sharded(): Gram results are partial sums over this
# rank's rows and are all-reduced before use (None: single process)
reduce_hook = None


def _reduced(out):
    return reduce_hook(out) if reduce_hook is not None else out


def _ws(rows, width):
    need = int(_lib.query("picrom_rom_workspace_bytes", int(rows), 1, 1, 1))
    key = torch.cuda.current_device()
    buf = _WS.get(key)
    if buf is None or buf.numel() < need:
        buf = _WS[key] = torch.empty(max(need, 1 << 20), dtype=torch.uint8, device="cuda")
    return buf


def _arr(ctype, vals):
    return (ctype * len(vals))(*vals)


def gram(blocks):
    """blocks: list of (tensor (M x w_i), jswap) -> numpy (W x W) Gram."""
    if not blocks:
        raise ConfigurationError("gram needs at least one block")
    rows = blocks[0][0].shape[0]
    for t, _ in blocks:
        if t.shape[0] != rows or t.dtype != torch.float64 or not t.is_cuda:
            raise ConfigurationError("gram blocks must be float64 CUDA tensors with equal rows")
    if len(blocks) > 8:
        # split into two Grams is not needed by any caller; keep the limit explicit
        raise ConfigurationError("at most 8 Gram blocks")
    blocks = [(t if t.is_contiguous() else t.contiguous(), j) for t, j in blocks]
    widths = [int(t.shape[1]) for t, _ in blocks]
    W = sum(widths)
    out = torch.empty((W, W), dtype=torch.float64, device="cuda")
    _lib.call("picrom_paired_gram", len(blocks),
              _arr(C.c_void_p, [t.data_ptr() for t, _ in blocks]),
              _arr(C.c_int, [int(t.stride(0)) for t, _ in blocks]),
              _arr(C.c_int, widths), _arr(C.c_int, [int(bool(j)) for _, j in blocks]),
              rows, out.data_ptr(), _ws(rows, W).data_ptr(), dev.stream_handle())
    return _reduced(out).cpu().numpy()


def cross_gram(a_blocks, b_blocks):
    """A^T B (host numpy, wa x wb) for A = column concatenation of a_blocks and
    B of b_blocks (tall device blocks, (tensor, jswap) pairs), picrom_cross_gram."""
    blocks = [(t if t.is_contiguous() else t.contiguous(), j) for t, j in a_blocks + b_blocks]
    rows = blocks[0][0].shape[0]
    widths = [int(t.shape[1]) for t, _ in blocks]
    wa = sum(widths[:len(a_blocks)])
    wb = sum(widths[len(a_blocks):])
    out = torch.empty((wa, wb), dtype=torch.float64, device="cuda")
    _lib.call("picrom_cross_gram", len(blocks), len(a_blocks),
              _arr(C.c_void_p, [t.data_ptr() for t, _ in blocks]),
              _arr(C.c_int, [int(t.stride(0)) for t, _ in blocks]),
              _arr(C.c_int, widths), _arr(C.c_int, [int(bool(j)) for _, j in blocks]),
              rows, out.data_ptr(), _ws(rows, wa + wb).data_ptr(), dev.stream_handle())
    return _reduced(out).cpu().numpy()


_ATB_WS = {}


def atb(a, b, to_host=True):
    """a^T b (host numpy, ca x k; the device tensor with to_host=False) for a
    WIDE tall device block a (N x ca, even ca <= 448: the DEIM sample window)
    and a block b (N x k, even k <= 48), picrom_tall_atb.  a and b may be
    column slices of wider row-major matrices (row strides even, 16-byte
    aligned rows)."""
    rows = a.shape[0]
    ca, k = int(a.shape[1]), int(b.shape[1])
    if a.stride(1) != 1:
        a = a.contiguous()
    if b.stride(1) != 1:
        b = b.contiguous()
    need = int(_lib.query("picrom_tall_atb_workspace_bytes", int(rows), ca, k))
    key = torch.cuda.current_device()
    ws = _ATB_WS.get(key)
    if ws is None or ws.numel() < need:
        ws = _ATB_WS[key] = torch.empty(need, dtype=torch.uint8, device="cuda")
    out = torch.empty((ca, k), dtype=torch.float64, device="cuda")
    _lib.call("picrom_tall_atb", a.data_ptr(), int(a.stride(0)), ca, b.data_ptr(), int(b.stride(0)), k,
              int(rows), out.data_ptr(), ws.data_ptr(), dev.stream_handle())
    out = _reduced(out)
    return out.cpu().numpy() if to_host else out


def combine_dev(block, mat_dev, out=None):
    """block (N x a, device) @ mat_dev (a x c, DEVICE, contiguous) -> (N x c):
    picrom_combine with the small matrix already on the device (no upload, no
    host round trip in a chain of tall products)."""
    rows, a = block.shape
    c = int(mat_dev.shape[1])
    if tuple(mat_dev.shape) != (a, c) or not mat_dev.is_contiguous():
        raise ConfigurationError("combine_dev: matrix must be a contiguous (width x c) device tensor")
    if out is None:
        out = torch.empty((rows, c), dtype=torch.float64, device="cuda")
    t = block if block.stride(1) == 1 else block.contiguous()
    _lib.call("picrom_combine", 1, _arr(C.c_void_p, [t.data_ptr()]), _arr(C.c_int, [int(t.stride(0))]),
              _arr(C.c_int, [int(a)]), _arr(C.c_int, [0]), _arr(C.c_int, [0]), mat_dev.data_ptr(),
              int(a * c), rows, out.data_ptr(), int(out.stride(0)), c, 0, dev.stream_handle())
    return out


def cholinv_dev(g_dev):
    """(R^-1, info) on the device for g = R^T R (k x k SPD device tensor, k <= 48);
    info = [min diag R, max diag R] (picrom_small_cholinv)."""
    k = int(g_dev.shape[0])
    rinv = torch.empty((k, k), dtype=torch.float64, device="cuda")
    info = torch.empty(2, dtype=torch.float64, device="cuda")
    _lib.call("picrom_small_cholinv", g_dev.data_ptr(), k, rinv.data_ptr(), info.data_ptr(),
              dev.stream_handle())
    return rinv, info


def rmul_dev(a_dev, b_dev, colscale=None):
    """a (r x k) @ b (k x k), column j scaled by colscale[j], all on the device
    (picrom_small_rmul)."""
    r, k = int(a_dev.shape[0]), int(a_dev.shape[1])
    out = torch.empty((r, k), dtype=torch.float64, device="cuda")
    _lib.call("picrom_small_rmul", a_dev.data_ptr(), r, k, b_dev.data_ptr(),
              None if colscale is None else colscale.data_ptr(), out.data_ptr(), dev.stream_handle())
    return out


def gram_tasks(blocks, tasks):
    """Selected block products of gram(blocks): tasks = [(i, j), ...] -> numpy (W x W)
    with block (i, j) = B_i^T B_j for each task (other entries unspecified)."""
    rows = blocks[0][0].shape[0]
    blocks = [(t if t.is_contiguous() else t.contiguous(), j) for t, j in blocks]
    widths = [int(t.shape[1]) for t, _ in blocks]
    W = sum(widths)
    out = torch.empty((W, W), dtype=torch.float64, device="cuda")
    _lib.call("picrom_gram_tasks", len(blocks),
              _arr(C.c_void_p, [t.data_ptr() for t, _ in blocks]),
              _arr(C.c_int, [int(t.stride(0)) for t, _ in blocks]),
              _arr(C.c_int, widths), _arr(C.c_int, [int(bool(j)) for _, j in blocks]),
              len(tasks), _arr(C.c_int, [int(i) for i, _ in tasks]),
              _arr(C.c_int, [int(j) for _, j in tasks]),
              rows, out.data_ptr(), _ws(rows, W).data_ptr(), dev.stream_handle())
    return _reduced(out).cpu().numpy()


def combine(terms, out=None, accumulate=False):
    """terms: list of (tensor (M x a_t), M_t numpy (a_t x c), jswap) -> tensor (M x c)."""
    rows = terms[0][0].shape[0]
    c = terms[0][1].shape[1]
    mats, offs = [], []
    off = 0
    for t, m, _ in terms:
        m = np.ascontiguousarray(m, dtype=np.float64)
        if m.shape != (t.shape[1], c):
            raise ConfigurationError(f"combine: matrix {m.shape} does not match block {tuple(t.shape)}")
        mats.append(m.ravel())
        offs.append(off)
        off += m.size
    buf = torch.from_numpy(np.concatenate(mats)).to("cuda")
    if out is None:
        out = torch.empty((rows, c), dtype=torch.float64, device="cuda")
        accumulate = False
    ts = [(t if t.is_contiguous() else t.contiguous()) for t, _, _ in terms]
    _lib.call("picrom_combine", len(terms), _arr(C.c_void_p, [t.data_ptr() for t in ts]),
              _arr(C.c_int, [int(t.stride(0)) for t in ts]), _arr(C.c_int, [int(t.shape[1]) for t in ts]),
              _arr(C.c_int, [int(bool(j)) for _, _, j in terms]), _arr(C.c_int, offs),
              buf.data_ptr(), int(off), rows, out.data_ptr(), int(out.stride(0)), int(c),
              int(bool(accumulate)), dev.stream_handle())
    return out


def split(G, widths):
    """Blocks of a Gram: split(G, [a, b])[i][j] is block_i^T block_j."""
    edges = np.concatenate([[0], np.cumsum(widths)])
    return [[G[edges[i]:edges[i + 1], edges[j]:edges[j + 1]] for j in range(len(widths))]
            for i in range(len(widths))]
