"""Tall-skinny Gram / combine kernels (the manifold building blocks of
reduction.py:143-182) against numpy on the same inputs: the DMMA and TMA fast
paths (equal block widths <= 32, >= 1024 rows) and the generic fallback."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _j(b):
    """J applied to a (2h x w) block: [X; V] -> [V; -X] (reduction.py:44-47)."""
    h = b.shape[0] // 2
    return np.concatenate([b[h:], -b[:h]])


def _cross(lib_built, blocks, na, rows):
    import torch
    from paper_2201_05555_b200 import _lib, _tall
    from paper_2201_05555_b200 import _device as dev
    widths = [int(t.shape[1]) for t, _ in blocks]
    wa, wb = sum(widths[:na]), sum(widths[na:])
    out = torch.empty((wa, wb), dtype=torch.float64, device="cuda")
    arr = _tall._arr
    _lib.call("picrom_cross_gram", len(blocks), na, arr(C.c_void_p, [t.data_ptr() for t, _ in blocks]),
              arr(C.c_int, [int(t.stride(0)) for t, _ in blocks]), arr(C.c_int, widths),
              arr(C.c_int, [int(j) for _, j in blocks]), rows, out.data_ptr(),
              _tall._ws(rows, wa + wb).data_ptr(), dev.stream_handle())
    return out.cpu().numpy()


@pytest.mark.parametrize("w", [8, 16, 20, 32])
@pytest.mark.parametrize("rows", [1024, 2 * 25013])
def test_gram_equal_widths(lib_built, w, rows):
    import torch
    from paper_2201_05555_b200 import _tall
    rng = np.random.default_rng(w * 7 + rows)
    hs = [rng.standard_normal((rows, w)) for _ in range(3)]
    blocks = [(torch.from_numpy(hs[0]).cuda(), False), (torch.from_numpy(hs[1]).cuda(), False),
              (torch.from_numpy(hs[1]).cuda(), True), (torch.from_numpy(hs[2]).cuda(), False)]
    W = np.concatenate([hs[0], hs[1], _j(hs[1]), hs[2]], axis=1)
    ref = W.T @ W
    got = _tall.gram(blocks)
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
    assert np.array_equal(got, got.T)
    assert np.array_equal(got, _tall.gram(blocks))       # deterministic


def test_gram_eight_blocks_and_cross(lib_built):
    import torch
    from paper_2201_05555_b200 import _tall
    rng = np.random.default_rng(5)
    rows = 2 * 40001
    hs = [rng.standard_normal((rows, 20)) for _ in range(8)]
    js = [False, True, False, False, True, False, False, True]
    blocks = [(torch.from_numpy(h).cuda(), j) for h, j in zip(hs, js)]
    W = np.concatenate([_j(h) if j else h for h, j in zip(hs, js)], axis=1)
    ref = W.T @ W
    got = _tall.gram(blocks)
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
    for na in (1, 3):
        cg = _cross(lib_built, blocks, na, rows)
        cref = W[:, :20 * na].T @ W[:, 20 * na:]
        assert np.abs(cg - cref).max() <= 1e-12 * np.abs(ref).max()


def test_gram_fallback_paths(lib_built):
    """Unequal widths / strided blocks take the generic kernels; same answers."""
    import torch
    from paper_2201_05555_b200 import _tall
    rng = np.random.default_rng(9)
    rows = 4096
    a = rng.standard_normal((rows, 20))
    b = rng.standard_normal((rows, 12))
    big = torch.from_numpy(rng.standard_normal((rows, 40))).cuda()
    blocks = [(torch.from_numpy(a).cuda(), False), (torch.from_numpy(b).cuda(), True), (big[:, :20], False)]
    W = np.concatenate([a, _j(b), big[:, :20].cpu().numpy()], axis=1)
    ref = W.T @ W
    got = _tall.gram(blocks)
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("rows", [1024, 2 * 25013])
def test_combine_terms(lib_built, rows):
    import torch
    from paper_2201_05555_b200 import _tall
    rng = np.random.default_rng(rows)
    x = rng.standard_normal((rows, 20))
    y = rng.standard_normal((rows, 20))
    e = rng.standard_normal((rows, 128))
    m1, m2, m3 = (rng.standard_normal((20, 20)), rng.standard_normal((20, 20)),
                  rng.standard_normal((128, 20)))
    got = _tall.combine([(torch.from_numpy(x).cuda(), m1, False),
                         (torch.from_numpy(y).cuda(), m2, True)]).cpu().numpy()
    ref = x @ m1 + _j(y) @ m2
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
    got = _tall.combine([(torch.from_numpy(e).cuda(), m3, False)]).cpu().numpy()
    ref = e @ m3
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
    out = torch.from_numpy(ref.copy()).cuda()
    _tall.combine([(torch.from_numpy(x).cuda(), m1, False)], out=out, accumulate=True)
    ref2 = ref + x @ m1
    assert np.abs(out.cpu().numpy() - ref2).max() <= 1e-12 * np.abs(ref2).max()


@pytest.mark.parametrize("rows", [1030, 2 * 25013])
@pytest.mark.parametrize("c", [7, 20, 32])
def test_combine_wide_term(lib_built, rows, c):
    """The wide-term combine (a 128- or 130-wide block, as E (N x p') in the basis
    velocity) with narrow and J-applied terms, into a strided output half."""
    import torch
    from paper_2201_05555_b200 import _tall
    rng = np.random.default_rng(rows + c)
    e = rng.standard_normal((rows, 130))
    x = rng.standard_normal((rows, 20))
    y = rng.standard_normal((rows, 20))
    me, mx, my = (rng.standard_normal((130, c)), rng.standard_normal((20, c)),
                  rng.standard_normal((20, c)))
    out = torch.zeros((2 * rows, c), dtype=torch.float64, device="cuda")
    _tall.combine([(torch.from_numpy(e).cuda(), me, False), (torch.from_numpy(x).cuda(), mx, False),
                   (torch.from_numpy(y).cuda(), my, True)], out=out[rows:])
    ref = e @ me + x @ mx + _j(y) @ my
    got = out.cpu().numpy()
    assert np.abs(got[rows:] - ref).max() <= 1e-12 * np.abs(ref).max()
    assert not got[:rows].any()


@pytest.mark.parametrize("ca,k,rows", [(420, 48, 30011), (420, 20, 4099), (48, 48, 2 * 25013),
                                       (140, 24, 1500), (6, 2, 333), (448, 48, 1024)])
def test_tall_atb_wide_left_operand(lib_built, ca, k, rows):
    """picrom_tall_atb (the DEIM window's W^T Q, Q^T W and sliding Gram update,
    hyper.py:262) against numpy, incl. column slices of a wider row-major
    matrix (row stride > width), ragged last tiles and few-row inputs."""
    import torch
    from paper_2201_05555_b200 import _tall
    rng = np.random.default_rng(ca * 3 + k + rows)
    big = rng.standard_normal((rows, ca + 12)) * np.logspace(0, -6, ca + 12)
    b = rng.standard_normal((rows, k))
    bd = torch.from_numpy(big).cuda()
    a_view = bd[:, 4:4 + ca]                  # stride ca + 12, offset 32 bytes
    got = _tall.atb(a_view, torch.from_numpy(b).cuda())
    ref = big[:, 4:4 + ca].T @ b
    scale = np.linalg.norm(big[:, 4:4 + ca], axis=0)[:, None] * np.linalg.norm(b, axis=0)[None, :]
    assert np.abs(got - ref).max() <= 1e-13 * scale.max()
    assert (np.abs(got - ref) <= 1e-12 * scale + 1e-300).all()
    assert np.array_equal(got, _tall.atb(a_view, torch.from_numpy(b).cuda()))     # deterministic


def test_tall_atb_rejects_unaligned(lib_built):
    import torch
    from paper_2201_05555_b200 import _tall
    from paper_2201_05555_b200.errors import ConfigurationError
    a = torch.zeros((64, 21), dtype=torch.float64, device="cuda")
    b = torch.zeros((64, 4), dtype=torch.float64, device="cuda")
    with pytest.raises((ConfigurationError, RuntimeError, ValueError)):
        _tall.atb(a, b)


@pytest.mark.parametrize("c", [40, 48])
def test_combine_up_to_48_columns(lib_built, c):
    """W (N x 420) @ M (420 x c): the subspace-iteration products of the window
    SVD through the wide-term DMMA combine."""
    import torch
    from paper_2201_05555_b200 import _tall
    rng = np.random.default_rng(c)
    rows = 20011
    w = rng.standard_normal((rows, 420))
    m = rng.standard_normal((420, c))
    got = _tall.combine([(torch.from_numpy(w).cuda(), m, False)]).cpu().numpy()
    ref = w @ m
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


def test_window_svd_tall_products_helpers(lib_built):
    """hyper._tsq / hyper._mul: odd widths, > 48 columns and > 448 columns are
    chunked or padded onto the library kernels."""
    import torch
    from paper_2201_05555_b200 import hyper
    rng = np.random.default_rng(3)
    rows = 5003
    a = rng.standard_normal((rows, 451))
    b = rng.standard_normal((rows, 51))
    ad, bd = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    ref = a.T @ b
    assert np.abs(hyper._tsq(ad, bd) - ref).max() <= 1e-12 * np.abs(ref).max()
    assert np.abs(hyper._tsq(bd, ad) - ref.T).max() <= 1e-12 * np.abs(ref).max()
    m = rng.standard_normal((451, 51))
    got = hyper._mul(ad, m).cpu().numpy()
    assert np.abs(got - a @ m).max() <= 1e-12 * np.abs(a @ m).max()


@pytest.mark.parametrize("k", [2, 20, 48])
def test_small_cholinv_and_rmul(lib_built, k):
    """picrom_small_cholinv / picrom_small_rmul (the device Cholesky-QR chain of
    the window SVD) against numpy."""
    import torch
    from paper_2201_05555_b200 import _tall
    rng = np.random.default_rng(k)
    y = rng.standard_normal((500, k)) * np.logspace(0, -1, k)
    g = y.T @ y
    rinv, info = _tall.cholinv_dev(torch.from_numpy(g).cuda())
    r = np.linalg.cholesky(g).T
    got = rinv.cpu().numpy()
    assert np.abs(got - np.linalg.inv(r)).max() <= 1e-12 * np.abs(np.linalg.inv(r)).max()
    q = y @ got
    assert np.abs(q.T @ q - np.eye(k)).max() <= 1e-12
    d = np.abs(np.diag(r))
    np.testing.assert_allclose(info.cpu().numpy(), [d.min(), d.max()], rtol=1e-13)
    a = rng.standard_normal((421, k))
    scale = rng.uniform(0.5, 2.0, k)
    out = _tall.rmul_dev(torch.from_numpy(a).cuda(), rinv, torch.from_numpy(scale).cuda()).cpu().numpy()
    ref = (a @ got) * scale
    assert np.abs(out - ref).max() <= 1e-13 * np.abs(ref).max()
    # not positive definite -> info[0] == 0
    bad = g.copy()
    bad[0, 0] = -1.0
    _, info2 = _tall.cholinv_dev(torch.from_numpy(bad).cuda())
    assert float(info2[0]) == 0.0


def test_window_svd_device_chain_matches_host_chain(lib_built, monkeypatch):
    """The device-resident Cholesky-QR chain of hyper._window_svd spans the same
    basis as the host chain (same algorithm, small algebra in LAPACK)."""
    import torch
    from paper_2201_05555_b200 import hyper
    rng = np.random.default_rng(9)
    rows, cols, dim = 5003, 80, 16
    left = np.linalg.qr(rng.standard_normal((rows, cols)))[0]
    right = np.linalg.qr(rng.standard_normal((cols, cols)))[0]
    samples = torch.from_numpy((left * np.logspace(0, -7, cols)) @ right.T).cuda()
    win = hyper.DeimWindow(1)
    win.append(samples)
    used = []
    real = hyper._refine_on_device
    monkeypatch.setattr(hyper, "_refine_on_device", lambda *a, **k: used.append(1) or real(*a, **k))
    psi_dev, d1 = hyper._window_svd(win, dim)
    assert used, "the device chain did not run"
    monkeypatch.setattr(hyper, "_refine_on_device", lambda *a, **k: None)
    psi_host, d2 = hyper._window_svd(win, dim)
    assert d1 == d2 == dim
    a, b = psi_dev.cpu().numpy(), psi_host.cpu().numpy()
    assert np.abs(a.T @ a - np.eye(dim)).max() <= 1e-12
    s = np.linalg.svd(a.T @ b, compute_uv=False)
    assert s.min() > 1 - 1e-13
    assert np.abs(np.abs(np.diag(a.T @ b)) - 1.0).max() <= 1e-9     # same vectors up to sign
