"""Memory-safety and race self-checks of the hot kernels.

compute-sanitizer is closed on this GPU pool (runs under it left GPUs needing a
reset), so the protocol checks are our own:
* guard bands: every buffer a kernel writes sits between NaN-filled guard
  regions of the same allocation; after the calls the guards must be intact
  (an out-of-bounds store would overwrite them);
* the cross-CTA ticket protocol of the fused step (last CTA of an instance
  solves it, last instance solve advances the step counter): the tickets are
  left at zero after every step and the counter advances exactly once per step;
* races: repeated runs are bitwise identical (the lane-phase fp64 path by its
  fixed summation order, the fixed-point path because integer sums commute),
  across CUDA-graph replay and plain launches.
"""

import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GUARD = 4096          # doubles of NaN on each side


class Guarded:
    """A device buffer of `count` elements with NaN guard bands (float64) or
    0x7f7f... (int64) on both sides."""

    def __init__(self, count, dtype=torch.float64, fill=0.0):
        self.count = count
        self.buf = torch.empty(count + 2 * GUARD, dtype=dtype, device="cuda")
        if dtype == torch.float64:
            self.buf.fill_(float("nan"))
        else:
            self.buf.fill_(0x7F7F7F7F7F7F7F7F)
        self.t = self.buf[GUARD:GUARD + count]
        self.t.fill_(fill)

    @property
    def ptr(self):
        return self.t.data_ptr()

    def intact(self):
        g = torch.cat([self.buf[:GUARD], self.buf[GUARD + self.count:]])
        if g.dtype == torch.float64:
            return bool(torch.isnan(g).all())
        return bool((g == 0x7F7F7F7F7F7F7F7F).all())


@pytest.fixture(scope="module")
def m(lib_built):
    from paper_2201_05555_b200 import _device as dev
    from paper_2201_05555_b200 import _lib, driver, fem, fullorder, hyper
    return type("M", (), dict(dev=dev, lib=_lib, driver=driver, fem=fem, fo=fullorder, hyper=hyper))


@pytest.mark.parametrize("nx", [64, 128, 512])
def test_pic_step_guards_tickets_counter(m, nx):
    """picrom_pic_step (both deposit paths) writes nothing outside its
    buffers, advances the counter exactly once per step, and leaves its
    tickets re-armed: a second identical sequence on the SAME (not re-zeroed)
    workspace reproduces the first bit for bit."""
    rng = np.random.default_rng(nx)
    n, p, d, L, steps, ring = 20_011, 5, 3, 10 * np.pi, 12, 4
    sysm = m.fo.VlasovSystem(m.fem.build_mesh(L, nx, d), m.fem.ChargeConfig(n, L))
    inst = sysm.inst(p)
    c = sysm.poisson.constants
    x0 = torch.from_numpy(rng.uniform(0, L, p * n)).cuda()
    v0 = torch.from_numpy(rng.standard_normal(p * n)).cuda()
    ws_bytes = int(m.lib.query("picrom_fom_workspace_bytes", n, p, nx, d))
    ws = Guarded((ws_bytes + 7) // 8, fill=0.0)
    s = m.dev.stream_handle()
    outs = []
    for rep in range(2):
        x, v, phi = Guarded(p * n), Guarded(p * n), Guarded(p * nx)
        x.t.copy_(x0)
        v.t.copy_(v0)
        counter = Guarded(2, dtype=torch.int64, fill=0)
        status = Guarded(2, dtype=torch.int64, fill=-1)
        hist = [Guarded(ring * p * nx), Guarded(ring * p * nx), Guarded(ring * p),
                Guarded(ring * p)]
        thist = Guarded(ring, dtype=torch.int64, fill=0)
        for k in range(steps):
            kick, kfull = (0.025, 0.0) if k == 0 else (0.05, 0.025)
            m.lib.call("picrom_pic_step", x.ptr, v.ptr, n, p, n, inst.data_ptr(), nx, d,
                       c.khat.data_ptr(), c.stencil.data_ptr(), phi.ptr, 0.05, kick, kfull, k,
                       counter.ptr, ring, p, hist[0].ptr, hist[1].ptr, hist[2].ptr, hist[3].ptr,
                       thist.ptr, ws.ptr, status.ptr, s)
        torch.cuda.synchronize()
        for b in [x, v, phi, ws, counter, status, thist] + hist:
            assert b.intact()
        assert int(counter.t[0]) == steps and int(counter.t[1]) == 0
        th = thist.t.cpu().numpy()
        assert np.all(th > 0)                 # every ring row stamped by its step's last solve
        assert int(status.t[0]) == -1
        assert bool(torch.isfinite(phi.t).all()) and bool(torch.isfinite(x.t).all())
        outs.append([b.t.cpu().numpy() for b in [x, v, phi] + hist])
    for a_, b_ in zip(*outs):
        np.testing.assert_array_equal(a_, b_)


@pytest.mark.parametrize("nx", [128, 512])
def test_fused_step_bitwise_repeatable(m, nx):
    """Five identical 40-step runs (CUDA-graph replay of two instance groups)
    give bitwise identical state and histories; a plain-launch run (no graph)
    matches them too."""
    rng = np.random.default_rng(1)
    n, p, L = 30_000, 6, 10 * np.pi
    x = rng.uniform(0, L, (n, p))
    v = np.where(rng.uniform(size=(n, p)) < 0.5, -2.5, 2.5) + 0.3 * rng.standard_normal((n, p))
    sysm = m.fo.VlasovSystem(m.fem.build_mesh(L, nx, 3), m.fem.ChargeConfig(n, L))
    outs = []
    for rep in range(5):
        rec = m.fo.run_full_order(sysm, m.fo.ParticleEnsemble(x, v), 0.05, 40 * 0.05,
                                  record=m.fo.RecordOptions(energy_stride=1,
                                                            record_snapshots=False))
        outs.append((rec.final_state.x.copy(), rec.final_state.v.copy(),
                     rec.charge_history.copy(), rec.electric_history.copy()))
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            np.testing.assert_array_equal(a, b)
    xd = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
    vd = torch.from_numpy(np.ascontiguousarray(v.T)).cuda()
    run = m.fo.PicRun(sysm, xd, vd, 0.05, 40)
    run.init_field()
    run.advance(40, use_graph=False)
    run.check()
    np.testing.assert_array_equal(run.x.cpu().numpy().T, outs[0][0])
    np.testing.assert_array_equal(run.rho_hist.cpu().numpy().transpose(0, 2, 1), outs[0][2])


def test_rom_kernels_and_greedy_guards(m):
    """rom_field / rom_gather_uv and the device DEIM greedy write only inside
    their outputs and workspaces, and repeat bit for bit."""
    from paper_2201_05555_b200 import _tall  # noqa: F401
    rng = np.random.default_rng(3)
    N, p, nb, nx = 5003, 7, 6, 32
    lengths = 2 * np.pi / rng.uniform(0.4, 0.6, p)
    gsys = m.driver.ParametricVlasovSystem(lengths, nx, 2, N)
    u = torch.from_numpy(np.linalg.qr(rng.standard_normal((2 * N, nb)))[0]).cuda()
    z = rng.standard_normal((nb, p)) * 3.0
    zd = torch.from_numpy(z).cuda()
    inst = gsys._inst
    c = gsys.poisson.constants
    ws_bytes = int(m.lib.query("picrom_rom_workspace_bytes", N, p, nb, nx))
    res = []
    for rep in range(2):
        ws = Guarded((ws_bytes + 7) // 8)
        phi = Guarded(p * nx)
        st = Guarded(2, dtype=torch.int64, fill=-1)
        e = Guarded(N * p)
        lam = Guarded(N * p)
        proj = [Guarded(nb * p), Guarded(nb * p)]
        s = m.dev.stream_handle()
        m.lib.call("picrom_rom_field", u.data_ptr(), N, nb, zd.data_ptr(), p, p, None,
                   inst.data_ptr(), nx, 2, c.khat.data_ptr(), c.stencil.data_ptr(), phi.ptr, None,
                   None, ws.ptr, st.ptr, None, s)
        m.lib.call("picrom_rom_gather_uv", u.data_ptr(), N, nb, zd.data_ptr(), p, p, None,
                   inst.data_ptr(), nx, 2, phi.ptr, 0, proj[0].ptr, proj[1].ptr, p, lam.ptr, e.ptr,
                   p, ws.ptr, st.ptr, s)
        torch.cuda.synchronize()
        for b in [ws, phi, st, e, lam] + proj:
            assert b.intact()
        assert int(st.t[0]) == -1
        res.append([b.t.cpu().numpy() for b in (phi, e, lam, proj[0], proj[1])])
    for a, b in zip(*res):
        np.testing.assert_array_equal(a, b)
    # device greedy
    n, d = 7001, 12
    psi = torch.from_numpy(np.linalg.qr(rng.standard_normal((n, d)))[0]).cuda()
    need = int(m.lib.query("picrom_deim_workspace_bytes", n, d))
    ws = Guarded((need + 7) // 8)
    idx = Guarded(d, dtype=torch.int64, fill=-5)
    rows = Guarded(d * d)
    keep = np.full(d, -1, dtype=np.int64)
    keep[3] = 11
    m.lib.call("picrom_deim_greedy", psi.data_ptr(), d, n, d, keep.ctypes.data_as(C.c_void_p),
               idx.ptr, rows.ptr, ws.ptr, m.dev.stream_handle())
    torch.cuda.synchronize()
    for b in (ws, idx, rows):
        assert b.intact()
    got = idx.t.cpu().numpy()
    assert got[3] == 11 and len(set(got.tolist())) == d
    from oracle import dmd_deim as odd
    np.testing.assert_array_equal(got, odd.greedy_indices(psi.cpu().numpy(), keep={3: 11}))
    np.testing.assert_array_equal(rows.t.cpu().numpy().reshape(d, d), psi.cpu().numpy()[got])


@pytest.mark.parametrize("ca,k", [(420, 48), (46, 46), (22, 6)])
def test_tall_atb_and_wide_combine_guards(m, ca, k):
    """picrom_tall_atb (both kernel variants) and the 40/48-column wide combine
    write only inside their outputs / workspace, also with a ragged last tile,
    and repeat bit for bit."""
    from paper_2201_05555_b200 import _tall
    rng = np.random.default_rng(ca + k)
    rows = 4099
    a = torch.from_numpy(rng.standard_normal((rows, ca))).cuda()
    b = torch.from_numpy(rng.standard_normal((rows, k))).cuda()
    need = int(m.lib.query("picrom_tall_atb_workspace_bytes", rows, ca, k))
    res = []
    for rep in range(2):
        ws = Guarded((need + 7) // 8)
        out = Guarded(ca * k)
        m.lib.call("picrom_tall_atb", a.data_ptr(), ca, ca, b.data_ptr(), k, k, rows, out.ptr, ws.ptr,
                   m.dev.stream_handle())
        torch.cuda.synchronize()
        assert ws.intact() and out.intact()
        res.append(out.t.cpu().numpy().reshape(ca, k))
    np.testing.assert_array_equal(res[0], res[1])
    ref = a.cpu().numpy().T @ b.cpu().numpy()
    assert np.abs(res[0] - ref).max() <= 1e-12 * np.abs(ref).max()
    # combine into a guarded (rows x k) block with a wider row stride
    mat = rng.standard_normal((ca, k))
    ldo = k + 6
    outc = Guarded(rows * ldo, fill=7.0)
    view = outc.t.view(rows, ldo)[:, :k]
    _tall.combine([(a, mat, False)], out=view)
    torch.cuda.synchronize()
    assert outc.intact()
    full = outc.t.view(rows, ldo).cpu().numpy()
    assert (full[:, k:] == 7.0).all()                      # pad columns untouched
    refc = a.cpu().numpy() @ mat
    assert np.abs(full[:, :k] - refc).max() <= 1e-12 * np.abs(refc).max()
