"""Reduced-order main loop on the GPU -- drop-in for picrom.driver's hot path.

Mirrors /root/reference/pkg/src/picrom/driver.py:63-274: ``exact_gradients``,
``make_full_stage`` and ``run_reduced`` (Algorithm 2).  The particle-count-
dependent work runs in the sm_100a library:

* the field half of F(U z) -- reconstruct X_r = U_X z in registers, deposit,
  one circulant solve per column (picrom_rom_field);
* the gather half -- reconstruct again, gather the field, project
  U_X^T E (picrom_rom_gather), harvesting the DEIM samples Lambda phi in the
  same pass;
* the basis update -- tall-skinny Grams and combines (reduction.py).

``ParametricVlasovSystem`` carries one mesh per parameter column (BASELINE C3/C4
draw a wavenumber per instance); with a single length it is the reference's
VlasovSystem.  Report assembly (run_full/rom/compare, rate fits) stays out of
scope.
"""

from __future__ import annotations

import ctypes as C
from collections import deque
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as dev
from . import _lib, _tall
from . import hyper as hyp
from .errors import ConfigurationError, DivergenceError, EvaluationError, StepFailureError
from .fem import ChargeConfig, PoissonOperator, build_mesh
from .fullorder import VlasovSystem
from .reduction import (
    complex_svd_basis,
    orthosymplectic_residuals,
    prk2_step,
    select_parameter_subset,
)

__all__ = ["ParametricVlasovSystem", "DeviceGradient", "exact_gradients", "make_full_stage",
           "run_reduced", "RomRecord"]


class ParametricVlasovSystem:
    """One periodic mesh per parameter column: lengths L_j, shared Nx, degree, N.

    ``mesh``/``charge``/``poisson`` refer to column 0 (what single-mesh code
    reads); per-column constants live in the device instance table."""

    def __init__(self, lengths, num_cells, degree, num_particles, charge=-1.0, mass=1.0,
                 background=1.0):
        self.lengths = np.asarray(lengths, dtype=float).reshape(-1)
        self.num_cells, self.degree = int(num_cells), int(degree)
        self.meshes = [build_mesh(L, num_cells, degree) for L in self.lengths]
        self.charges = [ChargeConfig(int(num_particles), float(L), charge, mass, background)
                        for L in self.lengths]
        self.mesh, self.charge = self.meshes[0], self.charges[0]
        self.poisson = PoissonOperator(self.mesh)
        self._inst = torch.from_numpy(
            dev.inst_rows_host(self.lengths, self.num_cells, self.charges)).to("cuda")

    def inst_table(self, p):
        return self._inst

    def column_charge(self, j):
        return self.charges[j]


def _inst_table(system, p):
    if isinstance(system, ParametricVlasovSystem):
        return system._inst
    return dev.inst_rows(system.mesh, system.charge, p)


def _column_charge(system, j):
    if isinstance(system, ParametricVlasovSystem):
        return system.charges[j]
    return system.charge


_WS = {}


def _rom_ws(N, p, n, nx):
    need = int(_lib.query("picrom_rom_workspace_bytes", int(N), int(p), int(n), int(nx)))
    key = torch.cuda.current_device()
    buf = _WS.get(key)
    if buf is None or buf.numel() < need:
        buf = _WS[key] = torch.empty(max(need, 1 << 20), dtype=torch.uint8, device="cuda")
    return buf


class _Cols:
    """Device int32 column->instance map (None = identity)."""

    def __init__(self, cols, p_total):
        self.host = None if cols is None else np.asarray(cols, dtype=np.int32)
        self.dev = (None if cols is None
                    else torch.from_numpy(self.host.copy()).to("cuda"))

    @property
    def ptr(self):
        return None if self.dev is None else self.dev.data_ptr()


def _partial_inst(inst):
    """Instance table of a row shard: the background bg*h is added by the
    background owner only (rho partials of all ranks sum to rho)."""
    from . import parallel
    sh = parallel.active()
    if sh is None or sh.background_owner():
        return inst
    loc = inst.clone()
    loc.view(-1, dev.INST_STRIDE)[:, 3] = 0.0           # I_BGH
    return loc


def _field_device(system, ud, z, cols, want_energy=False, status=None):
    """phi (p', nx) [, energy (p')] of X_r = U_X z on the device.  Row-sharded
    (parallel.row_sharded): the local charge partial is all-reduced before the
    replicated Poisson solve."""
    from . import parallel
    N2, n = ud.shape
    N = N2 // 2
    p = z.shape[1]
    mesh = system.mesh
    nx, d = mesh.num_cells, mesh.degree
    c = system.poisson.constants
    zd = torch.from_numpy(np.ascontiguousarray(z, dtype=np.float64)).to("cuda")
    inst = _inst_table(system, p if cols.dev is None else int(cols.host.max()) + 1)
    phi = torch.empty((p, nx), dtype=torch.float64, device="cuda")
    energy = torch.empty(p, dtype=torch.float64, device="cuda") if want_energy else None
    st = status if status is not None else dev.new_status()
    s = dev.stream_handle()
    sh = parallel.active()
    if sh is None or sh.world == 1:
        _lib.call("picrom_rom_field", ud.data_ptr(), N, n, zd.data_ptr(), p, p, cols.ptr,
                  inst.data_ptr(), nx, d, c.khat.data_ptr(), c.stencil.data_ptr(), phi.data_ptr(),
                  None, dev.ptr(energy), _rom_ws(N, p, n, nx).data_ptr(), st.data_ptr(), None, s)
        return zd, inst, phi, energy, st
    rho = torch.empty((p, nx), dtype=torch.float64, device="cuda")
    _lib.call("picrom_rom_field", ud.data_ptr(), N, n, zd.data_ptr(), p, p, cols.ptr,
              _partial_inst(inst).data_ptr(), nx, d, c.khat.data_ptr(), c.stencil.data_ptr(), None,
              rho.data_ptr(), None, _rom_ws(N, p, n, nx).data_ptr(), st.data_ptr(), None, s)
    parallel.allreduce_sum(rho)
    col_inst = inst if cols.dev is None else inst[torch.from_numpy(cols.host.astype(np.int64)).cuda()]
    _lib.call("picrom_poisson", rho.data_ptr(), p, nx, d, col_inst.data_ptr(), c.khat.data_ptr(),
              c.stencil.data_ptr(), phi.data_ptr(), dev.ptr(energy), s)
    return zd, inst, phi, energy, st


def _raise_eval(st, p):
    bad = dev.decode_status(st, p)
    if bad is not None:
        _, row, col = bad
        raise EvaluationError(f"non-finite particle position at index {(row, col)}",
                              index=(row, col))


class DeviceGradient:
    """F(U z) = [coef d/dx(phi.Lambda)(U_X z); U_V z] (2N x p') kept implicit:
    E (N x p') on the device plus (U, z).  ``times_matrix(M)`` = G @ M as two
    combines; ``dense()`` materialises G (API / tests)."""

    def __init__(self, u, z, e, ux_e=None, uv_e=None):
        self.u, self.z, self.e = u, np.asarray(z, dtype=float), e
        # U_X^T E and U_V^T E (n x p') from the same gather pass (host arrays)
        self.ux_e, self.uv_e = ux_e, uv_e

    @property
    def shape(self):
        return (self.u.shape[0], self.z.shape[1])

    def times_matrix(self, m):
        m = np.asarray(m, dtype=float)
        N = self.u.shape[0] // 2
        out = torch.empty((2 * N, m.shape[1]), dtype=torch.float64, device="cuda")
        _tall.combine([(self.e, m, False)], out=out[:N])
        _tall.combine([(self.u[N:], self.z @ m, False)], out=out[N:])
        return out

    def __matmul__(self, m):
        return self.times_matrix(m)

    def dense(self):
        N = self.u.shape[0] // 2
        out = torch.empty((2 * N, self.z.shape[1]), dtype=torch.float64, device="cuda")
        out[:N].copy_(self.e)
        for j in range(0, self.z.shape[1], 32):              # U_V z, 32 columns per combine
            _tall.combine([(self.u[N:], self.z[:, j:j + 32], False)], out=out[N:, j:j + 32])
        return out


def exact_gradients_device(system, ud, z, cols=None, harvest=True):
    """(DeviceGradient, phi (p', nx) device, lam (N x p') device|None) -- driver.py:63-76."""
    N2, n = ud.shape
    N = N2 // 2
    p = z.shape[1]
    colmap = cols if isinstance(cols, _Cols) else _Cols(cols, p)
    zd, inst, phi, _, st = _field_device(system, ud, z, colmap)
    e = torch.empty((N, p), dtype=torch.float64, device="cuda")
    lam = torch.empty((N, p), dtype=torch.float64, device="cuda") if harvest else None
    proj = torch.empty((2, n, p), dtype=torch.float64, device="cuda")
    mesh = system.mesh
    _lib.call("picrom_rom_gather_uv", ud.data_ptr(), N, n, zd.data_ptr(), p, p, colmap.ptr,
              inst.data_ptr(), mesh.num_cells, mesh.degree, phi.data_ptr(), 0,
              proj[0].data_ptr(), proj[1].data_ptr(), p, dev.ptr(lam), e.data_ptr(), p,
              _rom_ws(N, p, n, mesh.num_cells).data_ptr(), st.data_ptr(), dev.stream_handle())
    _raise_eval(st, p)
    from . import parallel
    ph = parallel.allreduce_sum(proj).cpu().numpy()      # U^T E partials (sharded runs)
    return DeviceGradient(ud, z, e, ph[0], ph[1]), phi, lam


def exact_gradients(system, u, z):
    """Full-state gradients at the reconstructed columns U z (driver.py:63-76):
    (g (2N, p'), phi (Nx, p'), lam (N, p')) as arrays of the input's kind."""
    was_np = not isinstance(u, torch.Tensor)
    ud = (torch.from_numpy(np.ascontiguousarray(u, dtype=np.float64)).to("cuda") if was_np
          else u.to(device="cuda", dtype=torch.float64).contiguous())
    z = z.cpu().numpy() if isinstance(z, torch.Tensor) else np.asarray(z, dtype=float)
    g, phi, lam = exact_gradients_device(system, ud, z)
    gd = g.dense()
    phi_t = phi.t().contiguous()
    if was_np:
        return gd.cpu().numpy(), phi_t.cpu().numpy(), lam.cpu().numpy()
    return gd, phi_t, lam


def make_full_stage(system):
    """Warm-up coefficient gradient U_mid^T F(U_mid z) on all columns (driver.py:79-89):
    g(z) = U_X^T E(U_X z) + (U_V^T U_V) z, E by the fused rom_field/rom_gather
    passes, the Gram once per stage."""

    from . import parallel
    from .reduction import DeviceFixedPoint
    hint = [None]                    # the previous step's fixed-point iteration count

    def factory(u_mid):
        N = u_mid.shape[0] // 2
        n = u_mid.shape[1]
        uvtuv = _tall.gram([(u_mid[N:], False)])
        mesh = system.mesh
        nx, d = mesh.num_cells, mesh.degree
        c = system.poisson.constants
        bufs = {}

        def ensure(p):
            if bufs.get("p") != p:
                bufs.update(p=p, zd=torch.empty((n, p), dtype=torch.float64, device="cuda"),
                            phi=torch.empty((p, nx), dtype=torch.float64, device="cuda"),
                            gout=torch.empty((n, p), dtype=torch.float64, device="cuda"),
                            st=dev.new_status(),
                            z_h=torch.empty((n, p), dtype=torch.float64, pin_memory=True),
                            out_h=torch.empty((n * p + 2,), dtype=torch.float64, pin_memory=True),
                            inst=_inst_table(system, p),
                            ws=_rom_ws(N, p, n, nx))

        def g(z):
            # the host fixed-point loop calls this ~9 times per step: buffers
            # are reused and the result and the status word come back in one sync
            z = np.ascontiguousarray(z, dtype=np.float64)
            p = z.shape[1]
            ensure(p)
            zd, phi, gout, st = bufs["zd"], bufs["phi"], bufs["gout"], bufs["st"]
            bufs["z_h"].numpy()[...] = z
            zd.copy_(bufs["z_h"], non_blocking=True)
            st.fill_(-1)
            sh = dev.stream_handle()
            if parallel.active() is None or parallel.active().world == 1:
                _lib.call("picrom_rom_field", u_mid.data_ptr(), N, n, zd.data_ptr(), p, p, None,
                          bufs["inst"].data_ptr(), nx, d, c.khat.data_ptr(),
                          c.stencil.data_ptr(), phi.data_ptr(), None, None,
                          bufs["ws"].data_ptr(), st.data_ptr(), None, sh)
            else:
                phi.copy_(_field_device(system, u_mid, z, _Cols(None, p), status=st)[2])
            _lib.call("picrom_rom_gather", u_mid.data_ptr(), N, n, zd.data_ptr(), p, p, None,
                      bufs["inst"].data_ptr(), nx, d, phi.data_ptr(), 0, gout.data_ptr(), p,
                      None, None, 0, bufs["ws"].data_ptr(), st.data_ptr(), None, sh)
            parallel.allreduce_sum(gout)                  # U_X^T E partials (sharded runs)
            out_h = bufs["out_h"]
            out_h[:n * p].copy_(gout.reshape(-1), non_blocking=True)
            out_h[n * p:].copy_(st.view(torch.float64), non_blocking=True)
            torch.cuda.current_stream().synchronize()
            stat = out_h[n * p:].view(torch.int64)
            if int(stat[0]) != -1:
                _raise_eval(stat, p)
            return out_h[:n * p].numpy().reshape(n, p).copy() + uvtuv @ z

        def launch_d(zeval, gout, skip, st):
            """D(zeval) = U_X^T E(U_X zeval) into gout: rom_field + rom_gather,
            both skipped once the device fixed point has converged."""
            p = zeval.shape[1]
            ensure(p)
            sh = dev.stream_handle()
            _lib.call("picrom_rom_field", u_mid.data_ptr(), N, n, zeval.data_ptr(), p, p, None,
                      bufs["inst"].data_ptr(), nx, d, c.khat.data_ptr(), c.stencil.data_ptr(),
                      bufs["phi"].data_ptr(), None, None, bufs["ws"].data_ptr(), st.data_ptr(),
                      skip.data_ptr(), sh)
            _lib.call("picrom_rom_gather", u_mid.data_ptr(), N, n, zeval.data_ptr(), p, p, None,
                      bufs["inst"].data_ptr(), nx, d, bufs["phi"].data_ptr(), 0, gout.data_ptr(),
                      p, None, None, 0, bufs["ws"].data_ptr(), st.data_ptr(), skip.data_ptr(), sh)

        if parallel.active() is None or parallel.active().world == 1:
            g.device_fixed_point = DeviceFixedPoint(n, launch_d, uvtuv, hint)
        return g

    return factory


@dataclass
class RomRecord:
    """Time series and reduced snapshots of a reduced run (driver.py:92-114):
    every field of the reference record, plus the DEIM indices of each hyper
    step and per-step wall seconds."""

    times: np.ndarray
    energy_times: np.ndarray
    electric_energy: np.ndarray       # (T_e, p), from reconstructed states
    hamiltonian: np.ndarray
    snapshot_times: np.ndarray
    bases: list                       # [(U, Z)] at snapshot times (U on the device)
    ortho_residuals: np.ndarray       # per step, after the step
    sympl_residuals: np.ndarray
    fp_iterations: np.ndarray
    dmd_ranks: np.ndarray
    s_conds: np.ndarray
    decomp_times: np.ndarray
    dh_total: np.ndarray
    dh_coeff: np.ndarray
    dh_coeff_dd: np.ndarray
    timers: object
    dmd_imag_defect: float
    hyper_engaged: bool
    notes: dict = field(default_factory=dict)
    deim_indices: list = field(default_factory=list)
    step_seconds: np.ndarray = None


def _diag_energies(system, ud, z):
    """Electric + kinetic energy of the reconstructed state (driver.py:160-170):
    kinetic 0.5 z_j^T (U_V^T U_V) z_j needs no reconstruction."""
    p = z.shape[1]
    N = ud.shape[0] // 2
    _, _, _, ee, st = _field_device(system, ud, z, _Cols(None, p), want_energy=True)
    _raise_eval(st, p)
    gv = _tall.gram([(ud[N:], False)])
    kin = 0.5 * np.einsum("ij,ij->j", z, gv @ z)
    return ee.cpu().numpy(), kin


def run_reduced(system, params, x0, v0, *, basis_dim, subsample, window, deim_dim, deim_period,
                deim_update, dt, t_final, svd_tol_dmd=1e-5, fp_tol=1e-9, fp_max_iter=100,
                hyper_reduction=True, printed_subset_variant=False, printed_deim_ranking=False,
                energy_stride=10, snapshot_stride=None, decomp_stride=50, record_snapshots=True,
                timers=None, u0=None, z0=None, sharding=None, init="host"):
    """Reduced-order run over all parameter columns (driver.py:117-274).

    U lives on the device for the whole run; Z and every small matrix on the
    host.  ``u0``/``z0`` may supply the initial basis (otherwise the complex
    SVD of the snapshots, as in the reference).  The host BLAS is capped at 4
    threads for the run: the n x n / window-size algebra gains nothing from
    more, and idle OpenBLAS threads spinning on 16 cores slowed every host
    step (profiles/r01b: the 420 x 420 DEIM eigh 48 -> 8 ms, argmax round
    trips 3x).

    ``init``: "host" (default) computes the initial basis by the reference's
    LAPACK complex SVD (bit-identical U, Z); "device" by
    reduction.complex_svd_basis_device (Hermitian Gram on the GPU: the same
    basis up to a phase per singular vector, ~100x faster at C3).

    ``sharding`` (parallel.RowSharding, under torchrun): this rank advances
    the particle rows [lo, hi) of U (u0 may be the global basis or the local
    rows); every N-row product is all-reduced, Z and the records are
    replicated, the snapshot bases hold the local rows.  No hyper-reduction
    in the sharded mode (the DEIM window and greedy are not sharded)."""
    from threadpoolctl import threadpool_limits

    from . import parallel
    if sharding is not None:
        if hyper_reduction:
            raise ConfigurationError("row-sharded reduced runs support hyper_reduction=False only")
        if u0 is None:
            u0, z0 = complex_svd_basis(x0, v0, basis_dim)
        if u0.shape[0] == 2 * sharding.N:
            u0 = sharding.local_u(u0 if isinstance(u0, torch.Tensor) else np.asarray(u0))
    with threadpool_limits(limits=4, user_api="blas"), parallel.row_sharded(sharding):
        return _run_reduced(system, params, x0, v0, basis_dim=basis_dim, subsample=subsample,
                            window=window, deim_dim=deim_dim, deim_period=deim_period,
                            deim_update=deim_update, dt=dt, t_final=t_final,
                            svd_tol_dmd=svd_tol_dmd, fp_tol=fp_tol, fp_max_iter=fp_max_iter,
                            hyper_reduction=hyper_reduction,
                            printed_subset_variant=printed_subset_variant,
                            printed_deim_ranking=printed_deim_ranking,
                            energy_stride=energy_stride, snapshot_stride=snapshot_stride,
                            decomp_stride=decomp_stride, record_snapshots=record_snapshots,
                            timers=timers, u0=u0, z0=z0, init=init)


def _run_reduced(system, params, x0, v0, *, basis_dim, subsample, window, deim_dim, deim_period,
                 deim_update, dt, t_final, svd_tol_dmd, fp_tol, fp_max_iter, hyper_reduction,
                 printed_subset_variant, printed_deim_ranking, energy_stride, snapshot_stride,
                 decomp_stride, record_snapshots, timers, u0, z0, init="host"):
    from .diagnostics import PhaseTimers
    params = np.asarray(params, dtype=float)
    num_steps = int(round(t_final / dt))
    snap_stride = (max(1, int(snapshot_stride)) if snapshot_stride is not None
                   else max(1, num_steps // 40))
    timers = timers or PhaseTimers()
    if u0 is None and init == "device":
        from .reduction import complex_svd_basis_device
        u, z = complex_svd_basis_device(x0, v0, basis_dim)
    elif u0 is None:
        u, z = complex_svd_basis(x0, v0, basis_dim, device=True)
    else:
        u = u0 if isinstance(u0, torch.Tensor) else torch.from_numpy(np.asarray(u0)).to("cuda")
        z = np.asarray(z0, dtype=float)
    sub = np.sort(select_parameter_subset(z, subsample, printed_variant=printed_subset_variant))
    subcols = _Cols(sub, z.shape[1])
    pot_window = deque(maxlen=window + 1)
    deim_window = hyp.DeimWindow(window + 1) if hyper_reduction else None
    dmd_model = deim_model = None
    main_counter = 0
    hyper_engaged = False
    full_stage = make_full_stage(system)

    def grad_sub(u_eval, z_sub):
        return exact_gradients_device(system, u_eval, z_sub, subcols, harvest=False)[0]

    energy_times, energies, hams = [], [], []
    snap_times, bases = [], []
    ortho_res = np.zeros(num_steps + 1)
    sympl_res = np.zeros(num_steps + 1)
    fp_iters = np.zeros(num_steps, dtype=int)
    dmd_ranks = np.zeros(num_steps, dtype=int)
    s_conds = np.zeros(num_steps)
    deim_hist = []
    step_seconds = np.zeros(num_steps)
    decomp_times, dh_tot, dh_z, dh_zdd = [], [], [], []
    imag_defect = 0.0

    def ham(u_now, z_now):
        ee, kin = _diag_energies(system, u_now, z_now)
        return kin + ee

    def diagnostics(tau, u_now, z_now):
        t_now = tau * dt
        if tau % energy_stride == 0 or tau == num_steps:
            ee, kin = _diag_energies(system, u_now, z_now)
            energy_times.append(t_now)
            energies.append(ee)
            hams.append(kin + ee)
        if record_snapshots and (tau % snap_stride == 0 or tau == num_steps):
            snap_times.append(t_now)
            bases.append((u_now.clone(), z_now.copy()))

    ortho_res[0], sympl_res[0] = orthosymplectic_residuals(u)
    diagnostics(0, u, z)
    import time as _time
    for tau in range(1, num_steps + 1):
        t_prev = (tau - 1) * dt
        tic = _time.perf_counter()
        try:
            with timers.phase("rom_basis"):
                g_sub0, phi_sub, lam_sub = exact_gradients_device(
                    system, u, z[:, sub], subcols, harvest=hyper_reduction)
            pot_window.append(phi_sub.t().cpu().numpy())
            if hyper_reduction:
                # the window's incremental Gram (new block x window) is the
                # DEIM fit's SVD work: timed with it
                with timers.phase("deim_fit"):
                    deim_window.append(lam_sub)
            hyper_now = hyper_reduction and len(pot_window) == window + 1
            if hyper_now:
                hyper_engaged = True
                # the window Gram's eigensolve (device, worker thread) runs under
                # the host-side DMD fit
                deim_window.prefetch_eigh()
                with timers.phase("dmd_fit"):
                    dmd_model = hyp.fit_parametric_dmd(list(pot_window), dt, t_prev, params, sub,
                                                       svd_tol=svd_tol_dmd)
                with timers.phase("deim_fit"):
                    deim_model = hyp.fit_deim_device(
                        deim_window, deim_dim, system.charge, prev=deim_model,
                        full=(main_counter % deim_period == 0), n_update=deim_update,
                        printed_ranking=printed_deim_ranking)
                main_counter += 1
                stage = hyp.make_hyper_stage_device(dmd_model, deim_model, t_prev + 0.5 * dt,
                                                    system, params)
                deim_hist.append(deim_model.indices.copy())
            else:
                stage = full_stage
            res = prk2_step(u, z, dt, sub, grad_sub, g_sub0, stage, fp_tol=fp_tol,
                            fp_max_iter=fp_max_iter, timers=timers)
        except EvaluationError as err:
            raise DivergenceError(f"reduced state diverged during step {tau} (t = {tau * dt:.6g})",
                                  time=tau * dt) from err
        except StepFailureError as err:
            raise StepFailureError(f"step {tau} (t = {tau * dt:.6g}): {err}",
                                   iterations=err.iterations,
                                   residual_trace=err.residual_trace) from err
        u_prev, z_prev = u, z
        u, z = res.u, res.z
        timers.flush_step()
        step_seconds[tau - 1] = _time.perf_counter() - tic
        ortho_res[tau], sympl_res[tau] = orthosymplectic_residuals(u)
        fp_iters[tau - 1] = res.fp_iterations
        s_conds[tau - 1] = res.s_cond
        if hyper_now:
            dmd_ranks[tau - 1] = dmd_model.rank
            imag_defect = max(imag_defect, dmd_model.imag_defect)
        if hyper_now and decomp_stride and tau % decomp_stride == 0:
            # Hamiltonian-error decomposition (driver.py:229-246): total, the
            # coefficient part at the midpoint basis, and its DMD-DEIM surrogate
            h_new, h_prev = ham(u, z), ham(u_prev, z_prev)
            h_mid_new, h_mid_prev = ham(res.u_mid, z), ham(res.u_mid, z_prev)
            hdd_new = hyp.hyper_hamiltonian_device(dmd_model, deim_model, res.u_mid, z, tau * dt,
                                                   system, params)
            hdd_prev = hyp.hyper_hamiltonian_device(dmd_model, deim_model, res.u_mid, z_prev,
                                                    t_prev, system, params)
            decomp_times.append(tau * dt)
            dh_tot.append(float(np.linalg.norm(np.atleast_1d(h_new - h_prev))))
            dh_z.append(float(np.linalg.norm(np.atleast_1d(h_mid_new - h_mid_prev))))
            dh_zdd.append(float(np.linalg.norm(np.atleast_1d(hdd_new - hdd_prev))))
        diagnostics(tau, u, z)

    notes = {} if hyper_engaged else {"no_hyper_reduction_engaged": True}
    return RomRecord(
        times=dt * np.arange(num_steps + 1), energy_times=np.asarray(energy_times),
        electric_energy=np.asarray(energies), hamiltonian=np.asarray(hams),
        snapshot_times=np.asarray(snap_times), bases=bases, ortho_residuals=ortho_res,
        sympl_residuals=sympl_res, fp_iterations=fp_iters, dmd_ranks=dmd_ranks, s_conds=s_conds,
        decomp_times=np.asarray(decomp_times), dh_total=np.asarray(dh_tot),
        dh_coeff=np.asarray(dh_z), dh_coeff_dd=np.asarray(dh_zdd), timers=timers,
        dmd_imag_defect=imag_defect, hyper_engaged=hyper_engaged, notes=notes,
        deim_indices=deim_hist, step_seconds=step_seconds)
