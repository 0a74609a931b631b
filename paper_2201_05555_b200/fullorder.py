"""Full-order geometric PIC on the GPU -- drop-in for picrom.fullorder.

Mirrors /root/reference/pkg/src/picrom/fullorder.py (ParticleEnsemble,
VlasovSystem, VerletStepper, RecordOptions, FullOrderRecord, run_full_order).

* ``VlasovSystem.field`` = deposit kernel -> circulant Poisson kernel -> gather
  kernel (fullorder.py:66-92); ``workers`` is accepted and ignored (columns are
  batched on the device).
* ``VerletStepper.step`` keeps the reference's kick-drift-kick operation order
  bit for bit (fullorder.py:122-134) with two fused passes
  (picrom_verlet_drift / picrom_verlet_kick) and the same end-of-step field
  cache, so it is the per-step drop-in; duck-typed systems (test doubles with
  a ``field`` method) take the generic array path exactly as the reference.
* ``run_full_order`` is the production loop: the state stays resident in HBM
  in (p, N) layout and each step is ONE fused gather-kick-drift-deposit pass
  over the particles (32 B/push) plus a per-instance solve, captured in a CUDA
  graph and replayed; energies, potentials and charges are recorded on device
  every step.  It integrates the same Stoermer-Verlet map in the algebraically
  identical half-step-velocity form; results agree with the
  reference to rounding.
"""

from __future__ import annotations

import time as _time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as dev
from . import _lib
from .errors import ConfigurationError, DivergenceError, EvaluationError
from .fem import ChargeConfig, PeriodicMesh, PoissonOperator

__all__ = ["ParticleEnsemble", "VlasovSystem", "VerletStepper", "RecordOptions", "run_full_order",
           "FullOrderRecord"]


@dataclass
class ParticleEnsemble:
    """Phase-space state of N particles for p parameter columns (fullorder.py:30-54)."""

    x: object
    v: object
    time: float = 0.0

    def __post_init__(self):
        if not isinstance(self.x, torch.Tensor):
            self.x = np.asarray(self.x, dtype=float)
        if not isinstance(self.v, torch.Tensor):
            self.v = np.asarray(self.v, dtype=float)
        if tuple(self.x.shape) != tuple(self.v.shape):
            raise ConfigurationError("positions and velocities must have equal shapes")

    @property
    def num_particles(self):
        return self.x.shape[0]

    @property
    def num_params(self):
        return 1 if self.x.ndim == 1 else self.x.shape[1]

    def stacked(self):
        if isinstance(self.x, torch.Tensor):
            x = self.x.reshape(self.x.shape[0], -1)
            v = self.v.reshape(self.v.shape[0], -1)
            return torch.cat([x, v], dim=0)
        return np.concatenate([np.atleast_2d(self.x.T).T, np.atleast_2d(self.v.T).T], axis=0)


def _kinetic_device(vd):
    """0.5 * sum v^2 per instance of a (p, N) device array."""
    p, n = vd.shape
    out = torch.empty(p, dtype=torch.float64, device="cuda")
    _lib.call("picrom_half_sumsq", vd.data_ptr(), n, p, n, out.data_ptr(), None,
              dev.stream_handle())
    return out


class VlasovSystem:
    """Grid, charge data, and the field evaluation they define (fullorder.py:57-99)."""

    def __init__(self, mesh: PeriodicMesh, charge: ChargeConfig, workers: int = 1):
        self.mesh = mesh
        self.charge = charge
        self.poisson = PoissonOperator(mesh)
        self.workers = max(1, int(workers))

    # -------------------------------------------------------------- device
    def inst(self, p):
        return dev.inst_rows(self.mesh, self.charge, p)

    def field_device(self, xd, ndim=2, want_rho=False, want_energy=False):
        """(E, phi[, rho][, energy]) on device for (p, N) positions xd."""
        p, n = xd.shape
        mesh = self.mesh
        nx, d = mesh.num_cells, mesh.degree
        inst = self.inst(p)
        c = self.poisson.constants
        s = dev.stream_handle()
        rho = torch.empty((p, nx), dtype=torch.float64, device="cuda")
        phi = torch.empty_like(rho)
        ee = torch.empty(p, dtype=torch.float64, device="cuda") if want_energy else None
        st = dev.new_status()
        _lib.call("picrom_deposit", xd.data_ptr(), n, p, n, inst.data_ptr(), nx, d,
                  rho.data_ptr(), dev.workspace(n, p, nx, d).data_ptr(), st.data_ptr(), s)
        dev.raise_if_bad(st, p, ndim)
        _lib.call("picrom_poisson", rho.data_ptr(), p, nx, d, inst.data_ptr(), c.khat.data_ptr(),
                  c.stencil.data_ptr(), phi.data_ptr(), dev.ptr(ee), s)
        e = torch.empty_like(xd)
        _lib.call("picrom_gather", xd.data_ptr(), n, p, n, inst.data_ptr(), nx, d, phi.data_ptr(),
                  1, e.data_ptr(), n, st.data_ptr(), s)
        out = (e, phi)
        if want_rho:
            out = out + (rho,)
        if want_energy:
            out = out + (ee,)
        return out

    # ------------------------------------------------------- reference API
    def field(self, x):
        """Per-particle field and nodal potential for each parameter column."""
        xd, meta = dev.to_device(x)
        e, phi = self.field_device(xd, meta.ndim)
        return dev.from_device(e, meta), dev.from_device(phi, meta)

    def hamiltonian(self, x, v):
        from .fem import hamiltonian
        return hamiltonian(x, v, self.poisson, self.charge)


def _is_device_system(system):
    return isinstance(system, VlasovSystem)


class VerletStepper:
    """Kick-drift-kick step; the closing field evaluation seeds the next step."""

    def __init__(self, system):
        self.system = system
        self._cache_time = None
        self._cache_field = None
        self.last_potential = None
        self._dev_cache = None          # (time, E (p, N) device) mirror of _cache_field

    def _field(self, x, time):
        try:
            return self.system.field(x)
        except EvaluationError as err:
            pidx = err.index[1] if err.index is not None and len(err.index) > 1 else err.index
            raise DivergenceError(
                f"state diverged at t = {time:.6g} (parameter index {pidx})",
                parameter_index=pidx, time=time) from err

    def step(self, ens: ParticleEnsemble, dt: float) -> ParticleEnsemble:
        if not _is_device_system(self.system):
            return self._generic_step(ens, dt)
        sysm = self.system
        xd, meta = dev.to_device(ens.x)
        vd, _ = dev.to_device(ens.v)
        p, n = xd.shape
        mesh = sysm.mesh
        nx, d = mesh.num_cells, mesh.degree
        if self._cache_time == ens.time and self._cache_field is not None:
            if self._dev_cache is not None and self._dev_cache[0] == ens.time:
                e0 = self._dev_cache[1]
            else:
                e0, _ = dev.to_device(self._cache_field)
        else:
            try:
                e0, phi0 = sysm.field_device(xd, meta.ndim)
            except EvaluationError as err:
                pidx = err.index[1] if err.index is not None and len(err.index) > 1 else err.index
                raise DivergenceError(
                    f"state diverged at t = {ens.time:.6g} (parameter index {pidx})",
                    parameter_index=pidx, time=ens.time) from err
            self.last_potential = dev.from_device(phi0, meta)
        t1 = ens.time + dt
        inst = sysm.inst(p)
        c = sysm.poisson.constants
        s = dev.stream_handle()
        x1 = torch.empty_like(xd)
        phi1 = torch.empty((p, nx), dtype=torch.float64, device="cuda")
        st = dev.new_status()
        _lib.call("picrom_verlet_drift", xd.data_ptr(), vd.data_ptr(), e0.data_ptr(), n, p, n,
                  inst.data_ptr(), nx, d, c.khat.data_ptr(), c.stencil.data_ptr(), float(dt), 0,
                  x1.data_ptr(), phi1.data_ptr(), None, None,
                  dev.workspace(n, p, nx, d).data_ptr(), st.data_ptr(), s)
        bad = dev.decode_status(st, p)
        if bad is not None:
            pidx = bad[2] if meta.ndim > 1 else bad[1]
            raise DivergenceError(f"state diverged at t = {t1:.6g} (parameter index {pidx})",
                                  parameter_index=pidx, time=t1)
        e1 = torch.empty_like(xd)
        v1 = torch.empty_like(xd)
        _lib.call("picrom_verlet_kick", x1.data_ptr(), vd.data_ptr(), e0.data_ptr(), n, p, n,
                  inst.data_ptr(), nx, d, phi1.data_ptr(), float(dt), e1.data_ptr(),
                  v1.data_ptr(), s)
        self._cache_time = t1
        self._cache_field = dev.from_device(e1, meta)
        self._dev_cache = (t1, e1)
        self.last_potential = dev.from_device(phi1, meta)
        return ParticleEnsemble(dev.from_device(x1, meta), dev.from_device(v1, meta), t1)

    def _generic_step(self, ens, dt):
        # duck-typed system (fullorder.py:122-134, identical arithmetic)
        if self._cache_time == ens.time and self._cache_field is not None:
            e0 = self._cache_field
        else:
            e0, self.last_potential = self._field(ens.x, ens.time)
        x1 = ens.x + dt * (ens.v + 0.5 * dt * e0)
        t1 = ens.time + dt
        e1, phi1 = self._field(x1, t1)
        v1 = ens.v + 0.5 * dt * (e0 + e1)
        self._cache_time = t1
        self._cache_field = e1
        self.last_potential = phi1
        return ParticleEnsemble(x1, v1, t1)


@dataclass
class RecordOptions:
    """What a trajectory run keeps (fullorder.py:137-149)."""

    energy_stride: int = 10
    snapshot_stride: int | None = None
    record_snapshots: bool = True

    def resolved_snapshot_stride(self, num_steps):
        if self.snapshot_stride is not None:
            return max(1, int(self.snapshot_stride))
        return max(1, num_steps // 40)


@dataclass
class FullOrderRecord:
    """Time series and snapshots from a full-order run (fullorder.py:152-166)."""

    times: np.ndarray
    energy_times: np.ndarray
    electric_energy: np.ndarray
    hamiltonian: np.ndarray
    potential_times: np.ndarray
    potentials: np.ndarray
    snapshot_times: np.ndarray
    snapshots_x: np.ndarray
    snapshots_v: np.ndarray
    step_seconds: np.ndarray
    phase_seconds: dict = field(default_factory=dict)
    # extras (not in the reference record): every-step device histories
    charge_history: np.ndarray | None = None       # (steps+1, Nx, p)
    potential_history: np.ndarray | None = None    # (steps+1, Nx, p)
    electric_history: np.ndarray | None = None     # (steps+1, p)
    kinetic_history: np.ndarray | None = None      # (steps+1, p)
    final_state: object = None                     # ParticleEnsemble at t_final


def _auto_groups(p, n):
    """Instance groups pipelined on separate streams: while one group's step
    drains (last CTAs, per-instance solve) the next group streams particles.
    Worth it where the per-step fixed cost is a visible share of the step
    (C2: 8 M particles, ~80 us); a single group for huge steps (C5) or p = 1."""
    if p < 2:
        return 1
    return 2 if n * p <= (64 << 20) else 1


class PicEngine:
    """Persistent device state of the leapfrog loop for one (system, p, N, dt):
    x, v (p, N), phi, per-group workspaces, status words and step counters,
    ring histories, plus one captured CUDA graph of `graph_steps` steps that
    every later run replays (all its pointers live here, so the graph stays
    valid).  The p instances are split into `groups` contiguous instance
    groups, each stepped by its own chain of fused kernels on its own stream;
    the chains only join at the ends of a block of steps, so one group's
    per-step tail (the last CTAs and the in-kernel Poisson solve) overlaps the
    next group's particle streaming."""

    def __init__(self, system, p, n, dt, graph_steps=64, groups=None):
        self.system = system
        self.p, self.n, self.dt = p, n, float(dt)
        mesh = system.mesh
        self.nx, self.degree = mesh.num_cells, mesh.degree
        self.inst = system.inst(p)
        self.c = system.poisson.constants
        self.groups = _auto_groups(p, n) if groups is None else max(1, min(int(groups), p))
        edges = np.linspace(0, p, self.groups + 1).astype(int)
        self.slices = [(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:])]
        self.ws = [torch.zeros(int(_lib.query("picrom_fom_workspace_bytes", n, b - a, self.nx,
                                              self.degree)), dtype=torch.uint8, device="cuda")
                   for a, b in self.slices]
        self.x = torch.empty((p, n), dtype=torch.float64, device="cuda")
        self.v = torch.empty((p, n), dtype=torch.float64, device="cuda")
        self.phi = torch.empty((p, self.nx), dtype=torch.float64, device="cuda")
        self.status = [dev.new_status() for _ in self.slices]
        self.init_status = dev.new_status()      # the initial all-instance deposit
        self.counters = [torch.zeros(2, dtype=torch.int64, device="cuda") for _ in self.slices]
        self.streams = [torch.cuda.Stream() for _ in self.slices] if self.groups > 1 else None
        self.ring = int(graph_steps)
        self.r_rho = torch.zeros((self.ring, p, self.nx), dtype=torch.float64, device="cuda")
        self.r_phi = torch.zeros_like(self.r_rho)
        self.r_ee = torch.zeros((self.ring, p), dtype=torch.float64, device="cuda")
        self.r_kin = torch.zeros_like(self.r_ee)
        # %globaltimer at the end of each ring step, per instance group
        self.r_t = torch.zeros((self.groups, self.ring), dtype=torch.int64, device="cuda")
        self.graph = None
        self.launches = 0

    def reset(self):
        self.init_status.fill_(-1)
        for st in self.status:
            st.fill_(-1)
        for ct in self.counters:
            ct.zero_()

    def _launch_group(self, g, first, stream):
        """One PIC step of instance group g: a single fused kernel (push +
        last-CTA solve) writing its slice of the shared ring histories."""
        a, b = self.slices[g]
        dt = self.dt
        kick, kfull = (0.5 * dt, 0.0) if first else (dt, 0.5 * dt)
        n, nx = self.n, self.nx
        _lib.call("picrom_pic_step", self.x.data_ptr() + 8 * a * n, self.v.data_ptr() + 8 * a * n,
                  n, b - a, n, self.inst.data_ptr() + 8 * dev.INST_STRIDE * a, nx, self.degree,
                  self.c.khat.data_ptr(), self.c.stencil.data_ptr(),
                  self.phi.data_ptr() + 8 * a * nx, dt, kick, kfull, 0,
                  self.counters[g].data_ptr(), self.ring, self.p,
                  self.r_rho.data_ptr() + 8 * a * nx, self.r_phi.data_ptr() + 8 * a * nx,
                  self.r_ee.data_ptr() + 8 * a, self.r_kin.data_ptr() + 8 * a,
                  self.r_t[g].data_ptr(), self.ws[g].data_ptr(), self.status[g].data_ptr(), stream)
        self.launches += 1

    def launch_block(self, steps, first=False):
        """`steps` consecutive PIC steps of every instance group; the group
        chains fork from and join the current stream once per block."""
        if self.streams is None:
            for k in range(steps):
                self._launch_group(0, first and k == 0, dev.stream_handle())
            return
        # group 0 runs on the current stream itself: one fork and one join per
        # extra group instead of two
        main = torch.cuda.current_stream()
        side = self.streams[1:]
        for st in side:
            st.wait_stream(main)
        for k in range(steps):
            for g in range(self.groups):
                stream = main.cuda_stream if g == 0 else self.streams[g].cuda_stream
                self._launch_group(g, first and k == 0, stream)
        for st in side:
            main.wait_stream(st)

    def launch(self, first):
        self.launch_block(1, first)

    def replay(self):
        if self.graph is None:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.launch_block(self.ring)
            self.launches -= self.ring * self.groups
            self.graph = g
        self.graph.replay()
        self.launches += self.ring * self.groups

    def bad(self):
        """None, or (step, row, global column) of the first non-finite position."""
        worst = None
        for (a, b), st in [((0, self.p), self.init_status)] + list(zip(self.slices, self.status)):
            bad = dev.decode_status(st, b - a)
            if bad is not None:
                bad = (bad[0], bad[1], bad[2] + a)
                if worst is None or (bad[0], bad[1] * self.p + bad[2]) < (worst[0], worst[1] * self.p + worst[2]):
                    worst = bad
        return worst


def _engine(system, p, n, dt, groups=None):
    cache = system.__dict__.setdefault("_engines", {})
    key = (p, n, float(dt), torch.cuda.current_device(), groups)
    eng = cache.get(key)
    if eng is None:
        cache.clear()                      # one resident engine per system
        eng = cache[key] = PicEngine(system, p, n, dt, groups=groups)
    return eng


class PicRun:
    """Device-resident leapfrog PIC loop (the production path of run_full_order).

    State lives in a cached PicEngine: x (p, N), v (p, N) -- v holds v_0 before
    the first step and the half-step velocity v_{n-1/2} afterwards.  Each step
    is picrom_pic_push + picrom_pic_solve; blocks of `ring` steps replay one
    CUDA graph.  Histories (device): rho/phi (steps+1, p, Nx), electric and
    kinetic energy (steps+1, p), filled from the engine's ring after each block.
    """

    def __init__(self, system, xd, vd, dt, num_steps, keep_rho=True, groups=None):
        self.system = system
        self.p, self.n = xd.shape
        self.e = _engine(system, self.p, self.n, dt, groups)
        self.e.x.copy_(xd)
        self.e.v.copy_(vd)
        self.e.reset()
        self.dt = float(dt)
        self.num_steps = int(num_steps)
        self.nx, self.degree = self.e.nx, self.e.degree
        rows = self.num_steps + 1
        self.rho_hist = (torch.zeros((rows, self.p, self.nx), dtype=torch.float64, device="cuda")
                         if keep_rho else None)
        self.phi_hist = torch.zeros((rows, self.p, self.nx), dtype=torch.float64, device="cuda")
        self.ee_hist = torch.zeros((rows, self.p), dtype=torch.float64, device="cuda")
        self.kin_hist = torch.zeros((rows, self.p), dtype=torch.float64, device="cuda")
        # device step end times (ns): row 0 = after the initial field, row k =
        # when step k's last instance-group solve finished (max over groups)
        self.t_hist = torch.zeros((self.e.groups, rows), dtype=torch.int64, device="cuda")
        self.tau = 0

    @property
    def x(self):
        return self.e.x

    @property
    def v(self):
        return self.e.v

    @property
    def phi(self):
        return self.e.phi

    @property
    def launches(self):
        return self.e.launches

    def init_field(self):
        """Initial deposit + solve (fullorder.py:183-186): phi_0, rho_0, energy_0."""
        e = self.e
        s = dev.stream_handle()
        rho0 = self.rho_hist[0] if self.rho_hist is not None else torch.empty(
            (self.p, self.nx), dtype=torch.float64, device="cuda")
        ws = dev.workspace(self.n, self.p, self.nx, self.degree)
        _lib.call("picrom_deposit", e.x.data_ptr(), self.n, self.p, self.n, e.inst.data_ptr(),
                  self.nx, self.degree, rho0.data_ptr(), ws.data_ptr(), e.init_status.data_ptr(), s)
        _lib.call("picrom_poisson", rho0.data_ptr(), self.p, self.nx, self.degree,
                  e.inst.data_ptr(), e.c.khat.data_ptr(), e.c.stencil.data_ptr(),
                  e.phi.data_ptr(), self.ee_hist[0].data_ptr(), s)
        self.phi_hist[0].copy_(e.phi)
        _lib.call("picrom_timestamp", self.t_hist[0, 0:1].data_ptr(), s)
        e.launches += 4

    def _drain(self, c0, count):
        """Copy ring rows of counters [c0, c0+count) into the full histories:
        the ring positions are contiguous modulo the ring, so at most two
        contiguous device-to-device copies per history (no index kernels)."""
        e = self.e
        r0 = c0 % e.ring
        parts = [(r0, min(count, e.ring - r0))]
        if parts[0][1] < count:
            parts.append((0, count - parts[0][1]))
        done = 0
        for r, m in parts:
            t = c0 + done
            self.kin_hist[t:t + m].copy_(e.r_kin[r:r + m])
            self.ee_hist[t + 1:t + m + 1].copy_(e.r_ee[r:r + m])
            self.phi_hist[t + 1:t + m + 1].copy_(e.r_phi[r:r + m])
            if self.rho_hist is not None:
                self.rho_hist[t + 1:t + m + 1].copy_(e.r_rho[r:r + m])
            for g in range(e.groups):
                self.t_hist[g, t + 1:t + m + 1].copy_(e.r_t[g, r:r + m])
            done += m

    def advance(self, k, use_graph=True):
        """Advance k steps; full ring-sized blocks replay the cached graph."""
        e = self.e
        while k > 0:
            if self.tau == 0:
                e.launch(first=True)
                self._drain(0, 1)
                self.tau, k = 1, k - 1
                continue
            if use_graph and k >= e.ring:
                e.replay()
                self._drain(self.tau, e.ring)
                self.tau += e.ring
                k -= e.ring
                continue
            # remainder (< one ring): one block of plain launches, one drain --
            # every fork/join of the group streams costs ~50 us of pipeline
            # fill and drain (measured: 67.1 us/step in 20-step blocks, 64.7 in
            # 100-step blocks at C2)
            m = min(k, e.ring)
            e.launch_block(m)
            self._drain(self.tau, m)
            self.tau += m
            k -= m

    def step_seconds(self):
        """Device seconds of each completed step (host array, one sync)."""
        t = self.t_hist[:, :self.tau + 1].cpu().numpy().max(axis=0).astype(np.float64)
        return np.diff(t) * 1e-9

    def full_velocity(self):
        """v_tau = v_{tau-1/2} + 0.5 dt E(x_tau) (device), or v_0 before any step."""
        e = self.e
        if self.tau == 0:
            return e.v.clone()
        ef = torch.empty_like(e.x)
        zeros = torch.zeros_like(e.x)
        vfull = torch.empty_like(e.x)
        _lib.call("picrom_verlet_kick", e.x.data_ptr(), e.v.data_ptr(), zeros.data_ptr(),
                  self.n, self.p, self.n, e.inst.data_ptr(), self.nx, self.degree,
                  e.phi.data_ptr(), self.dt, ef.data_ptr(), vfull.data_ptr(), dev.stream_handle())
        e.launches += 1
        return vfull

    def finish_kinetic(self):
        """Kinetic energy of the final full-step velocity into kin_hist[tau]."""
        vfull = self.full_velocity()
        _lib.call("picrom_half_sumsq", vfull.data_ptr(), self.n, self.p, self.n,
                  self.kin_hist[self.tau].data_ptr(), None, dev.stream_handle())
        self.e.launches += 1
        return vfull

    def check(self):
        bad = self.e.bad()
        if bad is not None:
            step, row, col = bad
            t = step * self.dt
            raise DivergenceError(f"state diverged at t = {t:.6g} (parameter index {col})",
                                  parameter_index=col, time=t)


def run_full_order(system, initial: ParticleEnsemble, dt, t_final,
                   record: RecordOptions | None = None) -> FullOrderRecord:
    """March the Verlet scheme to t_final and collect the requested series
    (fullorder.py:169-226)."""
    if dt <= 0 or t_final <= 0:
        raise ConfigurationError("dt and t_final must be positive")
    if not _is_device_system(system):
        return _run_generic(system, initial, dt, t_final, record)
    record = record or RecordOptions()
    num_steps = int(round(t_final / dt))
    snap_stride = record.resolved_snapshot_stride(num_steps)
    xd, meta = dev.to_device(initial.x)
    vd, _ = dev.to_device(initial.v)
    p = xd.shape[0]
    run = PicRun(system, xd, vd, dt, num_steps)

    snaps_t, snaps_x, snaps_v = [], [], []

    def snapshot(tau):
        snaps_t.append(tau * dt)
        snaps_x.append(dev.from_device(run.x, meta))
        snaps_v.append(dev.from_device(run.full_velocity(), meta))

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    run.init_field()
    try:
        run.check()
    except DivergenceError as err:
        raise DivergenceError(str(err), parameter_index=err.parameter_index, time=0.0) from None
    if record.record_snapshots:
        snapshot(0)
    stops = sorted({t for t in range(snap_stride, num_steps + 1, snap_stride)} | {num_steps}) \
        if record.record_snapshots else [num_steps]
    for stop in stops:
        run.advance(stop - run.tau)
        if record.record_snapshots:
            run.check()
            snapshot(stop)
    vfinal = run.finish_kinetic()
    ev1.record()
    ev1.synchronize()
    run.check()
    total = ev0.elapsed_time(ev1) / 1e3

    # host-side assembly of the reference record at the requested strides
    ee = dev.to_host(run.ee_hist)
    kin = dev.to_host(run.kin_hist)
    phi = dev.to_host(run.phi_hist).transpose(0, 2, 1)         # (rows, Nx, p)
    rho = dev.to_host(run.rho_hist).transpose(0, 2, 1) if run.rho_hist is not None else None
    taus = [t for t in range(num_steps + 1) if t % record.energy_stride == 0 or t == num_steps]
    energy_times = np.asarray([t * dt for t in taus])
    electric = ee[taus]
    ham = kin[taus] + ee[taus]
    pots = phi[taus]
    if meta.ndim == 1:
        pots = pots.reshape(len(taus), system.mesh.num_cells, 1)
    step_seconds = run.step_seconds()
    final = ParticleEnsemble(dev.from_device(run.x, meta), dev.from_device(vfinal, meta),
                             num_steps * dt)
    shape = tuple(initial.x.shape)
    return FullOrderRecord(
        times=dt * np.arange(num_steps + 1),
        energy_times=energy_times,
        electric_energy=electric,
        hamiltonian=ham,
        potential_times=energy_times.copy(),
        potentials=pots,
        snapshot_times=np.asarray(snaps_t),
        snapshots_x=_stack(snaps_x, shape),
        snapshots_v=_stack(snaps_v, shape),
        step_seconds=step_seconds,
        phase_seconds={"fom_step": float(total)},
        charge_history=rho,
        potential_history=phi,
        electric_history=ee,
        kinetic_history=kin,
        final_state=final,
    )


def _stack(items, shape):
    if not items:
        return np.empty((0,) + shape)
    if isinstance(items[0], torch.Tensor):
        return torch.stack(items).cpu().numpy()
    return np.asarray(items)


def _run_generic(system, initial, dt, t_final, record):
    """Reference loop for duck-typed systems (fullorder.py:169-226)."""
    from .fem import electric_energy
    record = record or RecordOptions()
    num_steps = int(round(t_final / dt))
    snap_stride = record.resolved_snapshot_stride(num_steps)
    stepper = VerletStepper(system)
    ens = initial
    e0, phi0 = stepper._field(ens.x, ens.time)
    stepper._cache_time, stepper._cache_field, stepper.last_potential = ens.time, e0, phi0
    p = initial.num_params
    energy_times, energies, hams, pot_list = [], [], [], []
    snap_times, snaps_x, snaps_v = [], [], []
    step_seconds = np.zeros(num_steps)

    def record_state(tau, ens, phi):
        if tau % record.energy_stride == 0 or tau == num_steps:
            energy_times.append(ens.time)
            ee = np.atleast_1d(electric_energy(system.poisson, phi, system.charge))
            kin = 0.5 * np.einsum("i...,i...->...", ens.v, ens.v)
            energies.append(ee)
            hams.append(np.atleast_1d(kin) + ee)
            pot_list.append(np.asarray(phi).reshape(system.mesh.num_cells, p).copy())
        if record.record_snapshots and (tau % snap_stride == 0 or tau == num_steps):
            snap_times.append(ens.time)
            snaps_x.append(np.array(ens.x, copy=True))
            snaps_v.append(np.array(ens.v, copy=True))

    record_state(0, ens, phi0)
    for tau in range(1, num_steps + 1):
        tic = _time.perf_counter()
        ens = stepper.step(ens, dt)
        step_seconds[tau - 1] = _time.perf_counter() - tic
        record_state(tau, ens, stepper.last_potential)
    energy_times = np.asarray(energy_times)
    return FullOrderRecord(
        times=dt * np.arange(num_steps + 1), energy_times=energy_times,
        electric_energy=np.asarray(energies), hamiltonian=np.asarray(hams),
        potential_times=energy_times.copy(), potentials=np.asarray(pot_list),
        snapshot_times=np.asarray(snap_times),
        snapshots_x=np.asarray(snaps_x) if snaps_x else np.empty((0,) + np.shape(ens.x)),
        snapshots_v=np.asarray(snaps_v) if snaps_v else np.empty((0,) + np.shape(ens.v)),
        step_seconds=step_seconds, phase_seconds={"fom_step": float(step_seconds.sum())},
        final_state=ens)
