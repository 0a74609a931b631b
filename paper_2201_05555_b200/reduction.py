"""Dynamical ortho-symplectic reduced basis on the GPU -- drop-in for picrom.reduction.

Same functions and argument meaning as /root/reference/pkg/src/picrom/
reduction.py (jmul, jrmul, complex_svd_basis, reconstruct,
orthosymplectic_residuals, SMatrix, select_parameter_subset, basis_velocity,
retraction, tangent_velocity, fixed_point, prk2_step, PRKResult).

The basis U (2N x n) stays on the device; every O(N) product is either one
tall-skinny Gram (picrom_paired_gram) or one tall-skinny combine
(picrom_combine).  The n x n / 2n x 2n algebra between them (Cholesky of S,
capacitance solve, transport solves) runs on the host in numpy/LAPACK exactly
as in the reference, from device-computed Grams:

* basis_velocity  (reduction.py:143-153): one Gram of [U, GZ^T, J GZ^T],
  one combine  xi = (J GZ^T) S^-1 + GZ^T (J S^-1) - U Q
* retraction      (reduction.py:156-167): one Gram of [U, xi], one combine
  U (I - M Y1/2 - Y2) + xi Y1 with the capacitance solve in between
* tangent_velocity (reduction.py:170-182): one Gram of [U, xi, r, x_eval],
  one combine
Small inputs (Z, S, subsets) are host numpy arrays as in the reference;
tall ones are CUDA tensors (numpy tall inputs are uploaded and the result
returned as numpy).
"""

from __future__ import annotations

import warnings
from contextlib import nullcontext
from dataclasses import dataclass

import numpy as np
import torch
from scipy.linalg import cho_factor, cho_solve, eigvalsh, svd

from . import _tall
from .errors import ConfigurationError, StepFailureError

__all__ = [
    "jmul", "jrmul", "complex_svd_basis", "reconstruct", "orthosymplectic_residuals", "SMatrix",
    "select_parameter_subset", "basis_velocity", "retraction", "tangent_velocity", "fixed_point",
    "prk2_step", "PRKResult", "complex_svd_basis_device",
]


def jmul(m):
    """J @ m for J = [[0, I], [-I, 0]] (reduction.py:44-47)."""
    half = m.shape[0] // 2
    if isinstance(m, torch.Tensor):
        return torch.cat([m[half:], -m[:half]], dim=0)
    return np.concatenate([m[half:], -m[:half]], axis=0)


def jrmul(m):
    """m @ J (reduction.py:50-53)."""
    half = m.shape[1] // 2
    if isinstance(m, torch.Tensor):
        return torch.cat([-m[:, half:], m[:, :half]], dim=1)
    return np.concatenate([-m[:, half:], m[:, :half]], axis=1)


class Scaled:
    """c * a for a tall device operand, kept lazy: retraction and
    tangent_velocity fold c into their Gram blocks and combine coefficients,
    so the PRK step's dt/2 * xi and dt * xi2 (reduction.py:236,258) cost no pass."""

    def __init__(self, a, c):
        self.a, self.c = a, float(c)

    @property
    def shape(self):
        return self.a.shape

    def materialize(self):
        ad, _ = _tall_in(self.a)
        return _tall.combine([(ad, self.c * np.eye(ad.shape[1]), False)])


def _scaled_in(a):
    """(CUDA tensor, scale, was_numpy) of a possibly lazy-scaled tall operand."""
    if isinstance(a, Scaled):
        t, _ = _tall_in(a.a)
        return t, a.c, False
    t, was_np = _tall_in(a)
    return t, 1.0, was_np


def _tall_in(a):
    """(CUDA tensor, was_numpy) for a tall operand."""
    if isinstance(a, Scaled):
        return a.materialize(), False
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=torch.float64).contiguous(), False
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to("cuda"), True


def _tall_out(t, was_numpy):
    return t.cpu().numpy() if was_numpy else t


def complex_svd_basis(x, v, n, device=False):
    """U = [[Phi, -Psi], [Psi, Phi]] from the complex SVD of x + i v (reduction.py:56-76).

    One-time initialisation: the SVD runs in host LAPACK exactly as in the
    reference (bit-identical U, Z); ``device=True`` returns U as a CUDA tensor.
    """
    if isinstance(x, torch.Tensor):
        x = x.cpu().numpy()
    if isinstance(v, torch.Tensor):
        v = v.cpu().numpy()
    x = np.atleast_2d(np.asarray(x, dtype=float).T).T
    v = np.atleast_2d(np.asarray(v, dtype=float).T).T
    if n % 2 or n < 2:
        raise ConfigurationError(f"basis dimension must be even and >= 2, got {n}")
    half = n // 2
    if half > min(x.shape):
        raise ConfigurationError(f"rank {half} complex basis needs at least {half} snapshots")
    uc = svd(x + 1j * v, full_matrices=False)[0]
    phi, psi = uc[:, :half].real, uc[:, :half].imag
    u = np.block([[phi, -psi], [psi, phi]])
    bign = x.shape[0]
    z = u[:bign].T @ x + u[bign:].T @ v
    if device:
        return torch.from_numpy(u).to("cuda"), z
    return u, z


def complex_svd_basis_device(x, v, n):
    """Device initial basis: the ortho-symplectic U of complex_svd_basis
    (reduction.py:56-76) from the p x p Hermitian Gram of A = x + i v instead of
    a host SVD of the N x p complex matrix (11 s of LAPACK at C3).

      A^H A = (X^T X + V^T V) + i (X^T V - V^T X)   one N-row Gram of [X, V]
      A^H A W = W Sigma^2                            p x p Hermitian eigensolve (host)
      A W_k Sigma_k^-1 = Phi + i Psi                 two N-row combines
      Z = U^T [x; v]                                 one N-row cross Gram

    Singular vectors are defined up to a phase per vector: the host LAPACK
    path and this one agree up to a per-column rotation of (Phi_j, Psi_j)
    (an ortho-symplectic change of reduced coordinates, under which U Z and
    every reduced quantity are invariant); tests compare modulo that phase.
    Returns (U (2N x n) CUDA tensor, Z (n x p) host)."""
    from scipy.linalg import eigh
    if n % 2 or n < 2:
        raise ConfigurationError(f"basis dimension must be even and >= 2, got {n}")
    xd, _ = _tall_in(x if not isinstance(x, np.ndarray) or x.ndim == 2 else np.atleast_2d(x.T).T)
    vd, _ = _tall_in(v if not isinstance(v, np.ndarray) or v.ndim == 2 else np.atleast_2d(v.T).T)
    N, p = xd.shape
    half = n // 2
    if half > min(N, p):
        raise ConfigurationError(f"rank {half} complex basis needs at least {half} snapshots")
    xx = _tall.gram([(xd, False)])
    vv = _tall.gram([(vd, False)])
    xv = _tall.cross_gram([(xd, False)], [(vd, False)])
    herm = (xx + vv) + 1j * (xv - xv.T)
    lam, w = eigh(herm)
    order = np.argsort(lam)[::-1][:half]
    lam, w = lam[order], w[:, order]
    sig = np.sqrt(np.clip(lam, 0.0, None))
    wr, wi = w.real / sig, w.imag / sig
    phi = _tall.combine([(xd, wr, False), (vd, -wi, False)])          # Re(A W / sigma)
    psi = _tall.combine([(xd, wi, False), (vd, wr, False)])           # Im(A W / sigma)
    u = torch.empty((2 * N, n), dtype=torch.float64, device="cuda")
    u[:N, :half] = phi
    u[:N, half:] = -psi
    u[N:, :half] = psi
    u[N:, half:] = phi
    # Z = U_X^T x + U_V^T v (two N-row cross Grams)
    zx = _tall.cross_gram([(u[:N], False)], [(xd, False)])
    zv = _tall.cross_gram([(u[N:], False)], [(vd, False)])
    return u, zx + zv


def reconstruct(u, z):
    """(U_X z, U_V z) (reduction.py:79-82); a plain library GEMM off the hot path
    (the hot path never forms the reconstruction, see rom_field/rom_gather)."""
    ud, was_np = _tall_in(u)
    zd = torch.as_tensor(np.asarray(z, dtype=np.float64) if not isinstance(z, torch.Tensor) else z,
                         dtype=torch.float64, device="cuda")
    half = ud.shape[0] // 2
    return _tall_out(ud[:half] @ zd, was_np), _tall_out(ud[half:] @ zd, was_np)


def orthosymplectic_residuals(u):
    """(||U^T U - I||_F, ||U^T J U - J_n||_F) (reduction.py:85-90) from one Gram."""
    ud, _ = _tall_in(u)
    n = ud.shape[1]
    G = _tall.gram([(ud, False), (ud, True)])
    utu, utju = G[:n, :n], G[:n, n:]
    return (float(np.linalg.norm(utu - np.eye(n))),
            float(np.linalg.norm(utju - jmul(np.eye(n)))))


class SMatrix:
    """Coefficient Gram S = Z Z^T + J^T Z Z^T J, Cholesky-factored (reduction.py:93-107).

    Z is a host (n x p*) array; the algebra is the reference's, in LAPACK."""

    def __init__(self, z, cond_warn=1e12):
        z = np.asarray(z, dtype=float)
        a = z @ z.T
        self.matrix = a - jmul(jrmul(a))
        eigs = eigvalsh(self.matrix)
        self.cond = float(eigs[-1] / max(eigs[0], np.finfo(float).tiny))
        if self.cond > cond_warn:
            warnings.warn(f"coefficient Gram matrix is ill-conditioned (cond ~ {self.cond:.2e})")
        self._cho = cho_factor(self.matrix)

    def solve_right(self, m):
        return cho_solve(self._cho, np.asarray(m).T).T


def select_parameter_subset(z, count, printed_variant=False):
    """Farthest-point greedy subsample of coefficient columns (reduction.py:110-140)."""
    z = np.asarray(z, dtype=float)
    p = z.shape[1]
    if not 1 <= count <= p:
        raise ConfigurationError(f"subset size must be in [1, {p}], got {count}")
    sel = [int(np.argmax(np.einsum("ij,ij->j", z, z)))]
    if printed_variant:
        for j in range(p):
            if len(sel) == count:
                break
            if j not in sel:
                sel.append(j)
        return np.asarray(sel, dtype=int)
    diff = z - z[:, [sel[0]]]
    d2 = np.einsum("ij,ij->j", diff, diff)
    while len(sel) < count:
        nxt = int(np.argmax(d2))
        sel.append(nxt)
        diff = z - z[:, [nxt]]
        d2 = np.minimum(d2, np.einsum("ij,ij->j", diff, diff))
    return np.asarray(sel, dtype=int)


def _times_zt(g, z):
    """G Z^T as a (2N x n) device tensor; G dense (2N x p') or a lazy device gradient."""
    if hasattr(g, "times_matrix"):
        return g.times_matrix(np.asarray(z, dtype=float).T)
    gd, _ = _tall_in(g)
    return _tall.combine([(gd, np.asarray(z, dtype=float).T, False)])


def basis_velocity(u, z, g, s=None):
    """(I - U U^T)(J G Z^T - G Z^T J^T) S^{-1} (reduction.py:143-153)."""
    ud, was_np = _tall_in(u)
    z = np.asarray(z, dtype=float)
    s = s or SMatrix(z)
    n = ud.shape[1]
    s_inv = s.solve_right(np.eye(n))
    js_inv = jmul(s_inv)                         # (G Z^T J) S^-1 = G Z^T (J S^-1)
    if getattr(g, "ux_e", None) is not None:
        return _tall_out(_basis_velocity_device(ud, z, g, s_inv, js_inv), was_np)
    gzt = _times_zt(g, z)
    G = _tall.gram_tasks([(ud, False), (gzt, False), (gzt, True)], [(0, 1), (0, 2)])
    u_gzt, u_jgzt = G[:n, n:2 * n], G[:n, 2 * n:]
    q = u_jgzt @ s_inv + u_gzt @ js_inv          # U^T m
    xi = _tall.combine([(gzt, s_inv, True), (gzt, js_inv, False), (ud, -q, False)])
    return _tall_out(xi, was_np)


def _basis_velocity_device(ud, z, g, s_inv, js_inv):
    """basis_velocity for an implicit device gradient G = [E; U_V Z] whose gather
    also returned U_X^T E and U_V^T E: with H = Z Z^T and the n x n blocks
    C_ab = U_a^T U_b of U (one Gram of its halves),
        U^T G Z^T   = (U_X^T E) Z^T + C_VV H
        U^T J G Z^T = C_XV H - (U_V^T E) Z^T
    and xi = J G Z^T S^-1 + G Z^T J S^-1 - U Q splits by halves into
        xi_X = E (Z^T J S^-1) + U_V (H S^-1) - U_X Q
        xi_V = E (-Z^T S^-1)  + U_V (H J S^-1 - Q),
    two combines over E and U: no G Z^T and no 2N-row Gram."""
    N = ud.shape[0] // 2
    n = ud.shape[1]
    ux, uv = ud[:N], ud[N:]
    C = _tall.gram([(ux, False), (uv, False)])
    cxv, cvv = C[:n, n:], C[n:, n:]
    zt = z.T
    H = z @ zt
    u_gzt = g.ux_e @ zt + cvv @ H
    u_jgzt = cxv @ H - g.uv_e @ zt
    q = u_jgzt @ s_inv + u_gzt @ js_inv
    out = torch.empty((2 * N, n), dtype=torch.float64, device="cuda")
    _tall.combine([(g.e, zt @ js_inv, False), (uv, H @ s_inv, False), (ux, -q, False)], out=out[:N])
    _tall.combine([(g.e, -(zt @ s_inv), False), (uv, H @ js_inv - q, False)], out=out[N:])
    return out


def _retraction_coeffs(G, n):
    P, M, X = G[:n, :n], G[:n, n:], G[n:, n:]
    utw = M - 0.5 * P @ M
    wtw = X - M.T @ M + 0.25 * M.T @ P @ M
    bta = np.block([[utw, -P], [wtw, -utw.T]])
    cap = np.eye(2 * n) - 0.5 * bta
    y = np.linalg.solve(cap, np.concatenate([P, utw.T], axis=0))
    y1, y2 = y[:n], y[n:]
    return np.eye(n) - 0.5 * M @ y1 - y2, y1


def retraction(u, xi):
    """Low-rank Cayley retraction cay(W U^T - U W^T) U (reduction.py:156-167):
    u + [w, -u] cap^{-1} [u, w]^T u with w = xi - U (U^T xi)/2, assembled from
    the Gram of [U, xi] as U (I - M Y1/2 - Y2) + xi Y1.  xi may be a lazy
    Scaled(x, c): the Gram of [U, x] is rescaled on the host."""
    ud, was_np = _tall_in(u)
    xd, c, _ = _scaled_in(xi)
    n = ud.shape[1]
    G = _tall.gram([(ud, False), (xd, False)])
    G[:n, n:] *= c
    G[n:, :n] *= c
    G[n:, n:] *= c * c
    cu, cx = _retraction_coeffs(G, n)
    return _tall_out(_tall.combine([(ud, cu, False), (xd, c * cx, False)]), was_np)


def tangent_velocity(u, xi, r_xi, x_eval):
    """Pull a velocity at r_xi = retraction(u, xi) back to u (reduction.py:170-182).
    Only the 7 needed block products of [U, xi, r, x_eval] are formed; xi and
    x_eval may be lazy Scaled operands."""
    ud, was_np = _tall_in(u)
    xd, cxi, _ = _scaled_in(xi)
    rd, _ = _tall_in(r_xi)
    ed, cev, _ = _scaled_in(x_eval)
    n = ud.shape[1]
    G = _tall.gram_tasks([(ud, False), (xd, False), (rd, False), (ed, False)],
                         [(0, 0), (0, 1), (0, 2), (0, 3), (1, 3), (2, 1), (2, 3)])
    b = _tall.split(G, [n, n, n, n])
    P, M, R, E = b[0][0], cxi * b[0][1], b[0][2], cev * b[0][3]
    F, rxi, rxe = cxi * cev * b[1][3], cxi * b[2][1], cev * b[2][3]
    eye = np.eye(n)
    t_u = 0.5 * M @ E + F - 0.5 * M.T @ E         # t = 2 x_eval - xi E + u t_u
    K = np.linalg.inv(R + eye)                     # ups = t (U^T r + I)^-1
    c_e, c_x, c_u = 2.0 * K, -E @ K, t_u @ K       # ups = x_eval c_e + xi c_x + u c_u
    rt_ups = rxe @ c_e + rxi @ c_x + R.T @ c_u
    ut_ups = E @ c_e + M @ c_x + P @ c_u
    lead = np.linalg.solve(R.T + eye, rt_ups + ut_ups)
    out = _tall.combine([(ed, cev * c_e, False), (xd, cxi * c_x, False),
                         (ud, c_u - lead - ut_ups.T, False)])
    return _tall_out(out, was_np)


def scaled(a, c):
    """c * a: a lazy Scaled for device operands (folded into the next Gram and
    combine), a plain product for host arrays."""
    if isinstance(a, np.ndarray):
        return c * a
    return Scaled(a, c)


def fixed_point(map_fn, z0, tol=1e-9, max_iter=100):
    """z <- map_fn(z) until the relative update is below tol (reduction.py:185-202)."""
    z = z0
    trace = []
    for it in range(1, max_iter + 1):
        z_new = map_fn(z)
        num = float(np.linalg.norm(z_new - z))
        den = max(float(np.linalg.norm(z_new)), np.finfo(float).tiny)
        trace.append(num / den)
        z = z_new
        if num <= tol * den:
            return z, it, trace
    raise StepFailureError(
        f"implicit coefficient stage did not converge in {max_iter} iterations "
        f"(last relative update {trace[-1]:.3e})", iterations=max_iter, residual_trace=trace)


class DeviceFixedPoint:
    """fixed_point (reduction.py:185-202) for the stage map k -> J g(z + dt/2 k)
    kept on the device: g(z) = D(z) + C z with D the stage's F-evaluation
    kernels (launched by `launch_d(zeval, gout, skip, status)`) and C = U_V^T U_V.
    Each iteration is D + picrom_fp_update (J, the relative-update test and the
    residual trace on the device); iterations are queued in chunks and the host
    syncs once per chunk -- the first chunk is the previous step's iteration
    count + 1, launches queued past convergence are skipped by the device flag.
    Same iteration count, convergence test and StepFailureError as fixed_point."""

    def __init__(self, n, launch_d, c_host, stream_owner=None):
        self.n = n
        self.launch_d = launch_d
        self.c = torch.from_numpy(np.ascontiguousarray(c_host, dtype=np.float64)).to("cuda")
        self.bufs = None
        self.hint = stream_owner

    def _alloc(self, p, max_iter):
        n = self.n
        f64 = dict(dtype=torch.float64, device="cuda")
        self.bufs = dict(p=p, zd=torch.empty((n, p), **f64), k=torch.empty((n, p), **f64),
                         ze=torch.empty((n, p), **f64), gout=torch.empty((n, p), **f64),
                         state=torch.zeros(4, dtype=torch.int64, device="cuda"),
                         trace=torch.zeros(max(max_iter, 1), **f64),
                         z_h=torch.empty((n, p), dtype=torch.float64, pin_memory=True),
                         flags_h=torch.empty(4, dtype=torch.int64, pin_memory=True))

    def __call__(self, z, dt, tol, max_iter):
        from . import _device as dev
        from . import _lib
        z = np.ascontiguousarray(z, dtype=np.float64)
        n, p = z.shape
        if self.bufs is None or self.bufs["p"] != p or self.bufs["trace"].numel() < max_iter:
            self._alloc(p, max_iter)
        b = self.bufs
        b["z_h"].numpy()[...] = z
        b["zd"].copy_(b["z_h"], non_blocking=True)
        b["k"].zero_()
        b["ze"].copy_(b["zd"])
        b["state"].zero_()
        st = b["state"][2:]                    # F-evaluation status word (min-reduced)
        st.fill_(-1)
        s = dev.stream_handle()
        hint = self.hint[0] if self.hint else None
        chunk = (hint + 1) if hint else 6
        it = 0
        done = False
        while it < max_iter:
            m = min(chunk, max_iter - it)
            for q in range(m):
                self.launch_d(b["ze"], b["gout"], b["state"], st)
                _lib.call("picrom_fp_update", b["gout"].data_ptr(), self.c.data_ptr(),
                          b["zd"].data_ptr(), b["k"].data_ptr(), b["ze"].data_ptr(), n, p,
                          0.5 * dt, float(tol), it + q, b["state"].data_ptr(),
                          b["trace"].data_ptr(), s)
            it += m
            b["flags_h"].copy_(b["state"], non_blocking=True)
            torch.cuda.current_stream().synchronize()
            flags = b["flags_h"].numpy()
            if int(flags[2]) != -1:
                from .driver import _raise_eval
                _raise_eval(b["flags_h"][2:], p)
            if int(flags[0]):
                done = True
                break
            chunk = 4
        if not done:
            trace = b["trace"][:max_iter].cpu().numpy().tolist()
            raise StepFailureError(
                f"implicit coefficient stage did not converge in {max_iter} iterations "
                f"(last relative update {trace[-1]:.3e})", iterations=max_iter,
                residual_trace=trace)
        iters = int(flags[1])
        if self.hint is not None:
            self.hint[0] = iters
        return b["k"].cpu().numpy(), iters, b["trace"][:iters].cpu().numpy().tolist()


@dataclass
class PRKResult:
    u: object
    z: np.ndarray
    u_mid: object
    z_mid: np.ndarray
    fp_iterations: int
    s_cond: float


class _NullTimers:
    def phase(self, name):
        return nullcontext()


def prk2_step(u, z, dt, sub, grad_sub, g_sub0, coeff_stage, fp_tol=1e-9, fp_max_iter=100,
              timers=None):
    """One partitioned RK2 step of (U, Z) (reduction.py:220-259), same seams:
    grad_sub(u, z_sub) and coeff_stage(u_mid) -> g(z) are injected callables."""
    timers = timers or _NullTimers()
    with timers.phase("rom_basis"):
        s0 = SMatrix(z[:, sub])
        xi1 = basis_velocity(u, z[:, sub], g_sub0, s=s0)
        half_step = scaled(xi1, 0.5 * dt)
        u_mid = retraction(u, half_step)
        g = coeff_stage(u_mid)
    with timers.phase("rom_coeff"):
        dfp = getattr(g, "device_fixed_point", None)
        if dfp is not None:
            k, iterations, _ = dfp(z, dt, fp_tol, fp_max_iter)
        else:
            k, iterations, _ = fixed_point(lambda kk: jmul(g(z + 0.5 * dt * kk)),
                                           np.zeros_like(z), fp_tol, fp_max_iter)
        z_new = z + dt * k
        z_mid = z + 0.5 * dt * k
    with timers.phase("rom_basis"):
        g_mid = grad_sub(u_mid, z_mid[:, sub])
        xi_mid = basis_velocity(u_mid, z_mid[:, sub], g_mid)
        xi2 = tangent_velocity(u, half_step, u_mid, xi_mid)
        u_new = retraction(u, scaled(xi2, dt))
    return PRKResult(u=u_new, z=z_new, u_mid=u_mid, z_mid=z_mid, fp_iterations=iterations,
                     s_cond=s0.cond)
