"""ORACLE (test infrastructure only): periodic cardinal B-spline FE, degree 1..3.

Restates /root/reference/pkg/src/picrom/fem.py, generalised to degree d:

* basis: lambda_i(x) = N_d(x/h - i + sigma), N_d the cardinal B-spline on
  [0, d+1], sigma = (d+1)//2.  A particle in cell c = floor(x/h) with fraction
  f touches the d+1 nodes (c - d//2 + m) mod Nx, m = 0..d, with weight
  N_d(f + d - m).  For d = 1 this is exactly fem.py's (i0, i0+1) pair with
  weights (1-f, f) (fem.py:119-136,179-182); for d = 3 the basis is centred on
  the nodes; for d = 2 the basis function lambda_i is centred on the cell
  midpoint (i + 1/2) h (documented choice).
* ``locate`` is fem.py:108-116 verbatim in arithmetic (IEEE division by the
  double h, floor, exact fraction, Python-style non-negative modulo) so the
  integer cell index is the parity anchor for all degrees.
* deposit = one flat bincount per table entry in row-major order
  (fem.py:151-166) plus background*h (fem.py:203-215).
* stiffness L_ij = int lambda_i' lambda_j' dx assembled exactly from rational
  B-spline products (circulant, half-bandwidth d); the solve adds 11^T/length
  and Cholesky-factorises once (fem.py:218-244).
* energy / field / Hamiltonian formulas are unchanged (fem.py:247-268).

At degree 1 every array is bit-identical to the reference (pinned by
tests/test_oracle_golden.py against tests/golden/fem_p1.npz).
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction
from functools import lru_cache

import numpy as np
from scipy.linalg import cho_factor, cho_solve


class OracleError(ValueError):
    """Mirror of picrom.errors.EvaluationError / ConfigurationError for the oracle."""

    def __init__(self, message, index=None):
        super().__init__(message)
        self.index = index


# --------------------------------------------------------------------------
# exact B-spline algebra
# --------------------------------------------------------------------------

@lru_cache(maxsize=None)
def spline_pieces(d):
    """Polynomial pieces of N_d: pieces[k] = ascending coefficients in u of N_d(k+u).

    Cox-de Boor recursion N_q(t) = t/q N_{q-1}(t) + (q+1-t)/q N_{q-1}(t-1),
    done in exact rational arithmetic.
    """
    pcs = [(Fraction(1),)]
    for q in range(1, d + 1):
        out = []
        for k in range(q + 1):
            acc = [Fraction(0)] * (q + 1)
            if k < q:
                for i, c in enumerate(pcs[k]):
                    acc[i] += c * Fraction(k, q)
                    acc[i + 1] += c * Fraction(1, q)
            if k >= 1:
                for i, c in enumerate(pcs[k - 1]):
                    acc[i] += c * Fraction(q + 1 - k, q)
                    acc[i + 1] -= c * Fraction(1, q)
            out.append(tuple(acc))
        pcs = out
    return tuple(pcs)


def _poly_mul(a, b):
    out = [Fraction(0)] * (len(a) + len(b) - 1)
    for i, x in enumerate(a):
        for j, y in enumerate(b):
            out[i + j] += x * y
    return out


def _poly_der(a):
    return [a[i] * i for i in range(1, len(a))] or [Fraction(0)]


def _poly_int01(a):
    return sum(c / (i + 1) for i, c in enumerate(a))


@lru_cache(maxsize=None)
def stiffness_stencil(d):
    """a_k = int N_d'(t) N_d'(t+k) dt, k = 0..d (exact rationals); L_{i,i+-k} = a_k / h."""
    pcs = spline_pieces(d)
    der = [_poly_der(list(p)) for p in pcs]
    out = []
    for k in range(d + 1):
        total = Fraction(0)
        for j in range(d + 1):          # t in [j, j+1]; t + k in piece j + k
            if j + k <= d:
                total += _poly_int01(_poly_mul(der[j], der[j + k]))
        out.append(total)
    return tuple(out)


def first_node_offset(d):
    """Node of table entry m is (cell + first_node_offset(d) + m) mod Nx."""
    return -(d // 2)


# --------------------------------------------------------------------------
# mesh / charge (fem.py:40-98)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class Mesh:
    length: float
    num_cells: int
    degree: int = 1

    def __post_init__(self):
        if not (self.length > 0.0 and np.isfinite(self.length)):
            raise OracleError(f"mesh length must be positive, got {self.length}")
        if self.num_cells < 2:
            raise OracleError(f"need at least 2 cells, got {self.num_cells}")
        if self.degree not in (1, 2, 3):
            raise OracleError(f"spline degree must be 1, 2 or 3, got {self.degree}")
        if self.degree > 1 and self.num_cells < 2 * self.degree + 1:
            raise OracleError("need num_cells >= 2*degree+1 for degree > 1")

    @property
    def h(self):
        return self.length / self.num_cells


@dataclass(frozen=True)
class Charge:
    num_particles: int
    length: float
    charge: float = -1.0
    mass: float = 1.0
    background: float = 1.0

    @property
    def weight(self):
        return -self.background * self.length / (self.charge * self.num_particles)

    @property
    def charge_weight(self):
        return self.charge * self.weight

    @property
    def particle_mass(self):
        return self.mass * self.weight


# --------------------------------------------------------------------------
# locate + basis tables (fem.py:101-200)
# --------------------------------------------------------------------------

def check_finite(x):
    bad = ~np.isfinite(x)
    if bad.any():
        first = tuple(int(i) for i in np.argwhere(bad)[0])
        raise OracleError(f"non-finite particle position at index {first}", index=first)


def locate(mesh, x):
    """(cell mod Nx as int64, fraction) -- fem.py:108-116 arithmetic."""
    x = np.asarray(x, dtype=float)
    check_finite(x)
    s = x / mesh.h
    cell = np.floor(s)
    frac = s - cell
    return cell.astype(np.int64) % mesh.num_cells, frac


def value_weights(d, f):
    """[N_d(f + d - m) for m = 0..d]; d = 1 is fem.py:182 verbatim."""
    if d == 1:
        return [1.0 - f, f]
    g = 1.0 - f
    if d == 2:
        return [0.5 * g * g, 0.75 - (f - 0.5) * (f - 0.5), 0.5 * f * f]
    f2 = f * f
    return [g * g * g / 6.0,
            (3.0 * f2 * f - 6.0 * f2 + 4.0) / 6.0,
            (-3.0 * f2 * f + 3.0 * f2 + 3.0 * f + 1.0) / 6.0,
            f2 * f / 6.0]


def grad_weights(d, f, h):
    """[d/dx lambda at entry m]; d = 1 is fem.py:188-190 verbatim (-1/h, +1/h)."""
    g = 1.0 / h
    if d == 1:
        shape = np.shape(f)
        return [np.full(shape, -g), np.full(shape, g)]
    if d == 2:
        return [(f - 1.0) * g, (1.0 - 2.0 * f) * g, f * g]
    e = 1.0 - f
    return [(-0.5 * e * e) * g,
            (1.5 * f * f - 2.0 * f) * g,
            (-1.5 * f * f + f + 0.5) * g,
            (0.5 * f * f) * g]


@dataclass(frozen=True)
class SplineTable:
    """Row table: entry m of row r sits at node nodes(m)[r] with weight w[m][r]."""

    mesh: Mesh
    kind: str
    i0: np.ndarray           # cell index mod Nx (the reference's i0)
    w: tuple                 # d+1 arrays

    def nodes(self, m):
        return (self.i0 + first_node_offset(self.mesh.degree) + m) % self.mesh.num_cells

    @property
    def i1(self):
        return self.nodes(1)

    @property
    def w0(self):
        return self.w[0]

    @property
    def w1(self):
        return self.w[1]

    def matvec(self, phi):
        phi = np.asarray(phi, dtype=float)
        out = None
        for m, wm in enumerate(self.w):
            idx = self.nodes(m)
            vals = phi[idx] if phi.ndim == 1 else np.take_along_axis(phi, idx, axis=0)
            term = wm * vals
            out = term if out is None else out + term
        return out

    def rmatvec(self, y):
        y = np.asarray(y, dtype=float)
        nx = self.mesh.num_cells
        if self.i0.ndim == 1:
            out = None
            for m, wm in enumerate(self.w):
                b = np.bincount(self.nodes(m), weights=wm * y, minlength=nx)
                out = b if out is None else out + b
            return out
        n, p = self.i0.shape
        col = np.broadcast_to(np.arange(p, dtype=np.int64) * nx, (n, p))
        out = None
        for m, wm in enumerate(self.w):
            flat = (self.nodes(m) + col).ravel()
            b = np.bincount(flat, weights=(wm * y).ravel(), minlength=nx * p)
            if out is None:
                out = b
            else:
                out += b
        return out.reshape(p, nx).T

    def toarray(self):
        if self.i0.ndim != 1:
            raise OracleError("dense form only for 1D position arrays")
        out = np.zeros((self.i0.size, self.mesh.num_cells))
        rows = np.arange(self.i0.size)
        for m, wm in enumerate(self.w):
            np.add.at(out, (rows, self.nodes(m)), wm)
        return out


def eval_basis(mesh, x):
    i0, f = locate(mesh, x)
    return SplineTable(mesh, "value", i0, tuple(value_weights(mesh.degree, f)))


def eval_basis_grad(mesh, x):
    i0, f = locate(mesh, x)
    return SplineTable(mesh, "gradient", i0, tuple(grad_weights(mesh.degree, f, mesh.h)))


def eval_basis_pair(mesh, x):
    i0, f = locate(mesh, x)
    return (SplineTable(mesh, "value", i0, tuple(value_weights(mesh.degree, f))),
            SplineTable(mesh, "gradient", i0, tuple(grad_weights(mesh.degree, f, mesh.h))))


def deposit_charge(basis, charge):
    """fem.py:203-215: basis^T (qw 1) + background * h."""
    if basis.kind != "value":
        raise OracleError("deposition needs a value table")
    rho = basis.rmatvec(np.full(basis.i0.shape, charge.charge_weight))
    rho += charge.background * basis.mesh.h
    return rho


def stiffness_matrix(mesh):
    nx, h, d = mesh.num_cells, mesh.h, mesh.degree
    a = stiffness_stencil(d)
    L = np.zeros((nx, nx))
    idx = np.arange(nx)
    if d == 1:     # fem.py:231-235 assignment order (matters only for nx = 2)
        L[idx, idx] = 2.0 / h
        L[idx, (idx + 1) % nx] = -1.0 / h
        L[idx, (idx - 1) % nx] = -1.0 / h
        return L
    L[idx, idx] = float(a[0]) / h
    for k in range(1, d + 1):
        L[idx, (idx + k) % nx] += float(a[k]) / h
        L[idx, (idx - k) % nx] += float(a[k]) / h
    return L


class Poisson:
    """fem.py:218-244: dense Cholesky of L + 11^T/length, zero-mean gauge."""

    def __init__(self, mesh):
        self.mesh = mesh
        self.stiffness = stiffness_matrix(mesh)
        nx = mesh.num_cells
        self._cho = cho_factor(self.stiffness + np.ones((nx, nx)) / mesh.length)

    def solve(self, rho):
        rho = np.asarray(rho, dtype=float)
        b = rho - rho.mean(axis=0, keepdims=True)
        phi = cho_solve(self._cho, b)
        return phi - phi.mean(axis=0, keepdims=True)


def electric_energy(poisson, phi, charge):
    phi = np.asarray(phi, dtype=float)
    lphi = poisson.stiffness @ phi
    return 0.5 / charge.particle_mass * np.einsum("i...,i...->...", phi, lphi)


def field_at_particles(grad, phi, charge):
    return -(charge.charge_weight / charge.particle_mass) * grad.matvec(phi)


def hamiltonian(x, v, poisson, charge):
    v = np.asarray(v, dtype=float)
    kinetic = 0.5 * np.einsum("i...,i...->...", v, v)
    rho = deposit_charge(eval_basis(poisson.mesh, x), charge)
    phi = poisson.solve(rho)
    return kinetic + electric_energy(poisson, phi, charge)
