"""Periodic B-spline finite elements on the GPU -- drop-in for picrom.fem.

Same names, signatures, argument meaning and error behaviour as
/root/reference/pkg/src/picrom/fem.py (the module's ``__all__``, fem.py:24-37);
``build_mesh``/``PeriodicMesh`` take an extra ``degree`` (1 = the reference's
P1 hats, 2 = quadratic, 3 = cubic B-splines; see DESIGN.md for the basis).
Every pointwise/grid operation runs in the sm_100a library
(include/picrom_b200.h) -- there is no CPU path.  Inputs may be numpy arrays
or torch tensors in the reference layouts ((N,), (N, p), (Nx,), (Nx, p));
results come back as the same kind.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as dev
from . import _lib
from .errors import ConfigurationError
from .splines import stiffness_stencil

__all__ = [
    "PeriodicMesh",
    "ChargeConfig",
    "BasisTable",
    "build_mesh",
    "eval_basis",
    "eval_basis_grad",
    "eval_basis_pair",
    "deposit_charge",
    "PoissonOperator",
    "electric_energy",
    "field_at_particles",
    "hamiltonian",
]


@dataclass(frozen=True)
class PeriodicMesh:
    """Uniform periodic grid on [0, length) with num_cells nodes (fem.py:40-59)."""

    length: float
    num_cells: int
    degree: int = 1

    def __post_init__(self):
        if not (self.length > 0.0 and np.isfinite(self.length)):
            raise ConfigurationError(f"mesh length must be positive, got {self.length}")
        if self.num_cells < 2:
            raise ConfigurationError(f"need at least 2 cells, got {self.num_cells}")
        if self.degree not in (1, 2, 3):
            raise ConfigurationError(f"spline degree must be 1, 2 or 3, got {self.degree}")
        if self.degree > 1 and self.num_cells < 2 * self.degree + 1:
            raise ConfigurationError("need num_cells >= 2*degree+1 for degree > 1")

    @property
    def h(self):
        return self.length / self.num_cells

    @property
    def nodes(self):
        return self.h * np.arange(self.num_cells)


def build_mesh(length, num_cells, degree=1):
    return PeriodicMesh(float(length), int(num_cells), int(degree))


@dataclass(frozen=True)
class ChargeConfig:
    """Macro-particle species data (fem.py:66-98): q N weight + background L = 0."""

    num_particles: int
    length: float
    charge: float = -1.0
    mass: float = 1.0
    background: float = 1.0

    def __post_init__(self):
        if self.num_particles < 1:
            raise ConfigurationError("need at least one particle")
        if self.charge == 0.0 or self.mass <= 0.0:
            raise ConfigurationError("charge must be nonzero and mass positive")

    @property
    def weight(self):
        return -self.background * self.length / (self.charge * self.num_particles)

    @property
    def charge_weight(self):
        return self.charge * self.weight

    @property
    def particle_mass(self):
        return self.mass * self.weight


# neutral charge used for kernels that need only the mesh part of the table
def _mesh_only_inst(mesh, p):
    return dev.inst_rows(mesh, ChargeConfig(1, mesh.length), p)


@dataclass
class BasisTable:
    """Basis data at particle positions (fem.py:119-176), evaluated lazily on the GPU.

    The device keeps only the positions; ``i0`` / ``w0`` / ``w1`` /
    ``weights`` are materialised on demand.  Entry m of a row sits at node
    (i0 - degree//2 + m) mod Nx.  ``matvec``/``rmatvec`` are the gather and the
    deposit kernels.
    """

    mesh: PeriodicMesh
    kind: str
    xd: torch.Tensor = field(repr=False)       # (p, N) device positions
    meta: dev.Meta = field(repr=False)
    _cache: dict = field(default_factory=dict, repr=False)

    @property
    def degree(self):
        return self.mesh.degree

    def _table(self):
        if "i0" not in self._cache:
            p, n = self.xd.shape
            d = self.degree
            i0 = torch.empty((p, n), dtype=torch.int64, device="cuda")
            w = torch.empty((d + 1, p, n), dtype=torch.float64, device="cuda")
            st = dev.new_status()
            kind = 0 if self.kind == "value" else 1
            _lib.call("picrom_basis_table", self.xd.data_ptr(), n, p, n,
                      _mesh_only_inst(self.mesh, p).data_ptr(), self.mesh.num_cells, d, kind,
                      i0.data_ptr(), w.data_ptr(), n, st.data_ptr(), dev.stream_handle())
            dev.raise_if_bad(st, p, self.meta.ndim)
            self._cache["i0"] = dev.from_device(i0, self.meta)
            self._cache["w"] = tuple(dev.from_device(w[m], self.meta) for m in range(d + 1))
        return self._cache["i0"], self._cache["w"]

    @property
    def i0(self):
        return self._table()[0]

    @property
    def weights(self):
        return self._table()[1]

    @property
    def w0(self):
        return self.weights[0]

    @property
    def w1(self):
        return self.weights[1]

    def nodes(self, m):
        return (self.i0 - self.degree // 2 + m) % self.mesh.num_cells

    @property
    def i1(self):
        return self.nodes(1)

    def _phi_device(self, phi):
        ph, meta = dev.to_device(phi)
        p = self.xd.shape[0]
        if ph.shape[1] != self.mesh.num_cells:
            raise ConfigurationError("potential length must equal num_cells")
        if ph.shape[0] == 1 and p > 1:
            ph = ph.expand(p, -1).contiguous()
        if ph.shape[0] != p:
            raise ConfigurationError("potential columns must match the position columns")
        return ph

    def matvec(self, phi):
        """sum_i phi_i lambda_i (value table) or its x-derivative (gradient table)."""
        kind = _lib_kind(self.kind, raw=True)
        return _gather(self.mesh, self.xd, self.meta, self._phi_device(phi), kind,
                       _mesh_only_inst(self.mesh, self.xd.shape[0]))

    def rmatvec(self, y):
        """Accumulate particle values y onto the nodes (the deposit kernel)."""
        yd, _ = dev.to_device(y)
        p, n = self.xd.shape
        if tuple(yd.shape) != (p, n):
            raise ConfigurationError("y must have the positions' shape")
        out = torch.empty((p, self.mesh.num_cells), dtype=torch.float64, device="cuda")
        st = dev.new_status()
        _lib.call("picrom_rmatvec", self.xd.data_ptr(), yd.data_ptr(), n, p, n,
                  _mesh_only_inst(self.mesh, p).data_ptr(), self.mesh.num_cells, self.degree,
                  0 if self.kind == "value" else 1, out.data_ptr(),
                  dev.workspace(n, p, self.mesh.num_cells, self.degree).data_ptr(),
                  st.data_ptr(), dev.stream_handle())
        dev.raise_if_bad(st, p, self.meta.ndim)
        return dev.from_device(out, self.meta)

    def toarray(self):
        """Dense (N, Nx) matrix; single-column tables only (test helper)."""
        if self.meta.ndim != 1:
            raise ConfigurationError("dense form only supported for 1D position arrays")
        i0 = np.asarray(_host(self.i0))
        out = np.zeros((i0.size, self.mesh.num_cells))
        rows = np.arange(i0.size)
        for m, wm in enumerate(self.weights):
            np.add.at(out, (rows, (i0 - self.degree // 2 + m) % self.mesh.num_cells), _host(wm))
        return out


def _host(a):
    return a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)


def _lib_kind(kind, raw=False):
    if kind == "value":
        return 0
    return 3 if raw else 1


def _gather(mesh, xd, meta, phd, kind, inst):
    p, n = xd.shape
    out = torch.empty((p, n), dtype=torch.float64, device="cuda")
    st = dev.new_status()
    _lib.call("picrom_gather", xd.data_ptr(), n, p, n, inst.data_ptr(), mesh.num_cells,
              mesh.degree, phd.data_ptr(), kind, out.data_ptr(), n, st.data_ptr(),
              dev.stream_handle())
    dev.raise_if_bad(st, p, meta.ndim)
    return dev.from_device(out, meta)


def _make_table(mesh, x, kind):
    xd, meta = dev.to_device(x)
    st = dev.new_status()
    p, n = xd.shape
    # fem._check_finite (fem.py:101-105): raise with the first non-finite index
    _lib.call("picrom_locate", xd.data_ptr(), n, p, n, _mesh_only_inst(mesh, p).data_ptr(),
              mesh.num_cells, None, None, n, st.data_ptr(), dev.stream_handle())
    dev.raise_if_bad(st, p, meta.ndim)
    return BasisTable(mesh, kind, xd, meta)


def eval_basis(mesh, x):
    """Basis values at positions x: rows sum to one (fem.py:179-182)."""
    return _make_table(mesh, x, "value")


def eval_basis_grad(mesh, x):
    """Basis derivatives at positions x (fem.py:185-190)."""
    return _make_table(mesh, x, "gradient")


def eval_basis_pair(mesh, x):
    """Value and gradient tables from a single lookup (fem.py:193-200)."""
    value = _make_table(mesh, x, "value")
    return value, BasisTable(mesh, "gradient", value.xd, value.meta)


def deposit_charge(basis, charge):
    """Nodal charge density basis^T (q w 1) + background*h (fem.py:203-215)."""
    if basis.kind != "value":
        raise ConfigurationError("deposition needs a value table, not a gradient table")
    mesh = basis.mesh
    p, n = basis.xd.shape
    rho = torch.empty((p, mesh.num_cells), dtype=torch.float64, device="cuda")
    st = dev.new_status()
    _lib.call("picrom_deposit", basis.xd.data_ptr(), n, p, n,
              dev.inst_rows(mesh, charge, p).data_ptr(), mesh.num_cells, mesh.degree,
              rho.data_ptr(), dev.workspace(n, p, mesh.num_cells, mesh.degree).data_ptr(),
              st.data_ptr(), dev.stream_handle())
    dev.raise_if_bad(st, p, basis.meta.ndim)
    return dev.from_device(rho, basis.meta)


class PoissonOperator:
    """Periodic stiffness matrix with the zero-mean solve (fem.py:218-244).

    ``stiffness`` is the dense Nx x Nx matrix (2/h, -1/h for P1, exactly as the
    reference builds it); ``solve`` runs the batched circulant solve kernel.
    """

    def __init__(self, mesh):
        self.mesh = mesh
        nx, h, d = mesh.num_cells, mesh.h, mesh.degree
        L = np.zeros((nx, nx))
        idx = np.arange(nx)
        if d == 1:
            L[idx, idx] = 2.0 / h
            L[idx, (idx + 1) % nx] = -1.0 / h
            L[idx, (idx - 1) % nx] = -1.0 / h
        else:
            a = stiffness_stencil(d)
            L[idx, idx] = float(a[0]) / h
            for k in range(1, d + 1):
                L[idx, (idx + k) % nx] += float(a[k]) / h
                L[idx, (idx - k) % nx] += float(a[k]) / h
        self.stiffness = L

    @property
    def constants(self):
        return dev.mesh_constants(self.mesh.num_cells, self.mesh.degree)

    def solve(self, rho):
        """Zero-mean potential solving stiffness @ phi = rho - mean(rho)."""
        rd, meta = dev.to_device(rho)
        p = rd.shape[0]
        phi = torch.empty_like(rd)
        c = self.constants
        _lib.call("picrom_poisson", rd.data_ptr(), p, self.mesh.num_cells, self.mesh.degree,
                  _mesh_only_inst(self.mesh, p).data_ptr(), c.khat.data_ptr(),
                  c.stencil.data_ptr(), phi.data_ptr(), None, dev.stream_handle())
        return dev.from_device(phi, meta)


def electric_energy(poisson, phi, charge):
    """Field energy (1/(2 m_p)) phi^T L phi per column (fem.py:247-251)."""
    pd, meta = dev.to_device(phi)
    p = pd.shape[0]
    out = torch.empty(p, dtype=torch.float64, device="cuda")
    c = poisson.constants
    mesh = poisson.mesh
    _lib.call("picrom_field_energy", pd.data_ptr(), p, mesh.num_cells, mesh.degree,
              dev.inst_rows(mesh, charge, p).data_ptr(), c.stencil.data_ptr(), out.data_ptr(),
              dev.stream_handle())
    return dev.per_instance(out, meta)


def field_at_particles(grad, phi, charge):
    """-(1/m_p)(q w) d/dx sum_i phi_i lambda_i at the particles (fem.py:254-256)."""
    p = grad.xd.shape[0]
    return _gather(grad.mesh, grad.xd, grad.meta, grad._phi_device(phi), 1,
                   dev.inst_rows(grad.mesh, charge, p))


def hamiltonian(x, v, poisson, charge):
    """0.5 v^T v + field energy of the self-consistent potential (fem.py:259-268)."""
    from .fullorder import _kinetic_device
    mesh = poisson.mesh
    xd, meta = dev.to_device(x)
    vd, _ = dev.to_device(v)
    p, n = xd.shape
    rho = torch.empty((p, mesh.num_cells), dtype=torch.float64, device="cuda")
    phi = torch.empty_like(rho)
    ee = torch.empty(p, dtype=torch.float64, device="cuda")
    st = dev.new_status()
    inst = dev.inst_rows(mesh, charge, p)
    c = poisson.constants
    s = dev.stream_handle()
    _lib.call("picrom_deposit", xd.data_ptr(), n, p, n, inst.data_ptr(), mesh.num_cells,
              mesh.degree, rho.data_ptr(), dev.workspace(n, p, mesh.num_cells, mesh.degree).data_ptr(),
              st.data_ptr(), s)
    dev.raise_if_bad(st, p, meta.ndim)
    _lib.call("picrom_poisson", rho.data_ptr(), p, mesh.num_cells, mesh.degree, inst.data_ptr(),
              c.khat.data_ptr(), c.stencil.data_ptr(), phi.data_ptr(), ee.data_ptr(), s)
    kin = _kinetic_device(vd)
    return dev.per_instance(kin + ee, meta)
