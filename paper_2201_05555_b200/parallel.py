"""Multi-GPU execution, one process per GPU (torchrun).

* Full-order PIC: instance sharding.  The parameter instances are
  independent, so each GPU advances its own slice of columns with no
  data-path collective; `torch.distributed` only does the plumbing (the
  barrier around the timed region, the max over ranks of device times,
  gathering the small per-instance records).
* Reduced model: particle-row sharding.  Each rank owns rows [lo, hi) of
  both halves of U (the same particles in U_X and U_V, so J stays a local
  row swap); Z and every n x n / 2n x 2n matrix are replicated.  Every
  N-row product becomes a local partial plus an all-reduce -- the charge
  rho (Nx x p, background added by rank 0 only) before the replicated
  Poisson solve, the projections U^T E (n x p) of the gather, and every
  tall Gram of the manifold maps (installed as a reduction hook in _tall);
  the combines are row-local.  That is one all-reduce per F-evaluation
  half and per manifold Gram, all small (<= (4n)^2 or Nx p doubles):
  latency-bound, NCCL over NVLink.
"""

from __future__ import annotations

import contextlib

import numpy as np
import torch
import torch.distributed as tdist


def shard_slice(p, rank, world):
    """Contiguous columns [lo, hi) of p instances owned by `rank` (balanced, in order)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(p, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_columns(a, rank, world):
    """Column block of an (N, p) array (or (p,) vector) owned by `rank`."""
    lo, hi = shard_slice(a.shape[-1], rank, world)
    return a[..., lo:hi]


def max_over_ranks(value, device=None):
    """Max of a scalar over all ranks (device-timed figures)."""
    if not (tdist.is_available() and tdist.is_initialized()) or tdist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    return float(t.item())


def gather_columns(local, p_total):
    """Reassemble per-rank (..., p_local) host arrays into (..., p_total) in rank order."""
    if not (tdist.is_available() and tdist.is_initialized()) or tdist.get_world_size() == 1:
        return np.asarray(local)
    parts = [None] * tdist.get_world_size()
    tdist.all_gather_object(parts, np.asarray(local))
    out = np.concatenate(parts, axis=-1)
    if out.shape[-1] != p_total:
        raise ValueError("gathered column count mismatch")
    return out


def run_sharded_full_order(system_factory, x0, v0, dt, t_final, record=None, device=None):
    """run_full_order on this rank's instance slice; returns (record, (lo, hi)).

    system_factory(lo, hi) builds the rank-local system (one mesh per run, or
    the matching per-instance rows)."""
    from .fullorder import ParticleEnsemble, run_full_order
    rank = tdist.get_rank() if tdist.is_initialized() else 0
    world = tdist.get_world_size() if tdist.is_initialized() else 1
    lo, hi = shard_slice(x0.shape[1], rank, world)
    rec = run_full_order(system_factory(lo, hi),
                         ParticleEnsemble(x0[:, lo:hi], v0[:, lo:hi], 0.0), dt, t_final, record)
    return rec, (lo, hi)


# ------------------------------------------------------------ row sharding

def _dist():
    return tdist.is_available() and tdist.is_initialized() and tdist.get_world_size() > 1


def allreduce_sum(a):
    """Sum of an array over all ranks, same kind/device back (identity when
    not distributed).  CUDA tensors go through NCCL in place; the gloo
    backend (CPU tests) reduces host copies."""
    if not _dist():
        return a
    if isinstance(a, np.ndarray):
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).clone()
        tdist.all_reduce(t, op=tdist.ReduceOp.SUM)
        return t.numpy()
    if a.is_cuda and tdist.get_backend() != "nccl":
        h = a.cpu()
        tdist.all_reduce(h, op=tdist.ReduceOp.SUM)
        a.copy_(h)
        return a
    tdist.all_reduce(a, op=tdist.ReduceOp.SUM)
    return a


class RowSharding:
    """Particle rows [lo, hi) of N owned by this rank (balanced, in order)."""

    def __init__(self, num_particles, rank=None, world=None):
        self.N = int(num_particles)
        self.rank = tdist.get_rank() if rank is None and _dist() else (rank or 0)
        self.world = tdist.get_world_size() if world is None and _dist() else (world or 1)
        self.lo, self.hi = shard_slice(self.N, self.rank, self.world)

    @property
    def rows(self):
        return self.hi - self.lo

    def local_u(self, u):
        """[U_X[lo:hi]; U_V[lo:hi]] (2 rows x n) of a global basis U (2N x n)."""
        N = self.N
        if isinstance(u, torch.Tensor):
            return torch.cat([u[self.lo:self.hi], u[N + self.lo:N + self.hi]], dim=0).contiguous()
        u = np.asarray(u)
        return np.ascontiguousarray(np.concatenate([u[self.lo:self.hi], u[N + self.lo:N + self.hi]]))

    def gather_u(self, u_local):
        """Global U (2N x n, host) from every rank's local rows (rank order)."""
        h = u_local.cpu().numpy() if isinstance(u_local, torch.Tensor) else np.asarray(u_local)
        if not _dist():
            return h
        parts = [None] * self.world
        tdist.all_gather_object(parts, h)
        half = [p[:p.shape[0] // 2] for p in parts], [p[p.shape[0] // 2:] for p in parts]
        return np.concatenate(half[0] + half[1])

    def background_owner(self):
        """The rank that adds the uniform background bg*h to the charge."""
        return self.rank == 0


_ACTIVE = None


def active():
    """The RowSharding of the enclosing row_sharded() block, or None."""
    return _ACTIVE


@contextlib.contextmanager
def row_sharded(sharding):
    """Run the reduced model's N-row products as local partials + all-reduces:
    _tall's Grams are summed over ranks, driver's F-evaluation reduces rho and
    the projections (see the module docstring)."""
    global _ACTIVE
    from . import _tall
    prev, prev_hook = _ACTIVE, _tall.reduce_hook
    _ACTIVE = sharding
    _tall.reduce_hook = allreduce_sum if sharding is not None and sharding.world > 1 else None
    try:
        yield sharding
    finally:
        _ACTIVE, _tall.reduce_hook = prev, prev_hook
