"""Multi-GPU execution of the full-order path: instance sharding.

The parameter instances of a batched PIC run are independent, so N GPUs
each advance their own slice of columns with no data-path collective: one
process per GPU (torchrun), `torch.distributed` only for plumbing (the
barrier before/after the timed region, the max-over-ranks of device
times, and gathering the small per-instance records at the end).

Particle sharding inside one instance would need an all-reduce of rho
(Nx x p fp64) before each solve; it is listed as next work in DESIGN.md §7.
"""

from __future__ import annotations

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
