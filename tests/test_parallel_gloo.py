"""Instance sharding host logic across 2 ranks (gloo, CPU): slices cover the
columns exactly once, per-rank results reassemble in order, and the timing
reduction is a max over ranks -- the logic bench.py and
parallel.run_sharded_full_order use under torchrun on GPUs."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2201_05555_b200 import parallel


def test_shard_slices_partition():
    for p in (1, 7, 32, 64, 128):
        for world in (1, 2, 3, 8):
            got = [parallel.shard_slice(p, r, world) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == p
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            sizes = [hi - lo for lo, hi in got]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as tdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = 7
        rng = np.random.default_rng(0)
        full = rng.standard_normal((5, p))
        local = parallel.shard_columns(full, rank, world) * 2.0      # per-rank "work"
        out = parallel.gather_columns(local, p)
        tmax = parallel.max_over_ranks(1.5 + rank)
        tdist.barrier()
        q.put((rank, np.allclose(out, 2.0 * full), tmax))
    finally:
        tdist.destroy_process_group()


def test_two_rank_gloo_shard_and_gather():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=120)
    res = sorted(q.get(timeout=5) for _ in range(world))
    assert all(pr.exitcode == 0 for pr in procs)
    assert all(ok for _, ok, _ in res)
    assert all(t == pytest.approx(2.5) for _, _, t in res)


def _rom_worker(rank, world, port, q):
    """Particle-row sharding of the reduced model, host composition: each rank
    deposits/projects its own rows (oracle arithmetic), the partials are
    all-reduced by parallel.allreduce_sum -- charge (background added by rank
    0 only), the projection U^T F, a tall Gram -- and equal the unsharded
    results."""
    import torch.distributed as tdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import fe_bspline as fe
        from oracle import manifold as mf
        from oracle import rom_loop as orl
        rng = np.random.default_rng(4)
        N, p, nb, nx, L = 3001, 5, 4, 16, 4 * np.pi
        x0 = rng.uniform(0, L, (N, p))
        v0 = rng.standard_normal((N, p))
        u, z = mf.csvd_basis(x0, v0, nb)
        sh = parallel.RowSharding(N)
        ul = sh.local_u(u)
        # charge: local particles, charge weight of the full N, background on rank 0
        mesh, charge = fe.Mesh(L, nx, 2), fe.Charge(N, L)
        xl = ul[:sh.rows] @ z
        rho_l = fe.deposit_charge(fe.eval_basis(mesh, xl), charge)
        if not sh.background_owner():
            rho_l -= charge.background * mesh.h
        rho = parallel.allreduce_sum(rho_l)
        want = fe.deposit_charge(fe.eval_basis(mesh, u[:N] @ z), charge)
        ok_rho = np.max(np.abs(rho - want)) <= 1e-12 * np.max(np.abs(want))
        # projection U^T F(U z) from local rows
        osys = orl.ParamSystem(np.full(p, L), nx, 2, N)
        g_full, phi, _ = orl.exact_gradients(osys, u, z)
        gl = np.concatenate([g_full[sh.lo:sh.hi], g_full[N + sh.lo:N + sh.hi]])
        proj = parallel.allreduce_sum(ul.T @ gl)
        ok_proj = np.max(np.abs(proj - u.T @ g_full)) <= 1e-12 * np.max(np.abs(u.T @ g_full))
        gram = parallel.allreduce_sum(ul.T @ ul)
        ok_gram = np.max(np.abs(gram - u.T @ u)) <= 1e-13
        ok_gather = np.array_equal(sh.gather_u(ul), u)
        sizes = [None] * world
        tdist.all_gather_object(sizes, (sh.lo, sh.hi))
        ok_cover = sizes[0][0] == 0 and sizes[-1][1] == N and sizes[0][1] == sizes[1][0]
        q.put((rank, bool(ok_rho and ok_proj and ok_gram and ok_gather and ok_cover)))
    finally:
        tdist.destroy_process_group()


def test_two_rank_gloo_rom_row_sharding_composition():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rom_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=180)
    res = sorted(q.get(timeout=5) for _ in range(world))
    assert all(pr.exitcode == 0 for pr in procs)
    assert all(ok for _, ok in res), res
