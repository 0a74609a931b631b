"""Row-sharded reduced model on the GPU, functional check:
two ranks (gloo all-reduces through host copies; both ranks on cuda:0 -- a
correctness run of the sharded code path, not a timing) advance their halves
of the particle rows of U; Z, the energies and the fixed-point counts must
equal the single-process run, the gathered U likewise."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

KW = dict(basis_dim=4, subsample=6, window=3, deim_dim=8, deim_period=3, deim_update=2,
          dt=0.05, t_final=0.3, hyper_reduction=False, energy_stride=2, decomp_stride=10**9,
          snapshot_stride=6)


def _problem():
    rng = np.random.default_rng(21)
    N, p, nx = 4001, 6, 32
    ks = rng.uniform(0.4, 0.6, p)
    lengths = 2 * np.pi / ks
    x0 = np.stack([rng.uniform(0, L, N) for L in lengths], axis=1)
    v0 = rng.standard_normal((N, p))
    params = np.stack([ks, rng.uniform(0.01, 0.1, p)], axis=1)
    return N, nx, lengths, x0, v0, params


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as tdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2201_05555_b200 import driver, parallel
        N, nx, lengths, x0, v0, params = _problem()
        gsys = driver.ParametricVlasovSystem(lengths, nx, 2, N)
        sh = parallel.RowSharding(N)
        rec = driver.run_reduced(gsys, params, x0, v0, sharding=sh, **KW)
        u_loc, z = rec.bases[-1]
        u = sh.gather_u(u_loc)
        q.put((rank, z, rec.electric_energy, rec.hamiltonian, rec.fp_iterations,
               rec.ortho_residuals, u))
    finally:
        tdist.destroy_process_group()


def test_two_rank_row_sharded_reduced_run(lib_built):
    from paper_2201_05555_b200 import driver
    N, nx, lengths, x0, v0, params = _problem()
    gsys = driver.ParametricVlasovSystem(lengths, nx, 2, N)
    ref = driver.run_reduced(gsys, params, x0, v0, **KW)
    u_ref, z_ref = ref.bases[-1]
    u_ref = u_ref.cpu().numpy()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    assert all(pr.exitcode == 0 for pr in procs)
    for rank, z, ee, ham, fp, orth, u in res:
        np.testing.assert_array_equal(fp, ref.fp_iterations)
        assert np.linalg.norm(z - z_ref) <= 1e-11 * np.linalg.norm(z_ref)
        assert np.max(np.abs(ee - ref.electric_energy) / np.abs(ref.electric_energy)) <= 1e-10
        assert np.max(np.abs(ham - ref.hamiltonian) / np.abs(ref.hamiltonian)) <= 1e-10
        assert np.linalg.norm(u - u_ref) <= 1e-11 * np.linalg.norm(u_ref)
        assert np.max(np.abs(orth - ref.ortho_residuals)) <= 1e-13
