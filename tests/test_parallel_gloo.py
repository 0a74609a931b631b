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
