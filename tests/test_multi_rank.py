"""Multi-rank coverage without several GPUs.

CPU (gloo, world_size 2, 127.0.0.1): the torch.distributed plumbing bench.py
and the sharded contexts use -- id broadcast, max-over-ranks timing, rank-order
sums -- and the tile partition every rank computes independently.

GPU (one device): EMULATED ranks (fdl_create_sharded with a NULL NCCL id) each
build and evaluate only their own upper-triangle tiles; the rank partials
summed in rank order must equal the single-context values.  This exercises
everything in the sharded path except the NCCL transport: tile ranges that
split strips, per-rank MS-BFS source ranges, work items, the per-row
reductions filtered to the local tiles, stress partials.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1711_01228_b200 import fdl


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1711_01228_b200 import dist as fdist

    payload = bytes(range(128)) if rank == 0 else None
    got = fdist.broadcast_bytes(payload, 128, 0)
    mx = fdist.max_over_ranks(1.5 + rank)
    sm = fdist.sum_in_rank_order(0.1 * (rank + 1))
    t0, t1 = fdl.shard_tiles(n, world, rank)
    ranges = [None] * world
    dist.all_gather_object(ranges, (t0, t1))
    q.put((rank, got == bytes(range(128)), mx, sm, ranges))
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [1000, 200000])
def test_gloo_world2_plumbing(n):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    nb = -(-n // fdl.FDL_TILE)
    total = nb * (nb + 1) // 2
    for rank, ok, mx, sm, ranges in res:
        assert ok
        assert mx == 2.5
        assert sm == pytest.approx(0.1 + 0.2, abs=0)
        # every rank derived the same partition; it covers the triangle once
        assert ranges[0][0] == 0 and ranges[-1][1] == total
        assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))


# -------------------------------------------------------------- GPU emulation
@pytest.mark.gpu
@pytest.mark.parametrize("name,world", [("C1", 2), ("C2", 3), ("C3", 2), ("C3", 8)])
def test_emulated_ranks_sum_to_single(name, world):
    from workloads import configs

    cfg = configs.CONFIGS[name]
    g = configs.graph_for(name)
    k = cfg.k_for(g.n)
    X = configs.positions_for(name, g.n, 2)
    p = fdl.make_params(dim=cfg.dim, k=k, omega=cfg.omega, tol=cfg.tol)
    single = fdl.Layout.from_graph(g, params=p, init_pos=X)
    R, A, f = single.eval_forces()
    Rs = np.zeros_like(R)
    As = np.zeros_like(A)
    fs = 0.0
    covered = 0
    for r in range(world):
        L = fdl.Layout.from_graph(g, params=p, init_pos=X, nccl_id=None, rank=r, world=world)
        info = L.get_info()
        covered += info.tile1 - info.tile0
        Rr, fr = L.eval_partial(0, X)
        Ar, _ = L.eval_partial(1, X)
        Rs += Rr
        As += Ar
        fs += fr
        with pytest.raises(fdl.FdlError):
            L.step()
        L.close()
    nb = -(-g.n // fdl.FDL_TILE)
    assert covered == nb * (nb + 1) // 2
    # same pair terms, different fp64 grouping of the partial sums
    assert np.linalg.norm(Rs - R) <= 1e-12 * np.linalg.norm(R)
    assert np.linalg.norm(As - A) <= 1e-12 * np.linalg.norm(A)
    assert abs(fs - f) <= 1e-12 * f
