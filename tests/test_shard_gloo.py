"""Multi-rank path on CPU: world_size 2 over gloo.

Each rank refines its slab (shard.slab_mesh), computes its one-sided rows
with the CPU oracle operator, and runs the real interface exchange
(shard.exchange_partials over torch.distributed).  The summed rows must
equal the single-domain operator on the whole box at every node, and the
duplicated interface rows must be bitwise identical on both ranks.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _ufun(X):
    return np.sin(3.0 * X[:, 0] + 2.0 * X[:, 1] + 5.0 * X[:, 2]) + X[:, 2]


def _kfun(X):
    return 2.0 + np.sin(2 * np.pi * X[:, 0]) * np.cos(np.pi * X[:, 1]) + X[:, 2]


def _worker(rank, world, port, level, variant, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle.assemble import CpuOperator
    from paper_1709_06793_b200.coefficients import sample_nodal
    from paper_1709_06793_b200.mesh import RefinedGrid
    from paper_1709_06793_b200.shard import InterfaceMap, exchange_partials, slab_mesh
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}",
                            rank=rank, world_size=world)
    try:
        nx = 2
        grid = RefinedGrid(slab_mesh(rank, world, nx=nx, ny=nx), level)
        kf = sample_nodal(_kfun, grid)
        op = CpuOperator(grid, variant, kf)
        u = _ufun(grid.node_coords)
        out = torch.from_numpy(op.apply(u))
        imap = InterfaceMap(grid, rank, world, 1.0 / nx)
        exchange_partials(out, imap, dist)
        owned = imap.owned_mask(grid.n_nodes)
        # dot product with the owner mask: every node counted once
        local = torch.tensor([float(np.dot(out.numpy()[owned], u[owned]))], dtype=torch.float64)
        dist.all_reduce(local)
        q.put((rank, grid.node_coords, out.numpy(), local.item(),
               {k: v for k, v in imap.neighbours.items()}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("variant,world", [("scaling", 2), ("nodal", 2), ("scaling", 3)])
def test_two_rank_slabs_equal_single_domain(variant, world):
    """world 3: the middle rank exchanges with both neighbours."""
    from oracle.assemble import CpuOperator
    from paper_1709_06793_b200.coefficients import sample_nodal
    from paper_1709_06793_b200.mesh import RefinedGrid, kuhn_blocks
    level = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, level, variant, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0

    gmesh = kuhn_blocks(np.linspace(0, 1, 3), np.linspace(0, 1, 3),
                        0.5 * np.arange(world + 1, dtype=float))
    grid = RefinedGrid(gmesh, level)
    op = CpuOperator(grid, variant, sample_nodal(_kfun, grid))
    u = _ufun(grid.node_coords)
    ref = op.apply(u)
    index = {tuple(x): i for i, x in enumerate(grid.node_coords)}
    scale = np.abs(ref).max()
    for rank, X, out, _, _ in res:
        gids = np.array([index[tuple(x)] for x in X])
        assert np.abs(out - ref[gids]).max() <= 1e-13 * scale
    # interface rows bitwise identical on both sides of every interface
    for a, b in zip(res[:-1], res[1:]):
        (ra, Xa, oa, da, na), (rb, Xb, ob, db, nb) = a, b
        assert np.array_equal(oa[na[rb]], ob[nb[ra]])
        assert np.array_equal(Xa[na[rb]], Xb[nb[ra]])
    # owner-masked dot == single-domain dot, the same on every rank
    dots = [r[3] for r in res]
    assert all(d == dots[0] for d in dots)
    assert abs(dots[0] - float(ref @ u)) <= 1e-12 * abs(float(ref @ u)) + 1e-12


def _cg_worker(rank, world, port, level, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle.assemble import CpuOperator
    from paper_1709_06793_b200.coefficients import sample_nodal
    from paper_1709_06793_b200.mesh import RefinedGrid
    from paper_1709_06793_b200.shard import (InterfaceMap, ShardedOperator, sharded_cg,
                                             slab_mesh)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}",
                            rank=rank, world_size=world)
    try:
        nx = 2
        grid = RefinedGrid(slab_mesh(rank, world, nx=nx, ny=nx), level)
        op = CpuOperator(grid, "scaling", sample_nodal(_kfun, grid))
        imap = InterfaceMap(grid, rank, world, 1.0 / nx)
        sop = ShardedOperator(op, imap, dist, grid.dirichlet_mask)
        # right-hand side = A u* with u* smooth and zero on the boundary
        X = grid.node_coords
        ustar = np.sin(np.pi * X[:, 0]) * np.sin(np.pi * X[:, 1]) * np.sin(np.pi * X[:, 2])
        ustar[grid.dirichlet_mask] = 0.0
        f = sop.apply(torch.from_numpy(ustar))
        x, its, res = sharded_cg(sop, f, tol=1e-10)
        r = sop.residual(x, f)
        q.put((rank, X, x.numpy(), its, res, float(torch.sqrt(sop.dot(r, r)).item())))
    finally:
        dist.destroy_process_group()


def test_two_rank_cg_matches_single_domain():
    from oracle.assemble import CpuOperator
    from paper_1709_06793_b200.coefficients import sample_nodal
    from paper_1709_06793_b200.mesh import RefinedGrid, kuhn_blocks
    world, level = 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cg_worker, args=(r, world, port, level, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-domain CG, same algorithm, global dots
    gmesh = kuhn_blocks(np.linspace(0, 1, 3), np.linspace(0, 1, 3), np.array([0.0, 0.5, 1.0]))
    grid = RefinedGrid(gmesh, level)
    op = CpuOperator(grid, "scaling", sample_nodal(_kfun, grid))
    X = grid.node_coords
    free = (~grid.dirichlet_mask).astype(float)
    ustar = np.sin(np.pi * X[:, 0]) * np.sin(np.pi * X[:, 1]) * np.sin(np.pi * X[:, 2])
    ustar[grid.dirichlet_mask] = 0.0
    f = op.apply(ustar)
    x = np.zeros_like(f)
    r = f * free
    p = r.copy()
    rs = r @ r
    b0 = np.sqrt(rs)
    for its in range(1, 10000):
        Ap = op.apply(p) * free
        a = rs / (p @ Ap)
        x += a * p
        r -= a * Ap
        rs_new = r @ r
        if np.sqrt(rs_new) <= 1e-10 * b0:
            break
        p = r + rs_new / rs * p
        rs = rs_new
    index = {tuple(c): i for i, c in enumerate(X)}
    for rank, Xr, xr, its_r, res_r, true_res in res:
        assert abs(its_r - its) <= 1, (its_r, its)
        gids = np.array([index[tuple(c)] for c in Xr])
        assert np.abs(xr - x[gids]).max() <= 1e-8 * np.abs(x).max()
        assert np.abs(xr - ustar[gids]).max() <= 1e-7     # solves A x = A u*
        assert true_res <= 1e-9 * b0
    assert res[0][3] == res[1][3]                         # ranks agree on the count


def test_sharded_operator_rejects_unknown_transport():
    from paper_1709_06793_b200.mesh import RefinedGrid
    from paper_1709_06793_b200.shard import InterfaceMap, ShardedOperator, slab_mesh
    grid = RefinedGrid(slab_mesh(0, 1, nx=2, ny=2), 2)
    imap = InterfaceMap(grid, 0, 1, 0.5)
    assert imap.neighbours == {}
    with pytest.raises(ValueError, match="transport"):
        ShardedOperator(object(), imap, None, grid.dirichlet_mask, transport="mpi")
