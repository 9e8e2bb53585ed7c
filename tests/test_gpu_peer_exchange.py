"""Peer-memory interface exchange (shard.PeerExchange) on one GPU.

Several ranks are emulated in one process on one device (the buffers a
neighbour would reach through CUDA IPC are passed directly).  Every rank's
push phase runs before any pull, so no kernel ever waits on another launch
of the same GPU (B200_PROFILING.md); the pulls find the counters already
set.  The completed interface rows must be bitwise the rank-ordered sums of
the NCCL path, and the double-buffered receive buffers must stay correct
over several applies.
"""
import numpy as np
import pytest

from paper_1709_06793_b200 import Operator, RefinedGrid, sample_nodal
from paper_1709_06793_b200.shard import InterfaceMap, PeerExchange, slab_mesh

pytestmark = pytest.mark.gpu


def _kfun(X):
    return 2.0 + np.sin(2 * np.pi * X[:, 0]) * np.cos(np.pi * X[:, 1]) + X[:, 2]


@pytest.mark.parametrize("world", [2, 3])
def test_peer_exchange_emulated_ranks(cuda, world):
    torch = cuda
    nx, level = 2, 4
    ranks = []
    for r in range(world):
        grid = RefinedGrid(slab_mesh(r, world, nx=nx, ny=nx), level)
        op = Operator(grid, "scaling", sample_nodal(_kfun, grid))
        imap = InterfaceMap(grid, r, world, 1.0 / nx)
        ranks.append((grid, op, imap, PeerExchange(op, imap)))
    peers = {r: ex for r, (_, _, _, ex) in enumerate(ranks)}
    for _, _, _, ex in ranks:
        ex.connect_local(peers)
    for it in range(3):                       # epochs 1..3: both parities
        us = [torch.as_tensor(np.sin((it + 1) * X[:, 0] + 2 * X[:, 1] - X[:, 2]) + X[:, 2],
                              device="cuda") for X in (g.node_coords for g, _, _, _ in ranks)]
        # reference: one-sided applies + rank-ordered sums on the host
        plain = [op.apply_device(u).cpu().numpy() for (_, op, _, _), u in zip(ranks, us)]
        want = [p.copy() for p in plain]
        for r, (_, _, imap, _) in enumerate(ranks):
            for nb, ids in imap.neighbours.items():
                theirs = plain[nb][ranks[nb][2].neighbours[r]]
                mine = plain[r][ids]
                want[r][ids] = (theirs + mine) if nb < r else (mine + theirs)
        outs = [ex.start(u) for (_, _, _, ex), u in zip(ranks, us)]
        for (_, _, _, ex), o in zip(ranks, outs):
            ex.finish(o)
        torch.cuda.synchronize()
        for r, ((_, _, _, ex), o) in enumerate(zip(ranks, outs)):
            ex.check()
            assert np.array_equal(o.cpu().numpy(), want[r]), (it, r)
    for _, _, _, ex in ranks:
        ex.close()


def _ipc_worker(rank, world, port, q):
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    from paper_1709_06793_b200 import Operator, RefinedGrid, sample_nodal
    from paper_1709_06793_b200.shard import InterfaceMap, PeerExchange, slab_mesh
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}",
                            rank=rank, world_size=world)
    try:
        nx = 2
        grid = RefinedGrid(slab_mesh(rank, world, nx=nx, ny=nx), 3)
        op = Operator(grid, "scaling", sample_nodal(_kfun, grid))
        imap = InterfaceMap(grid, rank, world, 1.0 / nx)
        ex = PeerExchange(op, imap)
        ex.connect(dist)                          # CUDA IPC handles over gloo
        X = grid.node_coords
        u = torch.as_tensor(np.sin(3 * X[:, 0] + 2 * X[:, 1] + 5 * X[:, 2]) + X[:, 2],
                            device="cuda")
        out = ex.start(u)
        torch.cuda.synchronize()
        dist.barrier()                            # every push has landed: no pull waits
        ex.finish(out)
        torch.cuda.synchronize()
        ex.check()
        q.put((rank, X, out.cpu().numpy(), {k: v for k, v in imap.neighbours.items()}))
        dist.barrier()
        ex.close()
    finally:
        dist.destroy_process_group()


def test_peer_exchange_ipc_two_processes(cuda):
    """The CUDA IPC plumbing (handles exchanged over torch.distributed) with
    two processes on this one GPU, sequenced by a host barrier."""
    import socket

    import torch.multiprocessing as mp
    from oracle.assemble import CpuOperator
    from paper_1709_06793_b200.mesh import kuhn_blocks
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    gmesh = kuhn_blocks(np.linspace(0, 1, 3), np.linspace(0, 1, 3), np.array([0.0, 0.5, 1.0]))
    grid = RefinedGrid(gmesh, 3)
    X = grid.node_coords
    ref = CpuOperator(grid, "scaling", sample_nodal(_kfun, grid)).apply(
        np.sin(3 * X[:, 0] + 2 * X[:, 1] + 5 * X[:, 2]) + X[:, 2])
    index = {tuple(x): i for i, x in enumerate(X)}
    for rank, Xr, out, _ in res:
        gids = np.array([index[tuple(x)] for x in Xr])
        assert np.abs(out - ref[gids]).max() <= 1e-13 * np.abs(ref).max()
    (_, X0, o0, n0), (_, X1, o1, n1) = res
    assert np.array_equal(o0[n0[1]], o1[n1[0]])


def test_nccl_pack_and_rank_order_add_kernels(cuda):
    """The NCCL transport's native pieces (hhg_gather, hhg_interface_add)
    reproduce index_select and the rank-ordered sums of the torch path
    bitwise (NCCL itself needs two GPUs; the kernels do not)."""
    torch = cuda
    from paper_1709_06793_b200._lib import check, lib
    gen = torch.Generator(device="cuda").manual_seed(7)
    out = torch.rand(10_000, dtype=torch.float64, device="cuda", generator=gen)
    ids = torch.randperm(10_000, device="cuda", generator=gen)[:3_001].to(torch.int64)
    theirs = torch.rand(3_001, dtype=torch.float64, device="cuda", generator=gen) * 1e3
    st = torch.cuda.current_stream().cuda_stream
    mine = torch.empty(3_001, dtype=torch.float64, device="cuda")
    check(lib.hhg_gather(3_001, ids.data_ptr(), out.data_ptr(), mine.data_ptr(), st), "gather")
    assert torch.equal(mine, out.index_select(0, ids))
    for first in (0, 1):
        got = out.clone()
        check(lib.hhg_interface_add(3_001, ids.data_ptr(), mine.data_ptr(), theirs.data_ptr(),
                                    first, got.data_ptr(), st), "interface_add")
        want = out.clone()
        want.index_copy_(0, ids, (theirs + mine) if first else (mine + theirs))
        assert torch.equal(got, want)
