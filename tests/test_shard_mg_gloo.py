"""The global surface level schedule of the sharded smoother on CPU (gloo,
world 2 and 3): every slab row gets exactly the level of the same node in
the single-domain schedule, so the lockstep sweep updates rows in an order
the single-domain lexicographic sweep admits."""
import os
import socket
import sys

import numpy as np
import pytest


def _levels_worker(rank, world, port, nx, lvl, q):
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    from paper_1709_06793_b200 import RefinedGrid
    from paper_1709_06793_b200.device import GridTables, SurfaceTables
    from paper_1709_06793_b200.shard import InterfaceMap, slab_mesh
    from paper_1709_06793_b200.shard_mg import global_levels
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        g = RefinedGrid(slab_mesh(rank, world, nx, nx), lvl)
        st = SurfaceTables(g, GridTables(g, tile_rows=12, mirror_cols=32))
        imap = InterfaceMap(g, rank, world, 1.0 / nx)
        rows = np.asarray(st.rows)
        iface = {nb: np.searchsorted(rows, ids) for nb, ids in imap.neighbours.items()}
        level = global_levels(st.gs_dag(), iface, dist)
        X = np.round(g.node_coords[rows], 9)
        q.put((rank, {tuple(x): int(v) for x, v in zip(X, level)}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_global_levels_equal_single_domain(world):
    import multiprocessing as mp
    from paper_1709_06793_b200 import mesh as M
    from paper_1709_06793_b200.device import GridTables, SurfaceTables
    nx, lvl = 2, 3
    h = 1.0 / nx
    full = M.RefinedGrid(M.kuhn_blocks(np.linspace(0, 1, nx + 1), np.linspace(0, 1, nx + 1),
                                       np.linspace(0, world * h, world + 1)), lvl)
    st = SurfaceTables(full, GridTables(full, tile_rows=12, mirror_cols=32))
    ref_level = SurfaceTables.levels_of(st.gs_dag())
    X = np.round(full.node_coords[np.asarray(st.rows)], 9)
    ref = {tuple(x): int(v) for x, v in zip(X, ref_level)}
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_levels_worker, args=(r, world, port, nx, lvl, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    seen = set()
    for rank, lv in out:
        for key, v in lv.items():
            assert ref[key] == v, (rank, key, v, ref[key])
            seen.add(key)
    assert seen == set(ref)          # every free surface row is on some rank
