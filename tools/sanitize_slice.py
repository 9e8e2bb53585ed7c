"""Small slices of every device path for compute-sanitizer (one tool per
gpurun call, B200_PROFILING.md):

    compute-sanitizer --tool memcheck  python tools/sanitize_slice.py
    compute-sanitizer --tool racecheck python tools/sanitize_slice.py
    compute-sanitizer --tool synccheck python tools/sanitize_slice.py

Config 1 (reference tetrahedron, level 4) and the config-3 mesh at level 4:
apply (bitwise mirror, FMA mirror, generic fast, nodal, const, stored),
residual, the per-element ABI, Gauss-Seidel smoothing (surface levels +
volume wavefronts), a V-cycle and CG, transfers, and the peer-memory
interface exchange with two ranks emulated in one process (every push
before any pull, so no kernel waits on another launch).  Prints one line
per slice; the sanitizer's own summary is the verdict."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1709_06793_b200 import Operator, RefinedGrid, sample_nodal  # noqa: E402
from paper_1709_06793_b200 import mesh as M  # noqa: E402
from paper_1709_06793_b200.multigrid import GridHierarchy, pcg, solve  # noqa: E402
from paper_1709_06793_b200.shard import InterfaceMap, PeerExchange, slab_mesh  # noqa: E402
from tests.cases import case_mesh, k_c1, k_c3  # noqa: E402


def slice_ops(tag, grid, kf):
    rng = np.random.default_rng(1)
    u = torch.as_tensor(rng.uniform(-1, 1, grid.n_nodes), device="cuda")
    f = torch.as_tensor(rng.uniform(-1, 1, grid.n_nodes), device="cuda")
    for name, op in (("scaling", Operator(grid, "scaling", kf)),
                     ("scaling-fast", Operator(grid, "scaling", kf, fast=True)),
                     ("nodal", Operator(grid, "nodal", kf)),
                     ("const", Operator(grid, "const", 2.0)),
                     ("matrix-free", Operator(grid, "scaling", kf, surface_mode="matrix-free"))):
        op.apply(u)
        op.residual(u, f)
        if name in ("scaling", "nodal"):
            op.smooth(u.clone(), f, sweeps=1)
            op.apply(u.cpu().numpy())
        print(f"{tag} {name}: apply / residual ok", flush=True)
    st = Operator(grid, "scaling", kf).store_stencils()
    st.apply(u)
    torch.cuda.synchronize()
    print(f"{tag} stored: ok", flush=True)


def slice_solvers():
    hier = GridHierarchy(M.unit_cube_6(), 4, "scaling", k_c3(), lmin=2)
    g = hier.grids[4]
    f = np.random.default_rng(2).normal(size=g.n_nodes)
    f[g.dirichlet_mask] = 0.0
    solve(hier, f, stop="iters:2", pre=2, post=2)
    pcg(hier, f, stop="iters:2", pre=1, post=1)
    hier.coarse_solve(np.random.default_rng(3).normal(size=hier.grids[2].n_nodes))
    torch.cuda.synchronize()
    print("solvers: V-cycle / PCG / coarse CG ok", flush=True)


def slice_peer():
    world, nx = 2, 2
    ranks = []
    kfun = lambda X: 2.0 + np.sin(2 * np.pi * X[:, 0]) + X[:, 2]  # noqa: E731
    for r in range(world):
        grid = RefinedGrid(slab_mesh(r, world, nx=nx, ny=nx), 3)
        op = Operator(grid, "scaling", sample_nodal(kfun, grid))
        ranks.append((grid, PeerExchange(op, InterfaceMap(grid, r, world, 1.0 / nx))))
    peers = {r: ex for r, (_, ex) in enumerate(ranks)}
    for _, ex in ranks:
        ex.connect_local(peers)
    for it in range(2):
        outs = [ex.start(torch.as_tensor(np.cos((it + 1) * g.node_coords[:, 0]), device="cuda"))
                for g, ex in ranks]
        for (_, ex), o in zip(ranks, outs):
            ex.finish(o)
        torch.cuda.synchronize()
        for _, ex in ranks:
            ex.check()
    for _, ex in ranks:
        ex.close()
    print("peer exchange (2 emulated ranks): ok", flush=True)


if __name__ == "__main__":
    g1 = RefinedGrid(case_mesh("c1"), 4)
    slice_ops("c1", g1, sample_nodal(k_c1(), g1))
    g3 = RefinedGrid(case_mesh("c3"), 4)
    slice_ops("c3-l4", g3, sample_nodal(k_c3(), g3))
    slice_solvers()
    slice_peer()
    print("all slices done", flush=True)
