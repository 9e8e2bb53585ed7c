"""Sharded multigrid: the reference's V-cycle and solve loop
(multigrid.py:197-270) on macro-element slabs, one rank per GPU.

Every rank owns a slab of the macro mesh (`shard.slab_mesh`) with its own
HHG numbering; a slab's numbering is the global numbering restricted to it
(vertex ids of `kuhn_blocks` grow with z, entities are sorted vertex tuples,
node ids rank barycentrics of the higher-id vertices), so every order
relation the reference's smoother uses between two nodes of one slab is
the same locally and globally.  Pieces:

* **smoother** (operators.py:517-536): forward Gauss-Seidel in global order
  = the surface rows in a level schedule of the *global* dependency graph,
  then every element's interior.  A row depends on its lower-id neighbours,
  all of which share an element with it, hence live on every rank that
  holds the row; only rows on an interface plane are held by two ranks.
  The levels are the longest-path levels of the union of the slabs'
  graphs: computed locally, the two copies of each interface row raise
  each other's level (exchange, max) until nothing changes.  A sweep walks
  the levels in lockstep: rows of one rank update directly; an interface
  row's two partial sums (each rank's own incidences, acc and diagonal) are
  exchanged, added in rank order, and both ranks finish it with the same
  numbers.  The interiors then sweep locally (ghost refresh, hyperplane
  wavefronts).
* **residual**: the sharded apply (interface rows completed).
* **restriction** (multigrid.py:135-138): each rank restricts its residual
  with shared fine nodes counted once (owner = lower rank), the coarse
  interface rows are completed like apply rows; **prolongation** is local
  (interface fine nodes are interpolated identically on both sides).
* **coarse solve** (multigrid.py:147-167): the reference's plain CG to
  ``coarse_tol`` on the sharded coarse system (`shard.sharded_cg`).

The sweep order is exactly the single-domain one, so a sharded solve
reproduces the single-domain cycle count and residual history to rounding
(different summation order of interface rows, dots and the coarse solve):
tests/test_gpu_shard_mg.py.
"""
from __future__ import annotations

import time

import numpy as np

from ._lib import check, lib
from .coefficients import sample_nodal
from .device import SurfaceTables, require_cuda
from .mesh import RefinedGrid
from .multigrid import DeviceTransfer, SolveReport, _parse_stop
from .operators import Operator
from .shard import InterfaceMap, ShardedOperator, sharded_cg, slab_mesh

__all__ = ["ShardedHierarchy", "sharded_vcycle", "sharded_solve", "global_levels"]


def _swap(dist, nbr, send):
    """Send `send` (1-D tensor) to rank nbr and receive its equally long
    counterpart, on send's device; gloo exchanges go through host memory,
    NCCL ones through device memory."""
    import torch
    stage = torch.device("cpu") if dist.get_backend() == "gloo" else torch.device("cuda")
    s = send.to(stage)
    r = torch.empty_like(s)
    reqs = dist.batch_isend_irecv([dist.P2POp(dist.isend, s, nbr),
                                   dist.P2POp(dist.irecv, r, nbr)])
    for q in reqs:
        q.wait()
    return r.to(send.device)


def _scalar(dist, v):
    import torch
    dev = "cpu" if dist.get_backend() == "gloo" else "cuda"
    return torch.tensor([v], dtype=torch.int64, device=dev)


def global_levels(dag, iface, dist):
    """Longest-path levels of the union of all ranks' surface dependency
    graphs, for this rank's rows: local levels (hhg_host_gs_levels_seeded)
    with the shared interface rows' levels raised to the maximum of both
    copies, repeated until no rank changes (every round carries a chain
    across one more interface crossing).  ``iface``: neighbour rank -> this
    rank's row indices of the shared rows in the interface map's common
    order."""
    import torch
    seed = np.zeros(len(dag[0]) - 1, dtype=np.int64)
    while True:
        level = SurfaceTables.levels_of(dag, seed)
        new = seed.copy()
        for nb, r in iface.items():
            theirs = _swap(dist, nb, torch.as_tensor(level[r])).numpy()
            new[r] = np.maximum(new[r], np.maximum(level[r], theirs))
        changed = _scalar(dist, int(np.any(new != seed)))
        dist.all_reduce(changed)
        if int(changed.item()) == 0:
            return level
        seed = new


class _SurfaceSchedule:
    """Level schedule of one rank's surface rows in the global order, and
    the per-level row lists (local rows; interface rows per neighbour in
    the interface map's common order)."""

    def __init__(self, sop: ShardedOperator):
        torch = require_cuda()
        op, imap, dist = sop.op, sop.imap, sop.dist
        self.op, self.sop, self.dist, self.rank = op, sop, dist, imap.rank
        st = op._device()["surf"].st
        rows = np.asarray(st.rows)
        dag = st.gs_dag()
        iface = {}
        for nb, ids in imap.neighbours.items():
            r = np.searchsorted(rows, ids)
            if len(ids) and (r.max() >= len(rows) or np.any(rows[r] != ids)):
                raise ValueError("interface node is not a free surface row")
            iface[nb] = r
        level = global_levels(dag, iface, dist)
        nlev = _scalar(dist, int(level.max()) + 1 if len(level) else 0)
        dist.all_reduce(nlev, op=dist.ReduceOp.MAX)
        self.nlev = int(nlev.item())
        shared = np.zeros(len(rows), dtype=bool)
        for r in iface.values():
            shared[r] = True
        dev = torch.device("cuda")
        order = np.argsort(level, kind="stable")
        ptr = np.searchsorted(level[order], np.arange(self.nlev + 1))
        self.local, self.shared = [], []
        for L in range(self.nlev):
            at = order[ptr[L]:ptr[L + 1]]
            loc = at[~shared[at]]
            self.local.append(torch.as_tensor(loc, device=dev) if len(loc) else None)
            per = {}
            for nb, r in iface.items():
                sel = r[level[r] == L]          # interface-map order
                if len(sel):
                    per[nb] = torch.as_tensor(sel, device=dev)
            self.shared.append(per)
        self.level = level

    def sweep(self, du, df, omega, volume):
        """One forward Gauss-Seidel sweep (surface levels, ghost refresh,
        interiors)."""
        torch = require_cuda()
        op = self.op
        D = op._device()
        dg, ds = D["grid"], D["surf"]
        gs = ds.gs_tables(dg)
        st = op._stream()
        for L in range(self.nlev):
            loc = self.local[L]
            if loc is not None:
                check(lib.hhg_smooth_surface_rows(dg.ref, ds.ref, gs["ref"], loc.data_ptr(),
                                                  loc.numel(), float(omega), du.data_ptr(),
                                                  df.data_ptr(), st), "smooth_surface_rows")
            for nb, rows in self.shared[L].items():
                m = rows.numel()
                part = torch.empty(2 * m, dtype=torch.float64, device="cuda")
                check(lib.hhg_smooth_surface_partial(dg.ref, ds.ref, gs["ref"], rows.data_ptr(),
                                                     m, du.data_ptr(), part.data_ptr(),
                                                     part[m:].data_ptr(), st),
                      "smooth_surface_partial")
                theirs = _swap(self.dist, nb, part)
                tot = (theirs + part) if nb < self.rank else (part + theirs)
                check(lib.hhg_smooth_surface_finish(dg.ref, ds.ref, gs["ref"], rows.data_ptr(),
                                                    m, tot.data_ptr(), tot[m:].data_ptr(),
                                                    float(omega), du.data_ptr(), df.data_ptr(),
                                                    st), "smooth_surface_finish")
        check(lib.hhg_ghost_update(dg.ref, du.data_ptr(), st), "ghost_update")
        volume()


class ShardedHierarchy:
    """One rank's levels lmin..lmax of a slab-sharded multigrid hierarchy
    (the reference's GridHierarchy, multigrid.py:92-128, per slab)."""

    def __init__(self, rank, world, dist, lmax, variant, coeff, lmin=0, nx=4, ny=None,
                 omega=1.0, coarse_tol=1e-12):
        if lmax < lmin:
            raise ValueError("lmax must be >= lmin")
        torch = require_cuda()
        self.torch, self.dist, self.rank, self.world = torch, dist, rank, world
        self.lmin, self.lmax = lmin, lmax
        self.omega, self.coarse_tol = omega, coarse_tol
        ny = nx if ny is None else ny
        mesh = slab_mesh(rank, world, nx, ny)
        h = 1.0 / max(nx, ny)
        self.grids, self.ops, self.sops, self.maps = {}, {}, {}, {}
        self._dT, self._sched = {}, {}
        for lvl in range(lmin, lmax + 1):
            grid = RefinedGrid(mesh, lvl)
            op = Operator(grid, variant, sample_nodal(coeff, grid))
            imap = InterfaceMap(grid, rank, world, h)
            sop = ShardedOperator(op, imap, dist, grid.dirichlet_mask)
            self.grids[lvl], self.ops[lvl], self.maps[lvl], self.sops[lvl] = grid, op, imap, sop
            if lvl > lmin:
                self._dT[lvl] = DeviceTransfer(self.ops[lvl - 1], op, torch)
        for lvl in range(lmin + 1, lmax + 1):
            self._sched[lvl] = _SurfaceSchedule(self.sops[lvl])
        self._owned = {lvl: torch.as_tensor(self.sops[lvl]._owned.astype(np.float64),
                                            device="cuda") for lvl in self.grids}

    def smooth(self, lvl, u, f, sweeps):
        vol = self.ops[lvl]._volume_sweeper(u, f, self.omega)
        for _ in range(sweeps):
            self._sched[lvl].sweep(u, f, self.omega, vol)

    def restrict(self, lvl, r):
        """P^T r with shared fine nodes counted once, coarse interface rows
        completed across ranks, coarse Dirichlet rows zero."""
        from .shard import exchange_partials
        torch = self.torch
        y = torch.empty(self.grids[lvl - 1].n_nodes, dtype=torch.float64, device="cuda")
        self._dT[lvl].restrict(r * self._owned[lvl], y,
                               stream=torch.cuda.current_stream().cuda_stream)
        return exchange_partials(y, self.maps[lvl - 1], self.dist,
                                 self.sops[lvl - 1]._index(y.device))

    def prolongate_add(self, lvl, ec, u):
        self._dT[lvl].prolongate(ec, u, accumulate=True,
                                 stream=self.torch.cuda.current_stream().cuda_stream)

    def coarse_solve(self, f):
        x, _, _ = sharded_cg(self.sops[self.lmin], f, tol=self.coarse_tol)
        return x


def sharded_vcycle(sh: ShardedHierarchy, u, f, level=None, pre=3, post=3):
    """One V(pre, post) cycle on the rank's device vectors (multigrid.py:
    197-214); updates u in place."""
    lvl = sh.lmax if level is None else level
    if lvl == sh.lmin:
        sol = sh.coarse_solve(f)
        d = torch_dirichlet(sh, lvl)
        sol.index_copy_(0, d, u.index_select(0, d))
        u.copy_(sol)
        return u
    sh.smooth(lvl, u, f, pre)
    r = sh.sops[lvl].residual(u, f)
    rc = sh.restrict(lvl, r)
    ec = sh.torch.zeros(sh.grids[lvl - 1].n_nodes, dtype=sh.torch.float64, device="cuda")
    sharded_vcycle(sh, ec, rc, lvl - 1, pre, post)
    sh.prolongate_add(lvl, ec, u)
    sh.smooth(lvl, u, f, post)
    return u


def torch_dirichlet(sh, lvl):
    key = ("dir", lvl)
    if key not in sh._sched:
        sh._sched[key] = sh.torch.as_tensor(np.nonzero(sh.grids[lvl].dirichlet_mask)[0],
                                            device="cuda")
    return sh._sched[key]


def sharded_solve(sh: ShardedHierarchy, f, u0=None, stop="iters:10", pre=3, post=3,
                  max_cycles=100):
    """Repeated sharded V-cycles with the reference's residual tracking
    (multigrid.py:226-270): residual norms over the global system (shared
    nodes counted once) scaled by 2^(-L d / 2).  f: the rank's device
    right-hand side (interface entries equal on both sides)."""
    torch = sh.torch
    sop = sh.sops[sh.lmax]
    grid = sh.grids[sh.lmax]
    u = torch.zeros(grid.n_nodes, dtype=torch.float64, device="cuda") if u0 is None \
        else u0.clone()
    mode, val = _parse_stop(stop)
    hscale = 2.0 ** (-sh.lmax * grid.dim / 2.0)

    def res_norm():
        r = sop.residual(u, f)
        return hscale * float(np.sqrt(sop.dot(r, r).item()))

    t0 = time.perf_counter()
    lib.hhg_status_reset()
    res = [res_norm()]
    target = val * res[0] if mode == "drop" else None
    fn = hscale * float(np.sqrt(sop.dot(f * sop._mask("free", f.device), f).item()))
    floor = 1e-15 * max(fn, 1e-300)
    n_cycles = val if mode == "iters" else max_cycles
    grow, diverged = 0, False
    if res[0] > floor:
        for _ in range(n_cycles):
            sharded_vcycle(sh, u, f, None, pre, post)
            res.append(res_norm())
            grow = grow + 1 if res[-1] > res[-2] else 0
            if grow >= 3:
                diverged = True
                break
            if mode == "drop" and res[-1] <= target:
                break
            if res[-1] <= floor:
                break
    wall = time.perf_counter() - t0
    check(lib.hhg_status(), "smooth")
    i_star = len(res) - 1
    rho = None
    if i_star > 5 and res[5] > 0:
        rho = float((res[i_star] / res[5]) ** (1.0 / (i_star - 5)))
    return u, SolveReport(residuals=res, iterations=i_star, rho=rho, wall_time=wall,
                          flops_add=0, flops_mul=0, diverged=diverged)
