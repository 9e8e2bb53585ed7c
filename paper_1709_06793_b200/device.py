"""Device-resident grid and surface tables for the batched kernels.

HBM layout:

* global vectors (u, f, out) stay in the reference's node numbering; the
  interior of macro element t is the contiguous run
  ``[vol_start[t], vol_start[t] + nvol)`` in (k, j, i) order, which is its
  lattice interior row by row — the volume kernel streams it directly;
* the ghost layer of t is a compact copy of its lattice shell (all points of
  the rows with k = 0, j = 0 or k + j >= n - 1, and the two end points
  i = 0, i = end of every other row), ``srow[k, j]`` gives a row's offset;
  ``shell_gid`` maps shell points to global ids and is the gather list of
  the ghost-layer update;
* the coefficient k lives in full lattice layout per element (8 B/point).

Host-side table construction is numpy; the device copies are torch tensors
used purely as buffers.
"""
from __future__ import annotations

import ctypes
import warnings
from functools import lru_cache

import numpy as np

from ._lib import HhgGrid, HhgSurface, lib
from .mesh import SimplexLattice, lattice_size
from .reference_stencils import CLASS_OF_MASK, class_element_masks
from .mesh import DIRS_3D

__all__ = ["shell_layout", "volume_tiles", "GridTables", "SurfaceTables", "FaceTables",
           "DeviceGrid", "DeviceSurface", "require_cuda"]


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the hhg_b200 operators run only on "
                           "the GPU (there is no CPU fallback)")
    return torch


@lru_cache(maxsize=16)
def shell_layout(n: int):
    """(srow[(n+1)^2] int32, shell lattice positions int64, shell size)."""
    lat = SimplexLattice(3, n)
    srow = np.full((n + 1) * (n + 1), -1, dtype=np.int32)
    pos = []
    off = 0
    for k in range(n + 1):
        for j in range(n + 1 - k):
            b = int(lat.base[k, j])
            rl = n + 1 - k - j
            srow[k * (n + 1) + j] = off
            if k >= 1 and j >= 1 and k + j <= n - 2:
                pos += [b, b + rl - 1]
                off += 2
            else:
                pos += list(range(b, b + rl))
                off += rl
    pos = np.asarray(pos, dtype=np.int64)
    srow.setflags(write=False)
    pos.setflags(write=False)
    return srow, pos, off


TILE_GROUP = 8   # macro elements whose j-bands are interleaved (L2 reuse)


def volume_tiles(n: int, ntets: int, tile_rows: int, group: int = TILE_GROUP,
                 tile_cols: int = 32):
    """(tet, i0, j0, kmax) work tiles ordered by (element group, j-band,
    element, i): tiles sharing a halo column run back to back, and a band's
    halo rows are re-read by the next band of the same element while they
    are still in L2 (a group of 8 level-8 elements streams ~50 MB between
    the two reads); deep k-marches (low j-bands) start first in each group."""
    tl = []
    for g0 in range(0, ntets, group):
        for j0 in range(1, n - 2, tile_rows):
            for t in range(g0, min(g0 + group, ntets)):
                for i0 in range(1, n - 1 - j0, tile_cols):
                    tl.append((t, i0, j0, n - 1 - i0 - j0))
    if not tl:
        return np.zeros((0, 4), dtype=np.int32)
    return np.ascontiguousarray(np.array(tl, dtype=np.int32))


class GridTables:
    """Host-side (numpy) tables of one grid level on one device."""

    def __init__(self, grid, tile_rows=None, mirror_cols=None):
        n = grid.n
        self.n = n
        self.ntets = grid.macro.n_elements
        self.L = lattice_size(n)
        self.nvol = grid.nodes_per_volume
        self.n_nodes = grid.n_nodes
        self.vol_start = np.ascontiguousarray(grid.vol_start, dtype=np.int64)
        self.srow, self.shell_pos, self.S = shell_layout(n)
        self.shell_gid = np.ascontiguousarray(grid.elem_gidx[:, self.shell_pos])
        if tile_rows is None:
            tile_rows = int(lib.hhg_volume_tile_rows())
        if mirror_cols is None:
            mirror_cols = int(lib.hhg_volume_tile_cols_mirror())
        self.tiles = volume_tiles(n, self.ntets, tile_rows)
        # the default scaling kernel (volume_kernel_mirror) may use wider tiles
        self.mtiles = self.tiles if mirror_cols == 32 else \
            volume_tiles(n, self.ntets, tile_rows, tile_cols=mirror_cols)


def _point_codes(lat, pos):
    c = lat.coords[pos]
    return (c[:, 0] | (c[:, 1] << 10) | (c[:, 2] << 20)).astype(np.int32), c


class SurfaceTables:
    """Incidence lists of the non-Dirichlet surface rows.

    Every shell point p of every macro element t whose global node r is a
    free surface node contributes one incidence (t, p, class(p)) to row r;
    rows are sorted by global id and incidences by t, so row sums have a
    fixed order.
    """

    def __init__(self, grid, gt: GridTables, nodal_kinds=frozenset()):
        n = grid.n
        lat = grid.lat
        free_surface = np.zeros(grid.n_nodes, dtype=bool)
        free_surface[:grid.n_surface_nodes] = True
        free_surface &= ~grid.dirichlet_mask
        code, coords = _point_codes(lat, gt.shell_pos)
        bary = np.column_stack([n - coords.sum(axis=1), coords])
        zmask = ((bary == 0) * (1 << np.arange(4))).sum(axis=1)
        cls = np.array([CLASS_OF_MASK.get(int(m), 255) for m in zmask], dtype=np.uint8)
        gid = gt.shell_gid                                   # (ntets, S)
        keep = free_surface[gid]
        tet = np.broadcast_to(np.arange(gt.ntets, dtype=np.int32)[:, None], gid.shape)
        g = gid[keep]
        order = np.lexsort((tet[keep], g))                   # by gid, then tet
        g = g[order]
        self.inc_tet = np.ascontiguousarray(tet[keep][order])
        spos = np.broadcast_to(np.arange(gt.S)[None, :], gid.shape)[keep][order]
        self.inc_code = np.ascontiguousarray(code[spos])
        self.inc_cls = np.ascontiguousarray(cls[spos])
        self.inc_spos = spos
        if (self.inc_cls == 255).any():
            raise AssertionError("interior lattice point listed as a shell incidence")
        self.rows, first = np.unique(g, return_index=True)
        self.inc_ptr = np.append(first, len(g)).astype(np.int32)
        kinds = grid.node_kind[self.rows]
        self.row_nodal = np.isin(kinds, [int(k) for k in nodal_kinds]).astype(np.uint8)
        self.dir_ids = np.nonzero(grid.dirichlet_mask)[0].astype(np.int64)
        # element-major copy: incidence order (tet, shell position) = lattice
        # order inside each element; row_inc maps row-major -> element-major
        key = self.inc_tet.astype(np.int64) * gt.S + spos
        emaj = np.argsort(key, kind="stable")
        self.p_tet = np.ascontiguousarray(self.inc_tet[emaj])
        self.p_code = np.ascontiguousarray(self.inc_code[emaj])
        self.p_cls = np.ascontiguousarray(self.inc_cls[emaj])
        row_of_inc = np.repeat(np.arange(len(self.rows)), np.diff(self.inc_ptr))
        self.p_nodal = np.ascontiguousarray(self.row_nodal[row_of_inc][emaj])
        inv = np.empty_like(emaj)
        inv[emaj] = np.arange(len(emaj))
        self.row_inc = np.ascontiguousarray(inv.astype(np.int32))
        self._grid = grid
        self._gt = gt

    def neighbour_gids(self):
        """(ninc, 14) global ids of each incidence's in-element neighbours
        (-1 for directions leaving the macro element)."""
        gt, grid = self._gt, self._grid
        lat = grid.lat
        n = gt.n
        i = self.inc_code & 1023
        j = (self.inc_code >> 10) & 1023
        k = (self.inc_code >> 20) & 1023
        _, dir_inside = class_element_masks()
        out = np.full((len(i), 14), -1, dtype=np.int64)
        for d, (di, dj, dk) in enumerate(DIRS_3D):
            ok = dir_inside[self.inc_cls, d]
            qi, qj, qk = i[ok] + di, j[ok] + dj, k[ok] + dk
            flat = lat.base[qk, qj] + qi
            out[ok, d] = grid.elem_gidx[self.inc_tet[ok], flat]
        return out

    def gs_dag(self):
        """Dependencies of the forward surface GS (ascending-id order): row r
        reads the new values of dep_idx[dep_ptr[r]:dep_ptr[r+1]] (its lower-
        id neighbour rows).  Returns (dep_ptr, dep_idx) int64."""
        nb = self.neighbour_gids()
        rows = self.rows
        nrows = len(rows)
        row_of_inc = np.repeat(np.arange(nrows), np.diff(self.inc_ptr))
        pos = np.searchsorted(rows, nb)
        pos_c = np.minimum(pos, nrows - 1)
        is_row = (nb >= 0) & (rows[pos_c] == nb)
        dep_row = np.where(is_row, pos_c, -1)
        src = np.repeat(row_of_inc, 14).reshape(-1, 14)
        m = (dep_row >= 0) & (dep_row < src)
        pairs = np.unique(np.column_stack([src[m], dep_row[m]]), axis=0)
        dep_ptr = np.searchsorted(pairs[:, 0], np.arange(nrows + 1)).astype(np.int64)
        dep_idx = np.ascontiguousarray(pairs[:, 1], dtype=np.int64)
        return dep_ptr, dep_idx

    @staticmethod
    def levels_of(dag, seed=None):
        """level[r] = max(seed[r], 1 + max level of r's dependencies)."""
        dep_ptr, dep_idx = dag
        nrows = len(dep_ptr) - 1
        level = np.zeros(nrows, dtype=np.int64)
        sd = None if seed is None else np.ascontiguousarray(seed, dtype=np.int64)
        nlev = lib.hhg_host_gs_levels_seeded(nrows, dep_ptr.ctypes.data, dep_idx.ctypes.data,
                                             None if sd is None else sd.ctypes.data,
                                             level.ctypes.data)
        if nlev < 0:
            raise AssertionError("surface dependency list is not lower triangular")
        return level

    def gs_levels(self):
        """Level schedule of the forward surface GS (ascending-id order)."""
        level = self.levels_of(self.gs_dag())
        nlev = int(level.max()) + 1 if len(level) else 0
        order = np.argsort(level, kind="stable")
        level_ptr = np.searchsorted(level[order], np.arange(nlev + 1))
        return order.astype(np.int64), level_ptr.astype(np.int64), int(nlev)

    def entry_ptr(self):
        """Row offsets of the precomputed surface rows: one entry per
        (incidence, in-element direction), in accumulation order."""
        _, dir_inside = class_element_masks()
        per_inc = dir_inside.sum(axis=1)[self.inc_cls]
        row_of_inc = np.repeat(np.arange(len(self.rows)), np.diff(self.inc_ptr))
        cnt = np.bincount(row_of_inc, weights=per_inc, minlength=len(self.rows))
        return np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)




def _face_layers(A, cls):
    """Where each stencil direction of a face point lands in the face-local
    layers of one incident element: (nb, dl[14], da[14], db[14]) with nb the
    offset of the inner layer (re-centred so that every offset is in
    [-1, 1]), dl 0 = face layer, 1 = inner layer, -1 = outside the element,
    and (da, db) the face-local offset within that layer."""
    from .reference_stencils import class_element_masks
    _, inside = class_element_masks()
    M = np.array([[A[0], A[1]], [A[2], A[3]], [A[4], A[5]]], dtype=np.float64)

    def solve(v):
        xy = np.rint(np.linalg.lstsq(M, np.asarray(v, dtype=np.float64), rcond=None)[0])
        return (int(xy[0]), int(xy[1])) if np.array_equal(M @ xy, v) else None

    dl, da, db = [-1] * 14, [0] * 14, [0] * 14
    nb = None
    for d in range(14):
        if not inside[cls, d]:
            continue
        xy = solve(DIRS_3D[d])
        if xy is not None:
            dl[d], (da[d], db[d]) = 0, xy
            continue
        if nb is None:
            nb = tuple(int(x) for x in DIRS_3D[d])
        xy = solve(np.asarray(DIRS_3D[d]) - np.asarray(nb))
        if xy is None:
            raise AssertionError("inner stencil direction not on the inner layer")
        dl[d], (da[d], db[d]) = 1, xy
    if nb is None:
        raise AssertionError("face class without inner directions")
    inner = [d for d in range(14) if dl[d] == 1]
    sa = (min(da[d] for d in inner) + max(da[d] for d in inner)) // 2
    sb = (min(db[d] for d in inner) + max(db[d] for d in inner)) // 2
    for d in inner:
        da[d] -= sa
        db[d] -= sb
    nb = tuple(int(x) for x in np.asarray(nb) + M.astype(np.int64) @ np.array([sa, sb]))
    if max(abs(x) for x in da + db) > 1:
        raise AssertionError("unexpected face stencil geometry")
    return nb, tuple(dl), tuple(da), tuple(db)


class FaceTables:
    """Free macro faces for the face-tiled surface kernel.

    Face-local coordinates (a, b) are the barycentrics of the face's second
    and third (sorted) global vertices, so the interior points of face F are
    the global ids face_start[F] + base2(b - 1) + a - 1 (the reference's face
    numbering, mesh.py:654-701).  Per face: its incident elements in
    ascending order with the face's boundary class in each, the affine maps
    (a, b) -> element lattice (i, j, k), the direction table of each
    element; and static layers over (a, b) in [-1, n+1]^2 - the face points
    and each element's layer next to the face: coefficient and global id of
    every lattice point (k never changes, so the kernel gathers only u).
    The remaining surface rows (macro edges and vertices) form a sub-list."""

    def __init__(self, grid, gt: GridTables, st: SurfaceTables, kc_values, tile=None):
        if tile is None:
            ft = int(lib.hhg_face_tile())
            tile = (ft >> 16, ft & 0xffff)
        ta, tb = tile
        self.tile = tile
        n = grid.n
        m = grid.macro
        rows = np.asarray(st.rows)
        npf = grid.nodes_per_face
        sq = n + 3
        self.sq = sq
        recs, tiles, ks, gs = [], [], [], []
        covered = np.zeros(len(rows), dtype=bool)
        inc = [[] for _ in range(len(m.faces))]
        if n >= 4:
            for t in range(m.n_elements):
                for f in range(4):
                    inc[int(m.elem_faces[t, f])].append((t, f))
        lat = grid.lat
        aa, bb = np.meshgrid(np.arange(-1, n + 2), np.arange(-1, n + 2))   # [b, a]
        aa, bb = aa.ravel(), bb.ravel()
        for F, tf in enumerate(inc):
            if not tf or len(tf) > 2:
                continue
            fs = int(grid.face_start[F])
            r0 = int(np.searchsorted(rows, fs))
            if r0 + npf > len(rows) or rows[r0] != fs or rows[r0 + npf - 1] != fs + npf - 1:
                continue                      # Dirichlet face (no rows) or not a plain block
            tf = sorted(tf)
            gA, gB, gC = (int(x) for x in m.faces[F])
            A, c, cls, lay = [], [], [], []
            kl = np.zeros((3, sq * sq))
            gl = np.zeros((3, sq * sq), dtype=np.int32)
            for e, (t, f) in enumerate(tf):
                conn = [int(x) for x in m.elements[t]]
                # barycentric slot s of local vertex s: 0 -> n-i-j-k, 1..3 -> i, j, k
                coef = np.zeros((4, 3), dtype=np.int64)       # slot value = coef @ (a, b, 1)
                coef[conn.index(gA)] = (-1, -1, n)
                coef[conn.index(gB)] = (1, 0, 0)
                coef[conn.index(gC)] = (0, 1, 0)
                Ae = tuple(int(x) for x in coef[1:, :2].ravel())   # (ia, ib, ja, jb, ka, kb)
                ce = tuple(int(x) for x in coef[1:, 2])
                A.append(Ae)
                c.append(ce)
                cls.append(CLASS_OF_MASK[1 << f])
                lay.append(_face_layers(Ae, cls[-1]))
                for l, off in ((0, (0, 0, 0)), (1 + e, lay[-1][0])) if e == 0 else \
                        ((1 + e, lay[-1][0]),):
                    i = ce[0] + off[0] + Ae[0] * aa + Ae[1] * bb
                    j = ce[1] + off[1] + Ae[2] * aa + Ae[3] * bb
                    k = ce[2] + off[2] + Ae[4] * aa + Ae[5] * bb
                    ok = (i >= 0) & (j >= 0) & (k >= 0) & (i + j + k <= n)
                    flat = lat.base[np.where(ok, k, 0), np.where(ok, j, 0)] + np.where(ok, i, 0)
                    kl[l] = np.where(ok, kc_values[t][flat], 0.0)
                    gl[l] = np.where(ok, grid.elem_gidx[t, flat], 0)
            if len(tf) == 1:
                t_, cls_, A_, c_ = (tf[0][0], -1), (cls[0], 0), (A[0], (0,) * 6), (c[0], (0,) * 3)
                lay.append(((0, 0, 0), (-1,) * 14, (0,) * 14, (0,) * 14))
            else:
                t_, cls_, A_, c_ = tuple(x for x, _ in tf), tuple(cls), tuple(A), tuple(c)
            recs.append((t_, cls_, A_, c_, tuple(lay), int(st.row_nodal[r0]), fs, r0))
            ks.append(kl)
            gs.append(gl)
            covered[r0:r0 + npf] = True
            fid = len(recs) - 1
            for b0 in range(1, n - 1, tb):
                for a0 in range(1, n - b0, ta):
                    tiles.append((fid, a0, b0, 0))
        self.faces = recs
        self.tiles = np.ascontiguousarray(np.array(tiles, dtype=np.int32).reshape(-1, 4))
        self.sub_rows = np.ascontiguousarray(np.nonzero(~covered)[0].astype(np.int32))
        self.layer_k = np.ascontiguousarray(np.stack(ks)) if ks else np.zeros((0, 3, sq * sq))
        self.layer_g = np.ascontiguousarray(np.stack(gs)) if gs else \
            np.zeros((0, 3, sq * sq), dtype=np.int32)
        if grid.n_nodes >= 2 ** 31:
            raise ValueError("face-tiled surface rows use 32-bit global ids")

    def packed(self):
        """The faces as an array of hhg_face structs (bytes)."""
        from ._lib import HhgFace
        arr = (HhgFace * max(len(self.faces), 1))()
        for x, (tet, cls, A, c, lay, nodal, fs, rb) in enumerate(self.faces):
            h = arr[x]
            for e in range(2):
                h.tet[e], h.cls[e] = tet[e], cls[e]
                for q in range(6):
                    h.A[e][q] = A[e][q]
                nb, dl, da, db = lay[e]
                for q in range(3):
                    h.c[e][q] = c[e][q]
                    h.nb[e][q] = nb[q]
                for d in range(14):
                    h.dl[e][d], h.da[e][d], h.db[e][d] = dl[d], da[d], db[d]
            h.nodal, h.fs, h.rbase = nodal, fs, rb
        return np.frombuffer(bytes(arr), dtype=np.uint8).copy()


class DeviceGrid:
    """Torch buffers + the hhg_grid descriptor of one level."""

    def __init__(self, gt: GridTables, kc_values: np.ndarray):
        torch = require_cuda()
        dev = torch.device("cuda")
        self.gt = gt
        def t(a, dt=None):
            a = np.ascontiguousarray(a) if dt is None else np.ascontiguousarray(a, dtype=dt)
            with warnings.catch_warnings():
                # read-only coefficient arrays: copied to the device, never written
                warnings.simplefilter("ignore", UserWarning)
                return torch.as_tensor(a, device=dev)
        self.vol_start = t(gt.vol_start)
        self.srow = t(gt.srow)
        self.shell_gid = t(gt.shell_gid)
        self.ghost = torch.zeros(gt.ntets * gt.S, dtype=torch.float64, device=dev)
        self.kc = t(kc_values, np.float64).reshape(-1)
        self.tiles = t(gt.tiles)
        self.mtiles = self.tiles if gt.mtiles is gt.tiles else t(gt.mtiles)
        d = HhgGrid()
        d.n, d.ntets = gt.n, gt.ntets
        d.lat_size, d.nvol, d.shell_size, d.n_nodes = gt.L, gt.nvol, gt.S, gt.n_nodes
        d.vol_start = self.vol_start.data_ptr()
        d.srow = self.srow.data_ptr()
        d.shell_gid = self.shell_gid.data_ptr()
        d.ghost = self.ghost.data_ptr()
        d.kc = self.kc.data_ptr()
        d.tiles = self.tiles.data_ptr() if len(gt.tiles) else None
        d.ntiles = len(gt.tiles)
        d.mtiles = self.mtiles.data_ptr() if len(gt.mtiles) else None
        d.nmtiles = len(gt.mtiles)
        self.desc = d
        self.ref = ctypes.byref(d)


class DeviceSurface:
    def __init__(self, st: SurfaceTables, psh, pfac, tensor=None, faces: FaceTables = None):
        torch = require_cuda()
        dev = torch.device("cuda")
        t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=dev)
        self.st = st
        self.rows = t(st.rows)
        self.row_nodal = t(st.row_nodal)
        self.inc_ptr = t(st.inc_ptr)
        self.inc_tet = t(st.inc_tet)
        self.inc_code = t(st.inc_code)
        self.inc_cls = t(st.inc_cls)
        self.psh = t(psh)
        self.pfac = t(pfac) if pfac is not None else None
        self.dir_ids = t(st.dir_ids)
        self.p_tet = t(st.p_tet)
        self.p_code = t(st.p_code)
        self.p_cls = t(st.p_cls)
        self.p_nodal = t(st.p_nodal)
        self.row_inc = t(st.row_inc)
        self.partial = torch.empty(max(len(st.p_tet), 1), dtype=torch.float64, device=dev)
        d = HhgSurface()
        d.nrows = len(st.rows)
        d.rows = self.rows.data_ptr()
        d.row_nodal = self.row_nodal.data_ptr()
        d.inc_ptr = self.inc_ptr.data_ptr()
        d.inc_tet = self.inc_tet.data_ptr()
        d.inc_code = self.inc_code.data_ptr()
        d.inc_cls = self.inc_cls.data_ptr()
        d.psh = self.psh.data_ptr()
        d.pfac = self.pfac.data_ptr() if self.pfac is not None else None
        d.ndir = len(st.dir_ids)
        d.dir_ids = self.dir_ids.data_ptr()
        d.ninc = len(st.p_tet)
        d.p_tet = self.p_tet.data_ptr()
        d.p_code = self.p_code.data_ptr()
        d.p_cls = self.p_cls.data_ptr()
        d.p_nodal = self.p_nodal.data_ptr()
        d.row_inc = self.row_inc.data_ptr()
        d.partial = self.partial.data_ptr()
        d.nfaces = 0
        self.faces = faces
        if faces is not None and len(faces.faces) and tensor is None:
            self.face_buf = t(faces.packed())
            self.face_tiles = t(faces.tiles)
            self.sub_rows = t(faces.sub_rows if len(faces.sub_rows) else np.zeros(1, np.int32))
            d.nfaces = len(faces.faces)
            d.faces = self.face_buf.data_ptr()
            d.nface_tiles = len(faces.tiles)
            d.face_tiles = self.face_tiles.data_ptr()
            d.nsub = len(faces.sub_rows)
            d.sub_rows = self.sub_rows.data_ptr()
            self.layer_k = t(faces.layer_k.reshape(-1))
            self.layer_g = t(faces.layer_g.reshape(-1))
            d.face_k = self.layer_k.data_ptr()
            d.face_g = self.layer_g.data_ptr()
            d.face_sq = faces.sq
        self.desc = d
        self.ref = ctypes.byref(d)
        self._levels = None
        self._csr = None
        self.tensor = tensor          # (M, device km [ntets*M*L]) or None

    def csr(self, dg):
        """Precomputed surface rows (neighbour ids + weights, filled on the
        device once; k does not change) for apply, residual and smoothing."""
        if self._csr is None:
            from ._lib import HhgSurfaceGS, check
            torch = require_cuda()
            ent_ptr = self.st.entry_ptr()
            nent = int(ent_ptr[-1])
            keep = [torch.as_tensor(ent_ptr, device="cuda"),
                    torch.empty(max(nent, 1), dtype=torch.int32, device="cuda"),
                    torch.empty(max(nent, 1), dtype=torch.float64, device="cuda"),
                    torch.empty(max(len(self.st.rows), 1), dtype=torch.float64, device="cuda")]
            d = HhgSurfaceGS()
            d.ent_ptr, d.ent_col = keep[0].data_ptr(), keep[1].data_ptr()
            d.ent_val, d.row_diag = keep[2].data_ptr(), keep[3].data_ptr()
            stream = torch.cuda.current_stream().cuda_stream
            if self.tensor is not None:
                M, km = self.tensor
                check(lib.hhg_tensor_surface_prepare(dg.ref, self.ref, ctypes.byref(d), M,
                                                     km.data_ptr(), stream),
                      "tensor_surface_prepare")
            else:
                check(lib.hhg_smooth_surface_prepare(dg.ref, self.ref, ctypes.byref(d),
                                                     stream), "smooth_surface_prepare")
            self._csr = {"desc": d, "ref": ctypes.byref(d), "keep": keep}
        return self._csr

    def gs_tables(self, dg):
        """Level schedule of the surface smoother on top of csr()."""
        c = self.csr(dg)
        if self._levels is None:
            torch = require_cuda()
            order, ptr, nlev = self.st.gs_levels()
            keep = [torch.as_tensor(order, device="cuda"), torch.as_tensor(ptr, device="cuda")]
            d = c["desc"]
            d.level_rows, d.level_ptr = keep[0].data_ptr(), keep[1].data_ptr()
            d.nlev = nlev
            # level-ordered slots of the one-cluster sweep
            from ._lib import SURF_SLOT_PF, check
            ns = len(order)
            slots = [torch.empty(max(ns, 1), dtype=torch.int64, device="cuda"),
                     torch.empty(max(ns, 1), dtype=torch.int32, device="cuda"),
                     torch.empty(max(ns, 1), dtype=torch.float64, device="cuda"),
                     torch.empty(max(ns, 1) * SURF_SLOT_PF, dtype=torch.int32, device="cuda"),
                     torch.empty(max(ns, 1) * SURF_SLOT_PF, dtype=torch.float64,
                                 device="cuda"),
                     torch.empty(max(ns, 1), dtype=torch.int32, device="cuda"),
                     torch.zeros(1, dtype=torch.int32, device="cuda")]
            d.nslots = ns
            (d.slot_gid, d.slot_cnt, d.slot_diag, d.slot_col, d.slot_val, d.slot_dyn,
             d.sweep_bar) = (x.data_ptr() for x in slots)
            # level of every schedule row by global id (entries of the
            # previous level are the ones read after the barrier)
            rows = np.asarray(self.st.rows, dtype=np.int64)
            lv = np.full(int(rows.max()) + 1 if len(rows) else 1, -1, dtype=np.int32)
            lv[rows[order]] = np.repeat(np.arange(nlev, dtype=np.int32), np.diff(ptr))
            lv_d = torch.as_tensor(lv, device="cuda")
            check(lib.hhg_smooth_surface_slots(dg.ref, self.ref, c["ref"], lv_d.data_ptr(),
                                               len(lv),
                                               torch.cuda.current_stream().cuda_stream),
                  "smooth_surface_slots")
            torch.cuda.current_stream().synchronize()   # lv_d is temporary
            c["keep"] += keep + slots
            self._levels = nlev
        return {"ref": c["ref"], "nlev": self._levels}
