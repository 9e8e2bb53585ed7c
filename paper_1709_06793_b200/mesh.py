"""Host-side macro meshes, barycentric lattices and the HHG global numbering.

This is the setup layer of the drop-in: it reproduces the node numbering of
the reference package exactly, because the device operators consume and
produce vectors in that numbering (so a user's `u` means the same thing on
both sides).  Numbering rules restated from the reference:

* macro mesh orientation — an element with negative signed volume swaps its
  local vertices 0 and 1 (`pkg/src/hhgscale/mesh.py:104-119`);
* macro edges / faces are the lexicographically sorted unique vertex tuples
  (`mesh.py:130-170`); boundary faces touch one element, boundary edges and
  vertices are those contained in a boundary face;
* global ids: macro vertices, then edge interiors (ordered by the barycentric
  coordinate of the higher-id endpoint), then face interiors (2-D lattice rank
  of the two higher-id barycentrics), then per-element volume blocks in
  (k, j, i) order (`mesh.py:579-621, 654-701`);
* lattice flat order is k-major, then j, then i (`mesh.py:457-504`), with the
  closed form ``base(k, j) = P(n) - P(n-k) + j (n+1-k) - j (j-1) / 2`` where
  ``P(m) = (m+1)(m+2)(m+3)/6`` is the point count of a size-m lattice.

Coordinates are built with the same floating-point expressions as the
reference so that coefficient samples are bitwise identical.

Only 3-D (tetrahedral) meshes carry operators in this package; 2-D lattices
are kept for face-interior ranking.
"""
from __future__ import annotations

import itertools
from enum import IntEnum
from functools import lru_cache

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

__all__ = [
    "PrimitiveKind", "MacroMesh", "MeshFormatError", "RefinedGrid",
    "SimplexLattice", "refine_uniform", "lattice_elements", "load_macro_mesh",
    "reference_simplex", "unit_cube_6", "unit_cube_12", "cylinder_shell_box",
    "kuhn_blocks", "DIRS_3D", "LOCAL_EDGES_3D", "LOCAL_FACES_3D",
    "lattice_base", "lattice_size", "classify_primitives", "neighborhood",
]

# The 14 stencil directions of an interior lattice node, (di, dj, dk); the
# second half mirrors the first (d + 7).  Order fixed by the reference
# (`mesh.py:44-48`) because stencil tables and kernels index it.
DIRS_3D = np.array(
    [(1, 0, 0), (0, 1, 0), (0, 0, 1), (1, -1, 0), (1, 0, -1), (0, 1, -1),
     (1, -1, 1),
     (-1, 0, 0), (0, -1, 0), (0, 0, -1), (-1, 1, 0), (-1, 0, 1), (0, -1, 1),
     (-1, 1, -1)], dtype=np.int64)

# The six directions of a 2-D (triangle) lattice node, mirrored the same way
# (`mesh.py:41-43`); used by the 2-D MA2 set-up (ma2.py) and kernels.
DIRS_2D = np.array([(1, 0), (0, 1), (1, -1), (-1, 0), (0, -1), (-1, 1)], dtype=np.int64)

LOCAL_EDGES_3D = ((0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3))
# face f is opposite local vertex f
LOCAL_FACES_3D = ((1, 2, 3), (0, 2, 3), (0, 1, 3), (0, 1, 2))



def _parallel(fn, count):
    """fn(0..count-1) on a thread pool (per-element numpy work on disjoint
    slices: same values as the serial loop)."""
    workers = min(count, os.cpu_count() or 1, 16)
    if workers <= 1 or count < 4:
        for i in range(count):
            fn(i)
        return
    with ThreadPoolExecutor(max_workers=workers) as ex:
        list(ex.map(fn, range(count)))

class PrimitiveKind(IntEnum):
    VERTEX = 0
    EDGE = 1
    FACE = 2
    VOLUME = 3


class MeshFormatError(ValueError):
    pass


# ---------------------------------------------------------------------------
# lattice arithmetic
# ---------------------------------------------------------------------------

def lattice_size(n: int, dim: int = 3) -> int:
    """Number of points of the size-n barycentric lattice."""
    if n < 0:
        return 0
    if dim == 2:
        return (n + 1) * (n + 2) // 2
    return (n + 1) * (n + 2) * (n + 3) // 6


def lattice_base(n, k, j):
    """Flat index of the first point of lattice row (k, j) (3-D, closed form)."""
    k = np.asarray(k, dtype=np.int64)
    j = np.asarray(j, dtype=np.int64)
    tot = (n + 1) * (n + 2) * (n + 3) // 6
    m = n - k
    below = (m + 1) * (m + 2) * (m + 3) // 6
    return tot - below + j * (n + 1 - k) - j * (j - 1) // 2


class SimplexLattice:
    """Points (i, j[, k]) >= 0 with coordinate sum <= n, flat k/j/i order."""

    def __init__(self, dim: int, n: int):
        if n < 0:
            raise ValueError("lattice size must be >= 0")
        if dim not in (2, 3):
            raise ValueError("dim must be 2 or 3")
        self.dim, self.n = dim, n
        self.size = lattice_size(n, dim)
        if dim == 2:
            j = np.arange(n + 1, dtype=np.int64)
            self.base = j * (n + 1) - j * (j - 1) // 2
            rows = np.repeat(j, n + 1 - j)
            ii = np.arange(self.size, dtype=np.int64) - self.base[rows]
            self.coords = np.column_stack([ii, rows])
            return
        kk, jj = np.meshgrid(np.arange(n + 1), np.arange(n + 1), indexing="ij")
        base = lattice_base(n, kk, jj)
        base[kk + jj > n] = -1
        self.base = base.astype(np.int64)
        if self.size == 0:
            self.coords = np.zeros((0, 3), dtype=np.int64)
            return
        valid = (kk + jj <= n)
        rk, rj = kk[valid], jj[valid]            # rows in flat (k, j) order
        rlen = n + 1 - rk - rj
        kcol = np.repeat(rk, rlen)
        jcol = np.repeat(rj, rlen)
        icol = np.arange(self.size, dtype=np.int64) - np.repeat(base[valid], rlen)
        self.coords = np.column_stack([icol, jcol, kcol]).astype(np.int64)

    def index(self, pts):
        pts = np.asarray(pts, dtype=np.int64)
        if self.dim == 2:
            return self.base[pts[..., 1]] + pts[..., 0]
        return self.base[pts[..., 2], pts[..., 1]] + pts[..., 0]


# ---------------------------------------------------------------------------
# macro mesh
# ---------------------------------------------------------------------------

class MacroMesh:
    """Conforming tetrahedral (or triangular) macro mesh.

    ``boundary_faces`` optionally overrides the boundary detection with a set
    of sorted vertex triples; sub-meshes of a sharded mesh use it so faces cut
    by the partition are not mistaken for Dirichlet boundary.
    """

    def __init__(self, vertices, elements, dim=None, boundary_faces=None):
        vertices = np.asarray(vertices, dtype=np.float64)
        elements = np.asarray(elements, dtype=np.int64)
        if vertices.ndim != 2 or vertices.shape[1] not in (2, 3):
            raise MeshFormatError("vertices must be (n, 2) or (n, 3)")
        self.dim = int(dim if dim is not None else vertices.shape[1])
        if vertices.shape[1] != self.dim:
            raise MeshFormatError("vertex coordinate count does not match DIM")
        if elements.ndim != 2 or elements.shape[1] != self.dim + 1:
            raise MeshFormatError(
                f"elements must have {self.dim + 1} vertex indices each")
        self.vertices = vertices
        self.elements = elements.copy()
        self._orient()
        self._entities(boundary_faces)

    def signed_volumes(self):
        v = self.vertices[self.elements]
        e = v[:, 1:] - v[:, :1]
        if self.dim == 2:
            return (e[:, 0, 0] * e[:, 1, 1] - e[:, 0, 1] * e[:, 1, 0]) / 2.0
        return np.linalg.det(e) / 6.0

    def _orient(self):
        nv = len(self.vertices)
        el = self.elements
        if el.size and (el.min() < 0 or el.max() >= nv):
            raise MeshFormatError("element vertex index out of range")
        srt = np.sort(el, axis=1)
        rep = (srt[:, 1:] == srt[:, :-1]).any(axis=1)
        if rep.any():
            raise MeshFormatError(f"element {int(np.argmax(rep))} repeats a vertex")
        vol = self.signed_volumes()
        if np.any(vol == 0.0):
            raise MeshFormatError(
                f"element {int(np.argmax(vol == 0.0))} is degenerate (zero volume)")
        neg = vol < 0
        el[neg, 0], el[neg, 1] = el[neg, 1].copy(), el[neg, 0].copy()

    def _entities(self, boundary_faces):
        el = self.elements
        nv = len(self.vertices)
        self._nv = nv
        if self.dim == 2:
            loc = ((0, 1), (0, 2), (1, 2))
        else:
            loc = LOCAL_EDGES_3D
        pairs = np.sort(el[:, loc], axis=2)                    # (ne, nloc, 2)
        ekey = pairs[..., 0] * nv + pairs[..., 1]
        self._edge_key, inv = np.unique(ekey.ravel(), return_inverse=True)
        self.edges = np.column_stack([self._edge_key // nv, self._edge_key % nv])
        self.elem_edges = inv.reshape(len(el), len(loc))
        if self.dim == 2:
            cnt = np.bincount(self.elem_edges.ravel(), minlength=len(self.edges))
            if cnt.max(initial=0) > 2:
                raise MeshFormatError("non-conforming mesh: edge shared by >2 elements")
            self.boundary_edge = cnt == 1
            self.boundary_vertex = np.zeros(nv, dtype=bool)
            self.boundary_vertex[self.edges[self.boundary_edge].ravel()] = True
            self.faces = np.zeros((0, 3), dtype=np.int64)
            self.elem_faces = np.zeros((len(el), 0), dtype=np.int64)
            self.boundary_face = np.zeros(0, dtype=bool)
            return
        tri = np.sort(el[:, LOCAL_FACES_3D], axis=2)           # (ne, 4, 3)
        fkey = (tri[..., 0] * nv + tri[..., 1]) * nv + tri[..., 2]
        self._face_key, finv = np.unique(fkey.ravel(), return_inverse=True)
        fk = self._face_key
        self.faces = np.column_stack([fk // (nv * nv), (fk // nv) % nv, fk % nv])
        self.elem_faces = finv.reshape(len(el), 4)
        cnt = np.bincount(self.elem_faces.ravel(), minlength=len(self.faces))
        if cnt.max(initial=0) > 2:
            raise MeshFormatError("non-conforming mesh: face shared by >2 elements")
        if boundary_faces is None:
            self.boundary_face = cnt == 1
        else:
            bf = np.asarray(sorted(tuple(sorted(f)) for f in boundary_faces),
                            dtype=np.int64).reshape(-1, 3)
            bkey = (bf[:, 0] * nv + bf[:, 1]) * nv + bf[:, 2]
            self.boundary_face = np.isin(fk, bkey)
        bfaces = self.faces[self.boundary_face]
        self.boundary_vertex = np.zeros(nv, dtype=bool)
        self.boundary_vertex[bfaces.ravel()] = True
        be = np.concatenate([bfaces[:, [0, 1]], bfaces[:, [0, 2]],
                             bfaces[:, [1, 2]]])
        self.boundary_edge = np.isin(self._edge_key, be[:, 0] * nv + be[:, 1])

    def edge_index(self, a, b):
        a, b = (a, b) if a < b else (b, a)
        key = a * self._nv + b
        i = int(np.searchsorted(self._edge_key, key))
        if i >= len(self._edge_key) or self._edge_key[i] != key:
            raise KeyError(f"no edge ({a}, {b})")
        return i

    def face_index(self, tri):
        a, b, c = sorted(int(x) for x in tri)
        key = (a * self._nv + b) * self._nv + c
        i = int(np.searchsorted(self._face_key, key))
        if i >= len(self._face_key) or self._face_key[i] != key:
            raise KeyError(f"no face {tri}")
        return i

    @property
    def n_elements(self):
        return len(self.elements)

    def element_scale(self):
        fac = 2.0 if self.dim == 2 else 6.0
        return float((fac * np.abs(self.signed_volumes()).mean()) ** (1.0 / self.dim))


def load_macro_mesh(source) -> MacroMesh:
    """Parse ``DIM d / VERTICES n ... / ELEMENTS m ...`` (``#`` comments)."""
    if hasattr(source, "read"):
        text = source.read()
    else:
        try:
            with open(source, "r", encoding="utf-8") as fh:
                text = fh.read()
        except (OSError, ValueError):
            text = str(source)
    lines = [(no, ln.split("#", 1)[0].strip())
             for no, ln in enumerate(text.splitlines(), start=1)]
    lines = [(no, ln) for no, ln in lines if ln]
    it = iter(lines)

    def header(word):
        try:
            no, ln = next(it)
        except StopIteration:
            raise MeshFormatError(f"unexpected end of file while reading {word}") from None
        parts = ln.split()
        if len(parts) != 2 or parts[0].upper() != word:
            raise MeshFormatError(f"line {no}: expected '{word} <int>', got {ln!r}")
        return int(parts[1]), no

    dim, no = header("DIM")
    if dim not in (2, 3):
        raise MeshFormatError(f"line {no}: DIM must be 2 or 3")

    def block(word, width, conv):
        cnt, _ = header(word)
        rows = []
        for _ in range(cnt):
            try:
                no, ln = next(it)
            except StopIteration:
                raise MeshFormatError(f"unexpected end of file in {word}") from None
            vals = ln.split()
            if len(vals) != width:
                raise MeshFormatError(f"line {no}: expected {width} values")
            rows.append([conv(v) for v in vals])
        return rows

    verts = block("VERTICES", dim, float)
    elems = block("ELEMENTS", dim + 1, int)
    rest = next(it, None)
    if rest is not None:
        raise MeshFormatError(f"line {rest[0]}: trailing content {rest[1]!r}")
    return MacroMesh(np.array(verts, dtype=float).reshape(-1, dim),
                     np.array(elems, dtype=np.int64).reshape(-1, dim + 1), dim=dim)


# ---------------------------------------------------------------------------
# generators (3-D)
# ---------------------------------------------------------------------------

def reference_simplex(dim=3) -> MacroMesh:
    if dim == 2:
        return MacroMesh([(0, 0), (1, 0), (0, 1)], [(0, 1, 2)])
    return MacroMesh([(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)], [(0, 1, 2, 3)])


def _kuhn_split(origin_vid, strides):
    """Six Kuhn tetrahedra of one hexahedral block: one per axis permutation,
    all sharing the main diagonal (corner 000 to corner 111)."""
    out = []
    for perm in itertools.permutations(range(3)):
        a = strides[perm[0]]
        b = a + strides[perm[1]]
        out.append((origin_vid, origin_vid + a, origin_vid + b,
                    origin_vid + strides[0] + strides[1] + strides[2]))
    return out


def kuhn_blocks(xs, ys, zs) -> MacroMesh:
    """Tensor-product box of (len(xs)-1)(len(ys)-1)(len(zs)-1) blocks, each
    split into six Kuhn tetrahedra.  Vertex id = i + nx1 (j + ny1 k); blocks
    in (k, j, i) order; per block the tets follow the axis permutations in
    lexicographic order — the same layout `cylinder_shell_box` uses
    (`mesh.py:425-450`)."""
    xs, ys, zs = (np.asarray(a, dtype=float) for a in (xs, ys, zs))
    nx1, ny1, nz1 = len(xs), len(ys), len(zs)
    K, J, I = np.meshgrid(np.arange(nz1), np.arange(ny1), np.arange(nx1),
                          indexing="ij")
    verts = np.column_stack([xs[I.ravel()], ys[J.ravel()], zs[K.ravel()]])
    strides = (1, nx1, nx1 * ny1)
    elems = []
    for k in range(nz1 - 1):
        for j in range(ny1 - 1):
            for i in range(nx1 - 1):
                elems += _kuhn_split(i + nx1 * (j + ny1 * k), strides)
    return MacroMesh(verts, elems)


def unit_cube_6() -> MacroMesh:
    """Unit cube as six tetrahedra around the (0,0,0)-(1,1,1) diagonal."""
    return kuhn_blocks([0.0, 1.0], [0.0, 1.0], [0.0, 1.0])


def unit_cube_12() -> MacroMesh:
    """Unit cube as twelve tetrahedra around the centre vertex."""
    corners = [(x, y, z) for z in (0, 1) for y in (0, 1) for x in (0, 1)]
    verts = np.array(corners + [(0.5, 0.5, 0.5)], dtype=float)
    quads = [(0, 2, 6, 4), (1, 3, 7, 5), (0, 1, 5, 4), (2, 3, 7, 6),
             (0, 1, 3, 2), (4, 5, 7, 6)]
    elems = []
    for a, b, c, d in quads:
        elems += [(a, b, c, 8), (a, c, d, 8)]
    return MacroMesh(verts, elems)


def cylinder_shell_box(nr=1, na=6, nz=8, r1=0.8, r2=1.0, z1=4.0) -> MacroMesh:
    """Reference box (r1, r2) x (0, pi) x (0, z1) as nr*na*nz Kuhn blocks."""
    return kuhn_blocks(np.linspace(r1, r2, nr + 1), np.linspace(0.0, np.pi, na + 1),
                       np.linspace(0.0, z1, nz + 1))


def unit_cube_blocks(nx, ny, nz, lz=None) -> MacroMesh:
    """Unit-spaced Kuhn block mesh on [0,nx/m]x... : nx*ny*nz cubes of edge
    1/max(nx,ny) stacked in z (BASELINE configs 3-5: 2x2x2 = 48 tets,
    4x4x1 slab = 96 tets per GPU)."""
    h = 1.0 / max(nx, ny)
    return kuhn_blocks(np.linspace(0.0, nx * h, nx + 1),
                       np.linspace(0.0, ny * h, ny + 1),
                       np.linspace(0.0, nz * h if lz is None else lz, nz + 1))


# ---------------------------------------------------------------------------
# fine elements (Bey red refinement) — used by the oracle and for shells
# ---------------------------------------------------------------------------

# children of a tet (v0..v3, then edge midpoints in LOCAL_EDGES_3D order 4..9)
_BEY_CHILDREN = ((0, 4, 5, 6), (4, 1, 7, 8), (5, 7, 2, 9), (6, 8, 9, 3),
                 (4, 5, 6, 8), (4, 5, 7, 8), (5, 6, 8, 9), (5, 7, 8, 9))


@lru_cache(maxsize=None)
def lattice_elements(dim: int, level: int, shell_only: bool = False):
    """Fine tetrahedra of the level-``level`` lattice as (nt, 4, 3) lattice
    coordinates (Bey's rule applied recursively from the macro tet).  With
    ``shell_only`` only elements with a vertex on the macro boundary."""
    if dim != 3:
        raise ValueError("only tetrahedral lattices are supported")
    n = 1 << level
    tets = np.array([[(0, 0, 0), (n, 0, 0), (0, n, 0), (0, 0, n)]], dtype=np.int64)
    for _ in range(level):
        mids = [(tets[:, a] + tets[:, b]) // 2 for a, b in LOCAL_EDGES_3D]
        pool = np.stack([tets[:, v] for v in range(4)] + mids, axis=1)
        tets = np.concatenate([pool[:, list(c)] for c in _BEY_CHILDREN], axis=0)
        if shell_only:
            last = n - tets.sum(axis=2)
            lo = np.minimum(tets.min(axis=(1, 2)), last.min(axis=1))
            tets = tets[lo == 0]
    tets.setflags(write=False)
    return tets


# ---------------------------------------------------------------------------
# refined grid with global numbering
# ---------------------------------------------------------------------------

class RefinedGrid:
    """Uniform refinement of a tetrahedral macro mesh to ``level``."""

    def __init__(self, macro: MacroMesh, level: int):
        if level < 0:
            raise ValueError("level must be >= 0")
        if macro.dim != 3:
            raise ValueError("the B200 operators are tetrahedral (dim 3)")
        self.macro = macro
        self.level = level
        self.dim = 3
        self.n = 1 << level
        self.lat = SimplexLattice(3, self.n)
        self._numbering()
        self._coords()
        self._gidx()
        self._dirichlet()

    # -- id ranges ------------------------------------------------------------
    def _numbering(self):
        m, n = self.macro, self.n
        nv = len(m.vertices)
        self.nodes_per_edge = max(n - 1, 0)
        self.nodes_per_face = (n - 1) * (n - 2) // 2 if n >= 3 else 0
        self.nodes_per_volume = (n - 1) * (n - 2) * (n - 3) // 6 if n >= 4 else 0
        ne, nf, nt = len(m.edges), len(m.faces), m.n_elements
        self.edge_start = nv + np.arange(ne, dtype=np.int64) * self.nodes_per_edge
        f0 = nv + ne * self.nodes_per_edge
        self.face_start = f0 + np.arange(nf, dtype=np.int64) * self.nodes_per_face
        v0 = f0 + nf * self.nodes_per_face
        self.vol_start = v0 + np.arange(nt, dtype=np.int64) * self.nodes_per_volume
        self.n_nodes = int(v0 + nt * self.nodes_per_volume)
        self.n_surface_nodes = int(v0) if nt else self.n_nodes
        kinds = [np.full(nv, PrimitiveKind.VERTEX, np.int8),
                 np.full(ne * self.nodes_per_edge, PrimitiveKind.EDGE, np.int8),
                 np.full(nf * self.nodes_per_face, PrimitiveKind.FACE, np.int8),
                 np.full(nt * self.nodes_per_volume, PrimitiveKind.VOLUME, np.int8)]
        owners = [np.arange(nv, dtype=np.int64),
                  np.repeat(np.arange(ne, dtype=np.int64), self.nodes_per_edge),
                  np.repeat(np.arange(nf, dtype=np.int64), self.nodes_per_face),
                  np.repeat(np.arange(nt, dtype=np.int64), self.nodes_per_volume)]
        self.node_kind = np.concatenate(kinds)
        self.node_owner = np.concatenate(owners)

    # -- coordinates (same float expressions as the reference, mesh.py:625-650)
    def _coords(self):
        m, n = self.macro, self.n
        V = m.vertices
        X = np.empty((self.n_nodes, 3))
        X[:len(V)] = V
        npe, npf, npv = self.nodes_per_edge, self.nodes_per_face, self.nodes_per_volume
        if npe:
            t = np.arange(1, n) / n
            for e, (a, b) in enumerate(m.edges):
                s = self.edge_start[e]
                X[s:s + npe] = V[a] + np.outer(t, V[b] - V[a])
        if npf:
            st = SimplexLattice(2, n - 3).coords + 1
            for f, (a, b, c) in enumerate(m.faces):
                s = self.face_start[f]
                X[s:s + npf] = V[a] + st[:, :1] / n * (V[b] - V[a]) \
                    + st[:, 1:] / n * (V[c] - V[a])
        if npv:
            # cast once: int64 @ float64 casts the lattice to float64 on
            # every call before the same float matmul (identical values)
            ijk = (SimplexLattice(3, n - 4).coords + 1).astype(np.float64)

            def element(t_):
                # V0 + (ijk @ E) / n evaluated in place (same operations)
                conn = m.elements[t_]
                s = self.vol_start[t_]
                E = V[conn[1:]] - V[conn[0]]
                dst = X[s:s + npv]
                np.matmul(ijk, E, out=dst)
                np.divide(dst, n, out=dst)
                np.add(V[conn[0]], dst, out=dst)

            # elements are independent slices; numpy releases the GIL
            _parallel(element, m.n_elements)
        self.node_coords = X

    # -- per-element lattice -> global id -----------------------------------
    def _gidx(self):
        m, n, lat = self.macro, self.n, self.lat
        P = lat.coords
        bary = np.stack([n - P.sum(axis=1), P[:, 0], P[:, 1], P[:, 2]])  # (4, L)
        pos = bary > 0
        npos = pos.sum(axis=0)
        g = np.empty((m.n_elements, lat.size), dtype=np.int64)
        vert_mask = npos == 1
        vert_which = np.argmax(pos[:, vert_mask], axis=0)
        edge_sel = {}
        for p, q in LOCAL_EDGES_3D:
            edge_sel[(p, q)] = np.nonzero(pos[p] & pos[q] & (npos == 2))[0]
        face_sel = {}
        for lf in LOCAL_FACES_3D:
            face_sel[lf] = np.nonzero(pos[lf[0]] & pos[lf[1]] & pos[lf[2]] & (npos == 3))[0]
        vol_sel = np.nonzero(npos == 4)[0]
        if len(vol_sel):
            vrank = SimplexLattice(3, n - 4).index(P[vol_sel] - 1)
        f2 = SimplexLattice(2, n - 3) if n >= 3 else None
        for t, conn in enumerate(m.elements):
            row = g[t]
            row[vert_mask] = conn[vert_which]
            for (p, q), sel in edge_sel.items():
                if not len(sel):
                    continue
                gp, gq = int(conn[p]), int(conn[q])
                e = m.edge_index(gp, gq)
                hi = q if gq > gp else p
                row[sel] = self.edge_start[e] + bary[hi, sel] - 1
            for lf, sel in face_sel.items():
                if not len(sel):
                    continue
                glob = conn[list(lf)]
                order = np.argsort(glob, kind="stable")
                lb, lc = lf[order[1]], lf[order[2]]
                f = m.face_index(glob)
                row[sel] = self.face_start[f] + f2.base[bary[lc, sel] - 1] + bary[lb, sel] - 1
            if len(vol_sel):
                row[vol_sel] = self.vol_start[t] + vrank
        self.elem_gidx = g

    def _dirichlet(self):
        m = self.macro
        mask = np.zeros(self.n_nodes, dtype=bool)
        mask[:len(m.vertices)] = m.boundary_vertex
        for e in np.nonzero(m.boundary_edge)[0]:
            s = self.edge_start[e]
            mask[s:s + self.nodes_per_edge] = True
        for f in np.nonzero(m.boundary_face)[0]:
            s = self.face_start[f]
            mask[s:s + self.nodes_per_face] = True
        self.dirichlet_mask = mask
        self.interior_ids = np.nonzero(~mask)[0]

    @property
    def n_interior(self) -> int:
        return len(self.interior_ids)

    def fine_elements(self, t: int, shell_only: bool = False) -> np.ndarray:
        le = lattice_elements(3, self.level, shell_only)
        return self.elem_gidx[t][self.lat.index(le)]

    def h_ref(self) -> float:
        return self.macro.element_scale() / self.n


def refine_uniform(mesh: MacroMesh, level: int) -> RefinedGrid:
    return RefinedGrid(mesh, level)


def classify_primitives(grid: "RefinedGrid"):
    """Number of nodes owned by each primitive kind, keyed by the lower-case
    kind name (mesh.py:748-752 of the reference)."""
    counts = np.bincount(grid.node_kind.astype(np.int64), minlength=len(PrimitiveKind))
    return {PrimitiveKind(k).name.lower(): int(c) for k, c in enumerate(counts) if c}


def neighborhood(grid: "RefinedGrid", t: int) -> np.ndarray:
    """Physical offsets of the 14 stencil neighbours of an interior node of
    macro element t: the lattice directions through the element's edge
    vectors, divided by the refinement n (mesh.py:755-765)."""
    V = np.asarray(grid.macro.vertices, dtype=np.float64)[np.asarray(grid.macro.elements[t])]
    return (DIRS_3D @ (V[1:] - V[0])) / grid.n

