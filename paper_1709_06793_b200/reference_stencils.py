"""Constant-coefficient reference stencils and the element patch tables.

Host-side setup for the device kernels: per macro element
the 14 half stencil entries ``sh = s/2`` of the scaling kernel and the 72
nodal-integration factors ``fac = A_t[0, slot] / 4``.  Everything is a pure
function of the macro element's edge matrix E and the level.

The patch of an interior lattice node is the 24 fine tetrahedra that touch it
(six shapes up to translation).  The element order, the 40-add schedule that
forms all 24 element coefficient sums, and the per-direction accumulation
terms are the ones of `pkg/src/hhgscale/reference_stencils.py:33-159`; they
fix the floating-point association of the nodal kernel, so they are data of
the algorithm rather than a design choice.
"""
from __future__ import annotations

from functools import lru_cache

import numpy as np

from .mesh import DIRS_3D, lattice_elements

__all__ = ["Environment", "environment", "element_gradients",
           "element_stiffness", "environment_matrices", "reference_stencil",
           "classify_edge_types", "partial_stencils", "BOUNDARY_CLASSES",
           "EDGE_GRAY", "EDGE_BLUE", "EDGE_GREEN", "EDGE_RED"]

EDGE_GRAY, EDGE_BLUE, EDGE_GREEN, EDGE_RED = 0, 1, 2, 3
_GRAY_DIR = 6           # (1, -1, 1): the direction parallel to no macro edge
_CANDIDATE_DIRS = (1, 4)

# Patch elements as sorted point-id tuples (0 = centre, 1 + d = neighbour d),
# in the canonical order of reference_stencils.py:48-55.
PATCH_ELEMENTS = (
    (0, 8, 11, 12), (0, 8, 12, 13), (0, 8, 11, 14), (0, 8, 10, 14),
    (0, 8, 9, 13), (0, 8, 9, 10), (0, 3, 11, 12), (0, 3, 12, 13),
    (0, 6, 11, 14), (0, 6, 10, 14), (0, 2, 3, 11), (0, 2, 6, 11),
    (0, 4, 9, 13), (0, 4, 9, 10), (0, 3, 7, 13), (0, 4, 7, 13),
    (0, 5, 6, 10), (0, 4, 5, 10), (0, 1, 2, 3), (0, 1, 3, 7),
    (0, 1, 2, 6), (0, 1, 5, 6), (0, 1, 4, 7), (0, 1, 4, 5),
)
# 40-addition schedule (dst, a, b): slot[dst] = slot[a] + slot[b]; slots 0..14
# hold k at the centre and the 14 neighbours (reference_stencils.py:64-75).
CSE_SCHEDULE = (
    (15, 0, 1), (16, 0, 10), (17, 0, 11), (18, 0, 13), (19, 8, 12),
    (20, 8, 14), (21, 8, 9), (22, 3, 12), (23, 6, 14), (24, 2, 3),
    (25, 2, 6), (26, 4, 9), (27, 3, 7), (28, 4, 7), (29, 5, 6), (30, 4, 5),
    (31, 17, 19), (32, 18, 19), (33, 17, 20), (34, 16, 20), (35, 18, 21),
    (36, 16, 21), (37, 17, 22), (38, 18, 22), (39, 17, 23), (40, 16, 23),
    (41, 17, 24), (42, 17, 25), (43, 18, 26), (44, 16, 26), (45, 18, 27),
    (46, 18, 28), (47, 16, 29), (48, 16, 30), (49, 15, 24), (50, 15, 27),
    (51, 15, 25), (52, 15, 29), (53, 15, 28), (54, 15, 30),
)
CSE_SUMS = tuple(range(31, 55))


class Environment:
    """Combinatorics of the 24-element patch around an interior node."""

    def __init__(self):
        self.dim = 3
        self.dirs = DIRS_3D
        self.ndirs = 14
        lookup = {tuple(d): i for i, d in enumerate(DIRS_3D.tolist())}
        le = lattice_elements(3, 2)
        rel = le - np.ones(3, dtype=np.int64)
        touching = rel[(rel == 0).all(axis=2).any(axis=1)]
        found = {}
        for tet in touching.tolist():
            ids = sorted(((0 if not any(v) else 1 + lookup[tuple(v)]), tuple(v))
                         for v in tet)
            found[tuple(i for i, _ in ids)] = np.array([v for _, v in ids])
        if set(found) != set(PATCH_ELEMENTS):
            raise AssertionError("patch does not match the frozen element table")
        self.nelems = len(PATCH_ELEMENTS)
        self.elem_pts = np.array(PATCH_ELEMENTS, dtype=np.int64)
        self.elem_offsets = np.stack([found[e] for e in PATCH_ELEMENTS])
        # distinct shapes modulo translation, in order of first appearance
        keys, shapes = {}, []
        self.elem_shape = np.empty(self.nelems, dtype=np.int64)
        self.elem_perm = np.empty((self.nelems, 4), dtype=np.int64)
        for t, offs in enumerate(self.elem_offsets):
            order = sorted(range(4), key=lambda v: tuple(offs[v]))
            canon = offs[order] - offs[order[0]]
            key = tuple(map(tuple, canon.tolist()))
            if key not in keys:
                keys[key] = len(shapes)
                shapes.append(canon)
            self.elem_shape[t] = keys[key]
            self.elem_perm[t, order] = np.arange(4)
        self.shape_offsets = np.array(shapes)
        self.nshapes = len(shapes)
        # accumulation terms of stencil direction d: (element, local slot)
        ptr, te, ts = [0], [], []
        for d in range(14):
            for t in range(self.nelems):
                for v in range(1, 4):
                    if self.elem_pts[t, v] == 1 + d:
                        te.append(t)
                        ts.append(v)
            ptr.append(len(te))
        self.term_ptr = np.array(ptr, dtype=np.int64)
        self.term_elem = np.array(te, dtype=np.int64)
        self.term_slot = np.array(ts, dtype=np.int64)
        self.dir_valence = np.diff(self.term_ptr)
        self.cse_schedule = np.array(CSE_SCHEDULE, dtype=np.int64)
        self.cse_sums = np.array(CSE_SUMS, dtype=np.int64)
        self.n_slots = 55
        slots = np.zeros(55)
        k = np.random.default_rng(12345).normal(size=15)
        slots[:15] = k
        for dst, a, b in CSE_SCHEDULE:
            slots[dst] = slots[a] + slots[b]
        if not np.allclose(slots[list(CSE_SUMS)], k[self.elem_pts].sum(axis=1)):
            raise AssertionError("element-sum schedule is inconsistent")


@lru_cache(maxsize=None)
def environment(dim: int = 3) -> Environment:
    if dim != 3:
        raise ValueError("only the 3-D patch is built for the device kernels")
    return Environment()


# ---------------------------------------------------------------------------
# element matrices (P1, exact)
# ---------------------------------------------------------------------------

def element_gradients(verts):
    """Barycentric gradients (m, 4, 3) and volumes (m,) of a simplex batch."""
    verts = np.asarray(verts, dtype=np.float64)
    single = verts.ndim == 2
    if single:
        verts = verts[None]
    d = verts.shape[2]
    E = verts[:, 1:] - verts[:, :1]
    det = np.linalg.det(E)
    if np.any(det == 0.0):
        raise ValueError("degenerate simplex")
    grads = np.empty((verts.shape[0], d + 1, d))
    grads[:, 1:] = np.swapaxes(np.linalg.inv(E), 1, 2)
    grads[:, 0] = -grads[:, 1:].sum(axis=1)
    vol = np.abs(det) / (2.0 if d == 2 else 6.0)
    return (grads[0], vol[0]) if single else (grads, vol)


def element_stiffness(verts, coeff=None):
    """Exact P1 stiffness matrices vol * grad_i . K grad_j; coeff is None,
    per-element scalars (m,) or tensors (m, 3, 3)
    (reference_stencils.py:196-215)."""
    grads, vol = element_gradients(verts)
    single = grads.ndim == 2
    if single:
        grads, vol = grads[None], np.atleast_1d(vol)
    if coeff is None:
        A = np.einsum("mid,mjd->mij", grads, grads)
    elif np.ndim(coeff) <= 1:
        A = np.einsum("m,mid,mjd->mij", np.atleast_1d(np.asarray(coeff, float)),
                      grads, grads)
    else:
        A = np.einsum("mid,mde,mje->mij", grads, np.asarray(coeff, float), grads)
    A *= vol[:, None, None]
    return A[0] if single else A


def environment_matrices(E, level, coeff=None):
    """Stiffness matrices of the 24 patch elements of a macro element with
    edge matrix E at ``level`` (one matrix per shape, expanded by index);
    ``coeff`` is an optional per-shape tensor stack (reference_stencils.py:
    244-261)."""
    env = environment(3)
    n = 1 << level
    verts = (env.shape_offsets @ E) / n
    shape_mats = element_stiffness(verts) if coeff is None else element_stiffness(verts, coeff)
    p = env.elem_perm
    return env, shape_mats[env.elem_shape[:, None, None], p[:, :, None], p[:, None, :]]


def _edge_matrix(grid, t):
    V = grid.macro.vertices[grid.macro.elements[t]]
    return V[1:] - V[0]


def reference_stencil(grid, t: int, level=None):
    """(centre, s[14]) of macro element t: s_d sums A_e[0, slot] over the
    patch elements sharing direction d (reference_stencils.py:264-281)."""
    level = grid.level if level is None else level
    env, mats = environment_matrices(_edge_matrix(grid, t), level)
    s = np.zeros(14)
    for d in range(14):
        lo, hi = env.term_ptr[d], env.term_ptr[d + 1]
        s[d] = mats[env.term_elem[lo:hi], 0, env.term_slot[lo:hi]].sum()
    return mats[:, 0, 0].sum(), s


def nodal_factors(grid, t: int):
    """fac[72] = A_e[0, slot] / 4 per accumulation term (operators.py:249-253)."""
    env, mats = environment_matrices(_edge_matrix(grid, t), grid.level)
    return mats[env.term_elem, 0, env.term_slot] / 4


def classify_edge_types(grid, t: int, level=None):
    """3-D edge colours of macro element t (gray / blue / green / red)."""
    centre, s = reference_stencil(grid, t, level=level)
    colors = np.full(14, EDGE_RED, dtype=np.int64)
    tol = 1e-12 * np.abs(s).max()
    colors[_GRAY_DIR] = EDGE_GRAY
    c1, c2 = _CANDIDATE_DIRS
    blue, green = (c2, c1) if (s[c2] > tol and s[c1] <= tol) else (c1, c2)
    colors[blue], colors[green] = EDGE_BLUE, EDGE_GREEN
    colors[7:] = colors[:7]
    return colors, s, centre


# ---------------------------------------------------------------------------
# partial stencils of boundary lattice points (device surface rows)
# ---------------------------------------------------------------------------

def _classes():
    """The 14 boundary classes of a lattice point, keyed by the set Z of
    vanishing barycentric coordinates (b0 = n-i-j-k, b1 = i, b2 = j, b3 = k):
    4 faces (|Z|=1), 6 edges (|Z|=2), 4 vertices (|Z|=3).  Class id order:
    faces by the vanishing coordinate, edges by LOCAL_EDGES pairs of the two
    *non*-vanishing... kept simple: enumerate Z as bitmasks 1..14 except 15."""
    out = []
    for size in (1, 2, 3):
        for mask in range(1, 15):
            if bin(mask).count("1") == size:
                out.append(mask)
    return tuple(out)


BOUNDARY_CLASSES = _classes()          # 14 bitmasks over barycentric coords
CLASS_OF_MASK = {m: i for i, m in enumerate(BOUNDARY_CLASSES)}


def _bary_offsets(off):
    """Barycentric change (db0, db1, db2, db3) of a lattice offset (di,dj,dk)."""
    off = np.asarray(off)
    return np.concatenate([[-off.sum()], off])


@lru_cache(maxsize=None)
def class_element_masks():
    """inside[c, e]: patch element e lies inside the closed macro element for
    a lattice point of boundary class c (every element vertex keeps the
    vanishing barycentric coordinates >= 0).  Also dir_inside[c, d]."""
    env = environment(3)
    inside = np.zeros((14, env.nelems), dtype=bool)
    dir_inside = np.zeros((14, 14), dtype=bool)
    for c, mask in enumerate(BOUNDARY_CLASSES):
        zs = [b for b in range(4) if mask >> b & 1]
        for e in range(env.nelems):
            ok = True
            for v in range(4):
                db = _bary_offsets(env.elem_offsets[e, v])
                if any(db[z] < 0 for z in zs):
                    ok = False
            inside[c, e] = ok
        for d in range(14):
            db = _bary_offsets(DIRS_3D[d])
            dir_inside[c, d] = all(db[z] >= 0 for z in zs)
    inside.setflags(write=False)
    dir_inside.setflags(write=False)
    return inside, dir_inside


def tensor_component_coeffs(dirs, nshapes):
    """Per-shape tensor of component m: None for the gradient component,
    c_m c_m^T otherwise (operators.py:221-230)."""
    out = []
    for m, c in enumerate(dirs):
        if m == 0:
            out.append(None)
        else:
            c = np.asarray(c)
            out.append(np.broadcast_to(np.outer(c, c), (nshapes, 3, 3)))
    return out


def tensor_tables(grid, t: int, dirs):
    """(shm (M, 14), facm (M, 72)) of macro element t for the M-component
    tensor operators: half stencils and nodal factors per component
    (operators.py:221-238)."""
    env = environment(3)
    E = _edge_matrix(grid, t)
    shm, facm = [], []
    for cf in tensor_component_coeffs(dirs, env.nshapes):
        _, mats = environment_matrices(E, grid.level, coeff=cf)
        s = np.empty(14)
        for d in range(14):
            lo, hi = env.term_ptr[d], env.term_ptr[d + 1]
            s[d] = mats[env.term_elem[lo:hi], 0, env.term_slot[lo:hi]].sum()
        shm.append(s / 2.0)
        facm.append(mats[env.term_elem, 0, env.term_slot] / 4)
    return np.ascontiguousarray(shm), np.ascontiguousarray(facm)


def partial_stencils(grid, t: int, coeff=None):
    """Half stencils restricted to the part of the patch inside macro element
    t, for each of the 14 boundary classes: psh[c, d] = 1/2 sum over inside
    elements of A_e[0, slot], and the nodal factors pfac[c, term] (zero for
    outside elements).  A surface row is the sum over the incident macro
    elements of these one-sided rows — the element-wise assembly of
    operators.py:329-365 grouped by neighbour direction."""
    env, mats = environment_matrices(_edge_matrix(grid, t), grid.level, coeff=coeff)
    inside, _ = class_element_masks()
    vals = mats[env.term_elem, 0, env.term_slot]          # (72,)
    psh = np.zeros((14, 14))
    pfac = np.zeros((14, 72))
    for c in range(14):
        keep = inside[c][env.term_elem]
        pfac[c] = np.where(keep, vals / 4, 0.0)
        for d in range(14):
            lo, hi = env.term_ptr[d], env.term_ptr[d + 1]
            psh[c, d] = vals[lo:hi][keep[lo:hi]].sum() / 2.0
    return psh, pfac
