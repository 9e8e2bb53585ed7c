"""2-D MA2 safeguard of the scaling variant: the marking of obtuse macro
triangles and the per-element inputs of the gray-edge selector kernels.

The reference applies the uniform-ellipticity modification only in 2-D
(operators.py:88-129 `ma2_marks`, :201-220 the `scaling_ma2` set-up,
kernels.py:751-783 / 907-937 the selector in `apply_scaling_2d` /
`gs_scaling_2d`).  The kernels are `hhg_apply_scaling_2d` /
`hhg_gs_scaling_2d` (csrc/hhg_ma2.cuh); this module is their host side:

* `reference_stencil_2d` - the six constant-coefficient stencil entries of a
  macro triangle at a level (reference_stencils.py:264-281 in 2-D: every
  lattice edge lies in one "up" and one "down" fine triangle, s_d is the sum
  of the two stiffness entries);
* `classify_edge_types_2d` (reference_stencils.py:302-332, 2-D branch):
  directions with a positive entry are gray;
* `lambda_min` (reference_stencils.py:339-371): smallest non-trivial
  eigenvalue of the local generalised problem A x = lambda (3I - 11^T) x;
* `kmin_values` (coefficients.py:63-92): nodal minimum over each node's
  closed lattice patch inside the element;
* `ma2_marks` - an obtuse element is marked when some lattice edge along
  its gray direction has (k_e - m_e) a12 > m_e lambda_min, with k_e, m_e
  the edge means of k and k_min and a12 = s_gray / 2;
* `ma2_inputs` - per element (sh, kc, kg, g) exactly as the reference's
  Operator feeds its 2-D kernels: marked elements take k_min on the gray
  pair, the others plain k.

Only the element level is built: the B200 operators are tetrahedral (the
2-D global assembly, numbering and solvers are outside the hot path), so
inputs are per-element lattice arrays (ne, (n+1)(n+2)/2) in the flat j/i
order of `SimplexLattice(2, n)`.
"""
from __future__ import annotations

import numpy as np

from .mesh import DIRS_2D, SimplexLattice
from .reference_stencils import EDGE_GRAY, element_stiffness

__all__ = ["Ma2Grid", "reference_stencil_2d", "classify_edge_types_2d", "lambda_min",
           "kmin_values", "ma2_marks", "ma2_inputs", "apply_ma2_elements", "EDGE_PLAIN"]

EDGE_PLAIN = 4      # 2-D non-gray direction (the reference's EDGE_PLAIN role)

# the six fine triangles around an interior lattice node, as offsets of
# their vertices; every edge (0, d) lies in exactly two of them
_PATCH_2D = (
    ((0, 0), (1, 0), (0, 1)), ((0, 0), (0, 1), (-1, 1)), ((0, 0), (-1, 1), (-1, 0)),
    ((0, 0), (-1, 0), (0, -1)), ((0, 0), (0, -1), (1, -1)), ((0, 0), (1, -1), (1, 0)),
)


class Ma2Grid:
    """A 2-D macro triangle mesh refined to ``level`` (element level only:
    lattice per element, no global numbering)."""

    def __init__(self, macro, level: int):
        if macro.dim != 2:
            raise ValueError("the safeguard marking is defined in 2D")
        self.macro, self.level, self.dim = macro, int(level), 2
        self.n = 1 << self.level
        self.lat = SimplexLattice(2, self.n)

    def element_coords(self, t: int):
        """Physical coordinates of element t's lattice points."""
        V = self.macro.vertices[self.macro.elements[t]]
        return V[0] + (self.lat.coords @ (V[1:] - V[0])) / self.n


def _canonical(offs):
    """Shape of a fine triangle up to translation: vertices sorted by their
    offset tuple, the first at the origin (the reference's environment
    canonicalisation), and where each original vertex went."""
    order = sorted(range(3), key=lambda v: tuple(offs[v]))
    canon = np.asarray(offs)[order] - np.asarray(offs)[order[0]]
    perm = np.empty(3, dtype=np.int64)
    perm[order] = np.arange(3)
    return canon, perm


def reference_stencil_2d(macro, t: int, level: int):
    """s[6] (DIRS_2D order) of macro triangle t at ``level``."""
    V = macro.vertices[macro.elements[t]]
    E = V[1:] - V[0]
    n = 1 << level
    shapes, keys, elem = [], {}, []
    for offs in _PATCH_2D:
        canon, perm = _canonical(offs)
        key = tuple(map(tuple, canon.tolist()))
        if key not in keys:
            keys[key] = len(shapes)
            shapes.append(canon)
        elem.append((keys[key], perm))
    mats = element_stiffness((np.array(shapes, dtype=np.float64) @ E) / n)
    lookup = {tuple(d): i for i, d in enumerate(DIRS_2D.tolist())}
    s = np.zeros(6)
    for (sh, perm), offs in zip(elem, _PATCH_2D):
        for v in (1, 2):
            s[lookup[tuple(offs[v])]] += mats[sh][perm[0], perm[v]]
    return s


def classify_edge_types_2d(macro, t: int, level: int):
    """(colors[6], s[6]): positive entries (beyond 1e-12 of the largest,
    rounding noise of right angles) are gray."""
    s = reference_stencil_2d(macro, t, level)
    tol = 1e-12 * np.abs(s).max()
    colors = np.full(6, EDGE_PLAIN, dtype=np.int64)
    colors[s > tol] = EDGE_GRAY
    return colors, s


_Q_2D = np.column_stack([np.array([1.0, -1.0, 0.0]) / np.sqrt(2.0),
                         np.array([1.0, 1.0, -2.0]) / np.sqrt(6.0)])


def lambda_min(verts):
    """(lambda_min, a12) of a triangle: nodes renumbered cyclically so the
    largest angle is last, A = P1 stiffness, lambda_min = smallest
    eigenvalue of Q^T A Q / 3 (Q: orthonormal basis of the complement of
    the constants, Q^T (3I - 11^T) Q = 3I), a12 = A[0, 1]."""
    verts = np.asarray(verts, dtype=np.float64)
    cos = []
    for i in range(3):
        a = verts[(i + 1) % 3] - verts[i]
        b = verts[(i + 2) % 3] - verts[i]
        cos.append((a @ b) / (np.linalg.norm(a) * np.linalg.norm(b)))
    big = int(np.argmin(cos))
    verts = verts[[(big + 1) % 3, (big + 2) % 3, big]]
    A = element_stiffness(verts)
    lam = np.linalg.eigvalsh(_Q_2D.T @ A @ _Q_2D / 3.0)
    return float(lam[0]), float(A[0, 1])


def _neighbor_table(n: int):
    lat = SimplexLattice(2, n)
    tbl = np.full((6, lat.size), -1, dtype=np.int64)
    for j, d in enumerate(DIRS_2D):
        q = lat.coords + d
        ok = (q >= 0).all(axis=1) & (q.sum(axis=1) <= n)
        tbl[j, ok] = lat.index(q[ok])
    return tbl


def kmin_values(values, n: int):
    """Per element and node: min of k over the node and its lattice
    neighbours inside the element (one-sided on macro boundaries)."""
    vals = np.asarray(values, dtype=np.float64)
    tbl = _neighbor_table(n)
    out = vals.copy()
    for j in range(6):
        m = tbl[j] >= 0
        out[:, m] = np.minimum(out[:, m], vals[:, tbl[j][m]])
    return out


def ma2_marks(grid: Ma2Grid, values):
    """(marked[ne], gray_pair[ne] (-1: no gray direction), kmin values)."""
    vals = np.asarray(values, dtype=np.float64)
    km = kmin_values(vals, grid.n)
    ne = grid.macro.n_elements
    marked = np.zeros(ne, dtype=bool)
    gray_pair = np.full(ne, -1, dtype=np.int64)
    p = grid.lat.coords
    for t in range(ne):
        colors, s = classify_edge_types_2d(grid.macro, t, grid.level)
        gray = np.nonzero(colors[:3] == EDGE_GRAY)[0]
        if len(gray) == 0:
            continue
        g = int(gray[0])
        gray_pair[t] = g
        lam, _ = lambda_min(grid.macro.vertices[grid.macro.elements[t]])
        a12 = s[g] / 2.0
        q = p + DIRS_2D[g]
        ok = (q >= 0).all(axis=1) & (q.sum(axis=1) <= grid.n)
        pi, qi = grid.lat.index(p[ok]), grid.lat.index(q[ok])
        k_e = 0.5 * (vals[t][pi] + vals[t][qi])
        m_e = 0.5 * (km[t][pi] + km[t][qi])
        if np.any((k_e - m_e) * a12 > m_e * lam):
            marked[t] = True
    return marked, gray_pair, km


def ma2_inputs(grid: Ma2Grid, values):
    """Per-element kernel inputs of the 2-D scaling_ma2 operator:
    (sh (ne, 6) = s/2, kc (ne, L), kg (ne, L), g (ne, 6) uint8, marked)."""
    vals = np.ascontiguousarray(values, dtype=np.float64)
    marked, gray_pair, km = ma2_marks(grid, vals)
    ne = grid.macro.n_elements
    sh = np.stack([reference_stencil_2d(grid.macro, t, grid.level) / 2.0 for t in range(ne)])
    g = np.zeros((ne, 6), dtype=np.uint8)
    kg = vals.copy()
    for t in range(ne):
        if marked[t] and gray_pair[t] >= 0:
            g[t, gray_pair[t]] = g[t, gray_pair[t] + 3] = 1
            kg[t] = km[t]
    return sh, vals, kg, g, marked


def apply_ma2_elements(grid: Ma2Grid, values, u_elem, omega=None, f_elem=None):
    """Interior rows of every element's 2-D scaling_ma2 operator on the GPU
    (hhg_apply_scaling_2d), or - with omega and f_elem - one in-place
    element Gauss-Seidel sweep (hhg_gs_scaling_2d); u_elem (ne, L) element
    lattices.  Returns numpy arrays."""
    import ctypes
    from .device import require_cuda
    from ._lib import check, lib
    torch = require_cuda()
    sh, kc, kg, g, _ = ma2_inputs(grid, values)
    n = grid.n
    nint = (n - 1) * (n - 2) // 2
    st = torch.cuda.current_stream().cuda_stream
    outs = []
    for t in range(grid.macro.n_elements):
        dv = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda")   # noqa: E731
        u, k1, k2, s = dv(u_elem[t]), dv(kc[t]), dv(kg[t]), dv(sh[t])
        sel = np.ascontiguousarray(g[t])
        if omega is None:
            out = torch.empty(nint, dtype=torch.float64, device="cuda")
            check(lib.hhg_apply_scaling_2d(n, None, u.data_ptr(), k1.data_ptr(), k2.data_ptr(),
                                           sel.ctypes.data_as(ctypes.c_void_p), s.data_ptr(),
                                           out.data_ptr(), st), "apply_scaling_2d")
            outs.append(out.cpu().numpy())
        else:
            fv = dv(f_elem[t])
            check(lib.hhg_gs_scaling_2d(n, None, u.data_ptr(), fv.data_ptr(), k1.data_ptr(),
                                        k2.data_ptr(), sel.ctypes.data_as(ctypes.c_void_p),
                                        s.data_ptr(), float(omega), st), "gs_scaling_2d")
            outs.append(u.cpu().numpy())
    return np.stack(outs) if outs else np.zeros((0, nint))
