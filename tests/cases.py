"""Seeded inputs of the BASELINE.json configurations, shared by the golden
generator, the tests, smoke() and bench.py.  No public dataset is involved:
the configs are synthetic meshes, analytic coefficients and seeded vectors.
"""
from __future__ import annotations

import numpy as np

from paper_1709_06793_b200 import mesh as M
from paper_1709_06793_b200.coefficients import gaussian_field


def case_mesh(cfg: str):
    """c1: reference tetrahedron; c2: unit cube (6 tets); c3/c4: unit cube as
    2x2x2 Kuhn blocks (48 tets); c5: 4x4x1 slab of Kuhn cubes (96 tets, the
    per-GPU share of the weak-scaling run)."""
    if cfg == "c1":
        return M.reference_simplex(3)
    if cfg == "c2":
        return M.unit_cube_6()
    if cfg in ("c3", "c4"):
        return M.unit_cube_blocks(2, 2, 2)
    if cfg == "c5":
        return M.unit_cube_blocks(4, 4, 1)
    raise KeyError(cfg)


def k_c1():
    """k = 2 + sin(2 pi x) sin(2 pi y) sin(2 pi z) (configs 1 and 5)."""
    def k(p):
        return 2.0 + np.sin(2 * np.pi * p[:, 0]) * np.sin(2 * np.pi * p[:, 1]) \
            * np.sin(2 * np.pi * p[:, 2])
    return k


k_c5 = k_c1


def k_c2():
    """k = 1 + 0.5 exp(-(x^2 + y^2 + z^2)) (config 2)."""
    def k(p):
        return 1.0 + 0.5 * np.exp(-(p[:, 0] ** 2 + p[:, 1] ** 2 + p[:, 2] ** 2))
    return k


def k_c3():
    """k = exp(x + y + z) / e (config 3)."""
    def k(p):
        return np.exp(p[:, 0] + p[:, 1] + p[:, 2]) / np.e
    return k


def c4_field():
    """k = clip(exp(g), 1e-2, 1e2), g seeded unit-variance Gaussian field with
    correlation length 0.1 (config 4)."""
    return gaussian_field(seed=0, corr_len=0.1, n_features=512)


def wiggle3d(x):
    return 1.5 + np.sin(13.7 * x[..., 0] + 8.9 * x[..., 1] + 21.1 * x[..., 2])


def checksum_weights(n):
    return np.random.default_rng(777).uniform(-1.0, 1.0, n)


# ---------------------------------------------------------------------------
# config-2 error norms (test harness restatement of analysis.error_norms,
# /root/reference/pkg/src/hhgscale/analysis.py:311-343, with the 15-point
# degree-5 tetrahedron rule of analysis.py:46-61; pinned against the
# reference's own values by tests/test_norms_golden.py)
# ---------------------------------------------------------------------------
def _tet_rule_5():
    """Barycentric points and weights (summing to 1) of the classical
    15-point degree-5 tetrahedron rule: centroid, two 4-point orbits
    (a, a, a, 1-3a) and one 6-point orbit (b, b, 1/2-b, 1/2-b)."""
    r = np.sqrt(15.0)
    pts, wts = [np.full(4, 0.25)], [16.0 / 135.0]
    for a, w in (((7.0 + r) / 34.0, (2665.0 - 14.0 * r) / 37800.0),
                 ((7.0 - r) / 34.0, (2665.0 + 14.0 * r) / 37800.0)):
        for pos in range(3, -1, -1):
            p = np.full(4, a)
            p[pos] = 1.0 - 3.0 * a
            pts.append(p)
            wts.append(w)
    b = (10.0 - 2.0 * r) / 40.0
    for pair in ((2, 3), (1, 3), (1, 2), (0, 3), (0, 2), (0, 1)):
        p = np.full(4, b)
        p[list(pair)] = 0.5 - b
        pts.append(p)
        wts.append(10.0 / 189.0)
    return np.array(pts), np.array(wts)


def c2_exact(X):
    return np.sin(np.pi * X[:, 0]) * np.sin(np.pi * X[:, 1]) * np.sin(np.pi * X[:, 2])


def c2_exact_grad(X):
    s = np.sin(np.pi * X)
    c = np.cos(np.pi * X)
    return np.pi * np.column_stack([c[:, 0] * s[:, 1] * s[:, 2], s[:, 0] * c[:, 1] * s[:, 2],
                                    s[:, 0] * s[:, 1] * c[:, 2]])


def c2_error_norms(u_h, grid):
    """(discrete L2, quadrature L2, H1-seminorm) errors of a P1 solution
    against u* = sin(pi x) sin(pi y) sin(pi z): per fine element, the P1
    gradient from the inverse edge matrix and the errors at the 15 points."""
    e = u_h - c2_exact(grid.node_coords)
    free = ~grid.dirichlet_mask
    l2d = float(np.sqrt(grid.h_ref() ** 3 * np.sum(e[free] ** 2)))
    bar, wts = _tet_rule_5()
    l2 = h1 = 0.0
    for t in range(grid.macro.n_elements):
        ids = grid.fine_elements(t)
        V = grid.node_coords[ids]
        E = V[:, 1:] - V[:, :1]
        vol = np.abs(np.linalg.det(E)) / 6.0
        uv = u_h[ids]
        grad = np.einsum("kda,ka->kd", np.linalg.inv(E), uv[:, 1:] - uv[:, :1])
        for q in range(len(wts)):
            xq = np.einsum("j,kjd->kd", bar[q], V)
            l2 += wts[q] * float(vol @ (uv @ bar[q] - c2_exact(xq)) ** 2)
            h1 += wts[q] * float(vol @ np.sum((grad - c2_exact_grad(xq)) ** 2, axis=1))
    return l2d, float(np.sqrt(l2)), float(np.sqrt(h1))
