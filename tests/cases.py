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
