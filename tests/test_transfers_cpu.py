"""The lattice-rule prolongation (multigrid.prolongation_matrix, also the
rules of the device transfer kernels) against the reference's P on golden
vectors: P x and P^T r (coarse Dirichlet rows zeroed) bitwise; structure
properties on a second mesh."""
import numpy as np
import pytest

from paper_1709_06793_b200 import mesh as M
from paper_1709_06793_b200.device import shell_layout
from paper_1709_06793_b200.multigrid import (_coarse_surface_rows, _fine_surface_rows,
                                             _fine_volume_rows, prolongation_matrix)
from tests.conftest import golden


def test_prolongation_matches_reference_bitwise():
    g = golden("mg_small")
    cube = M.unit_cube_6()
    gc, gf = M.RefinedGrid(cube, 2), M.RefinedGrid(cube, 3)
    P = prolongation_matrix(gc, gf)
    assert np.array_equal(P @ g["prolong_in"], g["prolong"])
    r = P.T @ g["restrict_in"]
    r[gc.dirichlet_mask] = 0.0
    assert np.array_equal(r, g["restrict"])


@pytest.mark.parametrize("cfg,lvl", [("cube6", 4), ("kuhn48", 3)])
def test_device_transfer_tables_reproduce_P(cfg, lvl):
    """The tables the device kernels use (closed-form volume rows, surface
    rows of P, coarse surface rows of P^T) emulated on the host give P x
    and P^T x exactly as the assembled P (same sums in the same order)."""
    from tests.cases import case_mesh
    mesh = M.unit_cube_6() if cfg == "cube6" else case_mesh("c3")
    gc, gf = M.RefinedGrid(mesh, lvl - 1), M.RefinedGrid(mesh, lvl)
    P = prolongation_matrix(gc, gf)
    rng = np.random.default_rng(lvl)
    xc, xf = rng.normal(size=gc.n_nodes), rng.normal(size=gf.n_nodes)
    y = np.empty(gf.n_nodes)
    for t in range(gf.macro.n_elements):
        lo, hi, odd = _fine_volume_rows(gc, gf, t)
        s0 = gf.vol_start[t]
        y[s0:s0 + gf.nodes_per_volume] = np.where(odd, 0.5 * xc[lo] + 0.5 * xc[hi], xc[lo])
    _, pos, _ = shell_layout(gf.n)
    rows, lo, hi, odd = _fine_surface_rows(gc, gf, gf.elem_gidx[:, pos], pos)
    y[rows] = np.where(odd, 0.5 * xc[lo] + 0.5 * xc[hi], xc[lo])
    assert np.array_equal(y, P @ xc)
    want = P.T @ xf
    _, cpos, _ = shell_layout(gc.n)
    rr, ptr, col, val = _coarse_surface_rows(gc, gf, gc.elem_gidx[:, cpos], cpos)
    for r in range(len(rr)):
        acc = 0.0
        for e in range(ptr[r], ptr[r + 1]):
            acc += val[e] * xf[col[e]]
        assert acc == want[rr[r]], r
    assert set(rr) == set(range(gc.n_surface_nodes))
