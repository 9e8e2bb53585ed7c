"""Host logic of the matrix-free surface rows, checked without a GPU.

A numpy emulation of `surface_kernel` (csrc/hhg_surface.cuh) built from the
exact tables the device receives (incidence lists, boundary classes,
one-sided partial stencils) must reproduce the reference's surface rows,
which the reference assembles element-wise into a CSR
(operators.py:329-365).  Also checks the level schedule of the surface
Gauss-Seidel against sequential order.
"""
import numpy as np
import pytest

from tests.conftest import golden
from paper_1709_06793_b200 import mesh as M
from paper_1709_06793_b200.coefficients import sample_nodal
from paper_1709_06793_b200.device import GridTables, SurfaceTables
from paper_1709_06793_b200.mesh import PrimitiveKind
from paper_1709_06793_b200.reference_stencils import (class_element_masks,
                                                     environment, partial_stencils)
from tests.cases import case_mesh, k_c1, k_c3, wiggle3d


def emulate_surface(grid, kf, u, nodal_kinds=frozenset(), const=None):
    gt = GridTables(grid, tile_rows=16)
    st = SurfaceTables(grid, gt, nodal_kinds)
    env = environment(3)
    parts = [partial_stencils(grid, t) for t in range(grid.macro.n_elements)]
    _, dir_inside = class_element_masks()
    nb = st.neighbour_gids()
    lat = grid.lat
    i = st.inc_code & 1023
    j = (st.inc_code >> 10) & 1023
    k = (st.inc_code >> 20) & 1023
    flat = lat.base[k, j] + i
    kvals = (np.full((grid.macro.n_elements, lat.size), const) if const is not None
             else kf.values)
    out = np.zeros(grid.n_nodes)
    row_of = np.repeat(np.arange(len(st.rows)), np.diff(st.inc_ptr))
    for e in range(len(st.inc_tet)):
        t, c = st.inc_tet[e], st.inc_cls[e]
        r = st.rows[row_of[e]]
        v0 = u[r]
        k0 = kvals[t, flat[e]]
        q_k = np.zeros(14)
        q_v = np.full(14, v0)
        for d in range(14):
            if dir_inside[c, d]:
                off = M.DIRS_3D[d]
                q_k[d] = kvals[t, lat.base[k[e] + off[2], j[e] + off[1]] + i[e] + off[0]]
                q_v[d] = u[nb[e, d]]
        if st.row_nodal[row_of[e]]:
            fac = parts[t][1][c]
            buf = np.zeros(55)
            buf[0] = k0
            buf[1:15] = q_k
            for dst, a, b in env.cse_schedule:
                buf[dst] = buf[a] + buf[b]
            part = 0.0
            for d in range(14):
                lo, hi = env.term_ptr[d], env.term_ptr[d + 1]
                s = sum(buf[env.cse_sums[env.term_elem[tt]]] * fac[tt] for tt in range(lo, hi))
                part += s * (q_v[d] - v0)
        else:
            sh = parts[t][0][c]
            part = sum((k0 + q_k[d]) * sh[d] * (q_v[d] - v0)
                       for d in range(14) if dir_inside[c, d])
        out[r] += part
    return out, st


CASES = [("cube6_l3", M.unit_cube_6, 3, wiggle3d, "scaling", frozenset()),
         ("cube6_l3", M.unit_cube_6, 3, wiggle3d, "nodal", frozenset(PrimitiveKind)),
         ("cube6_l3", M.unit_cube_6, 3, wiggle3d, "hybrid:wv+we",
          frozenset({PrimitiveKind.VERTEX, PrimitiveKind.EDGE})),
         ("cube12_l3", M.unit_cube_12, 3, wiggle3d, "scaling", frozenset()),
         ("kuhn48_l3", lambda: case_mesh("c3"), 3, k_c3(), "nodal", frozenset(PrimitiveKind))]


@pytest.mark.parametrize("tag,make,lvl,kfn,name,kinds", CASES)
def test_partial_stencil_rows_match_reference(tag, make, lvl, kfn, name, kinds):
    g = golden(tag)
    grid = M.RefinedGrid(make(), lvl)
    kf = sample_nodal(kfn, grid)
    out, st = emulate_surface(grid, kf, g["u"], kinds)
    want = g[f"apply_{name}"]
    rows = st.rows
    assert np.abs(out[rows] - want[rows]).max() <= 1e-13 * np.abs(want).max()


def test_partial_stencils_sum_to_full_stencil():
    # the one-sided stencils of the two sides of a face add up to the full
    # interior stencil when both sides are the same macro element shape
    grid = M.RefinedGrid(M.reference_simplex(3), 3)
    psh, pfac = partial_stencils(grid, 0)
    from paper_1709_06793_b200.reference_stencils import reference_stencil
    full = reference_stencil(grid, 0)[1] / 2.0
    # face classes: every direction's terms split between inside/outside
    inside, _ = class_element_masks()
    env = environment(3)
    for c in range(4):
        outside = np.zeros(14)
        from paper_1709_06793_b200.reference_stencils import environment_matrices
        E = grid.macro.vertices[grid.macro.elements[0]][1:] - grid.macro.vertices[0]
        _, mats = environment_matrices(E, 3)
        vals = mats[env.term_elem, 0, env.term_slot]
        for d in range(14):
            lo, hi = env.term_ptr[d], env.term_ptr[d + 1]
            outside[d] = vals[lo:hi][~inside[c][env.term_elem[lo:hi]]].sum() / 2.0
        assert np.allclose(psh[c] + outside, full, atol=1e-15)


def test_constant_coefficient_surface_rows_annihilate_constants():
    grid = M.RefinedGrid(case_mesh("c3"), 2)
    out, st = emulate_surface(grid, None, np.ones(grid.n_nodes), const=2.0)
    assert np.abs(out[st.rows]).max() < 1e-13


def test_gs_levels_respect_sequential_order():
    grid = M.RefinedGrid(M.unit_cube_12(), 3)
    gt = GridTables(grid, tile_rows=16)
    st = SurfaceTables(grid, gt)
    try:
        order, ptr, nlev = st.gs_levels()
    except Exception as exc:            # needs the host helper of libhhg_b200.so
        pytest.skip(f"libhhg_b200.so not available: {exc}")
    level = np.empty(len(st.rows), dtype=np.int64)
    for lv in range(nlev):
        level[order[ptr[lv]:ptr[lv + 1]]] = lv
    nb = st.neighbour_gids()
    row_of = np.repeat(np.arange(len(st.rows)), np.diff(st.inc_ptr))
    pos = {g: r for r, g in enumerate(st.rows)}
    for e in range(len(row_of)):
        r = row_of[e]
        for q in nb[e]:
            if q >= 0 and q in pos and pos[q] != r:
                if pos[q] < r:
                    assert level[pos[q]] < level[r]
    assert nlev >= 1
