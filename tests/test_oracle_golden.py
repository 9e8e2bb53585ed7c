"""Pin the CPU oracle to vectors produced by the reference itself.

The oracle (oracle/) is the checker of the CUDA path, so it is pinned first:
its C kernels must reproduce the numba kernels bit for bit, and its operator
restatement must reproduce Operator.apply / residual / smooth of the
reference on the golden grids (volume rows bitwise, surface rows to
1e-13 relative — they are assembled in a different summation order).
"""
import numpy as np
import pytest

from tests.conftest import golden
from oracle import kernels as ok
from oracle.assemble import CpuOperator, assemble_global, rel_apply_err
from paper_1709_06793_b200 import mesh as M
from paper_1709_06793_b200.coefficients import sample_nodal
from paper_1709_06793_b200.operators import parse_hybrid_set
from paper_1709_06793_b200.reference_stencils import environment
from tests.cases import case_mesh, k_c1, k_c2, k_c3, wiggle3d


@pytest.mark.parametrize("n", [8, 16])
def test_c_kernels_bitwise_equal_numba(n):
    g = golden("kernels")
    p = lambda k: g[f"n{n}_{k}"]
    lat = M.SimplexLattice(3, n)
    env = environment(3)
    assert np.array_equal(ok.apply_scaling_3d(n, lat.base, p("v"), p("kc"), p("sh")),
                          p("scaling"))
    assert np.array_equal(ok.apply_nodal_3d(n, lat.base, p("v"), p("kc"), env.cse_schedule,
                                            env.cse_sums, p("fac"), env.term_ptr,
                                            env.term_elem), p("nodal"))
    s = p("s")
    assert np.array_equal(ok.apply_const_3d(n, lat.base, p("v"), s, -s.sum()), p("const"))
    assert np.array_equal(ok.apply_stored_3d(n, lat.base, p("v"), p("w")), p("stored"))
    u = p("v").copy()
    ok.gs_scaling_3d(n, lat.base, u, p("fv"), p("kc"), p("shg"), 1.0)
    assert np.array_equal(u, p("gs_scaling"))
    u = p("v").copy()
    ok.gs_scaling_3d(n, lat.base, u, p("fv"), p("kc"), p("shg"), 0.8)
    assert np.array_equal(u, p("gs_scaling_w08"))
    u = p("v").copy()
    ok.gs_nodal_3d(n, lat.base, u, p("fv"), p("kc"), env.cse_schedule, env.cse_sums,
                   p("facg"), env.term_ptr, env.term_elem, 1.0)
    assert np.array_equal(u, p("gs_nodal"))


def test_c_csr_gs_bitwise():
    g = golden("kernels")
    import scipy.sparse as sp
    A = sp.csr_matrix((g["csr_data"], g["csr_indices"], g["csr_indptr"]), shape=(60, 60))
    u = g["csr_u0"].copy()
    ok.csr_gs(g["csr_rows"], A.indptr, A.indices, A.data, A.diagonal(), u, g["csr_f"], 0.9)
    assert np.array_equal(u, g["csr_result"])


def test_gs_zero_diagonal_raises():
    n = 8
    lat = M.SimplexLattice(3, n)
    u = np.ones(lat.size)
    with pytest.raises(ValueError, match="zero central"):
        ok.gs_scaling_3d(n, lat.base, u, np.zeros(35), np.ones(lat.size), np.zeros(14), 1.0)


APPLY_SETS = [
    ("c1_simplex_l4", lambda: M.reference_simplex(3), 4, k_c1(), ["scaling", "nodal"]),
    ("cube6_l3", M.unit_cube_6, 3, wiggle3d,
     ["scaling", "nodal", "const", "hybrid:wv+we", "hybrid:w", "scaling_ma2"]),
    ("cube12_l3", M.unit_cube_12, 3, wiggle3d, ["scaling", "nodal"]),
    ("kuhn48_l3", lambda: case_mesh("c3"), 3, k_c3(), ["scaling", "nodal"]),
]


def _cpu_op(grid, kf, name):
    hn = frozenset()
    v = name
    if name.startswith("hybrid:"):
        hn = parse_hybrid_set(name.split(":", 1)[1])
        v = "hybrid"
    if v == "scaling_ma2":
        v = "scaling"
    if v == "const":
        return CpuOperator(grid, "const", 2.5)
    return CpuOperator(grid, v, kf, hybrid_nodal=hn)


@pytest.mark.parametrize("tag,make,lvl,kfn,variants", APPLY_SETS)
def test_cpu_operator_matches_reference(tag, make, lvl, kfn, variants):
    g = golden(tag)
    grid = M.RefinedGrid(make(), lvl)
    kf = sample_nodal(kfn, grid)
    u = g["u"]
    vol = ~np.zeros(grid.n_nodes, dtype=bool)
    vol[:grid.n_surface_nodes] = False
    for name in variants:
        op = _cpu_op(grid, kf, name)
        out = op.apply(u)
        want = g[f"apply_{name}"]
        assert np.array_equal(out[vol], want[vol]), name           # volume: bitwise
        assert np.array_equal(out[grid.dirichlet_mask], want[grid.dirichlet_mask])
        assert np.abs(out - want).max() <= 1e-13 * np.abs(want).max(), name


def test_cpu_residual_and_smooth_match_reference():
    g = golden("cube6_l3")
    grid = M.RefinedGrid(M.unit_cube_6(), 3)
    kf = sample_nodal(wiggle3d, grid)
    op = CpuOperator(grid, "scaling", kf)
    r = op.residual(g["u"], g["f"])
    want = g["residual_scaling"]
    assert np.abs(r - want).max() <= 1e-13 * np.abs(want).max()
    for nm, var, om, sw in [("smooth_scaling_w1", "scaling", 1.0, 1),
                            ("smooth_scaling_w08", "scaling", 0.8, 1),
                            ("smooth_scaling_2sw", "scaling", 1.0, 2),
                            ("smooth_nodal_w1", "nodal", 1.0, 1)]:
        o = CpuOperator(grid, var, kf)
        u = g["u"].copy()
        o.smooth(u, g["f"], sweeps=sw, omega=om)
        assert np.abs(u - g[nm]).max() < 1e-12, nm


def test_assembled_oracle_matches_reference_apply():
    g = golden("cube12_l3")
    grid = M.RefinedGrid(M.unit_cube_12(), 3)
    kf = sample_nodal(wiggle3d, grid)
    for v in ("scaling", "nodal"):
        A = assemble_global(grid, v, kf)
        want = g[f"apply_{v}"]
        assert rel_apply_err(want, A, g["u"], grid.dirichlet_mask) < 1e-13


def test_assembled_oracle_structure():
    grid = M.RefinedGrid(M.unit_cube_6(), 3)
    kf = sample_nodal(wiggle3d, grid)
    for v in ("scaling", "nodal"):
        A = assemble_global(grid, v, kf)
        s = A.dot(np.ones(grid.n_nodes))
        s[grid.dirichlet_mask] = 0.0
        scale = np.abs(A.data).max()
        assert np.abs(s).max() < 1e-12 * scale                     # zero row sums
        R = assemble_global(grid, v, kf, reduced=True)
        assert abs(R - R.T).max() < 1e-12 * scale                  # symmetry


def test_c_ma2_2d_kernels_bitwise():
    """C restatement of the reference's 2-D scaling kernels with the MA2
    gray-edge selector against the reference's own outputs."""
    g = golden("ma2_2d")
    for n in (8, 16):
        base = np.array([j * (n + 1) - j * (j - 1) // 2 for j in range(n + 1)], dtype=np.int64)
        p = lambda k: g[f"n{n}_{k}"]
        for gp in (-1, 0, 1, 2):
            sel = np.zeros(6, dtype=bool)
            if gp >= 0:
                sel[gp] = sel[gp + 3] = True
            out = ok.apply_scaling_2d(n, base, p("v"), p("kc"), p("kg"), sel, p("sh"))
            assert np.array_equal(out, p(f"g{gp}_apply")), (n, gp)
            for om in (1.0, 0.8):
                u = p("v").copy()
                ok.gs_scaling_2d(n, base, u, p("fv"), p("kc"), p("kg"), sel, p("sh"), om)
                assert np.array_equal(u, p(f"g{gp}_gs{int(om * 10)}")), (n, gp, om)
