"""Tensor-coefficient (M = 6) operators: SURVEY.md §8(f) item 3.

CPU: the oracle's C tensor kernels against the reference's numba tensor
kernels (bitwise), the oracle operator against the reference's tensor
Operator goldens, the component splitting and SPD checks, and a numpy
emulation of the device surface rows built from the per-component partial
stencils.  GPU: the C ABI and the drop-in Operator / GridHierarchy against
the same goldens (volume rows bitwise, surface rows 1e-13, smoothing 1e-12).
"""
import ctypes

import numpy as np
import pytest

from tests.conftest import golden
from oracle import kernels as ok
from oracle.assemble import CpuOperator, assemble_global, rel_apply_err
from paper_1709_06793_b200 import mesh as M
from paper_1709_06793_b200.coefficients import (TENSOR_DIRS_3D, TensorCoefficient,
                                                catalog, tensor_decompose_3d)
from paper_1709_06793_b200.device import GridTables, SurfaceTables
from paper_1709_06793_b200.operators import Operator, parse_hybrid_set
from paper_1709_06793_b200.reference_stencils import (class_element_masks, environment,
                                                     partial_stencils,
                                                     tensor_component_coeffs)

TOL_SURF = 1e-13
SETS = [("tensor_cube6_l3", M.unit_cube_6, 3, "poly", ["scaling", "nodal", "hybrid:wv+we"]),
        ("tensor_cube6_l5", M.unit_cube_6, 5, "poly", ["scaling", "nodal"]),
        ("tensor_cyl_l3", lambda: M.cylinder_shell_box(nr=1, na=2, nz=2), 3, "cyl",
         ["scaling", "nodal"])]


def _K(name):
    if name == "poly":
        return catalog("tensor3d_poly")
    return catalog("cylinder_blend")[1]


def _vol(grid):
    return np.arange(grid.n_nodes) >= grid.n_surface_nodes


# -- CPU: oracle pins ----------------------------------------------------------

@pytest.mark.parametrize("n", [8, 16])
def test_oracle_tensor_kernels_bitwise_equal_numba(n):
    g = golden("tensor_kernels")
    p = lambda k: g[f"n{n}_{k}"]
    lat = M.SimplexLattice(3, n)
    env = environment(3)
    assert np.array_equal(ok.apply_scaling_tensor_3d(n, lat.base, p("v"), p("km"), p("shm")),
                          p("scaling"))
    tabs = (env.cse_schedule, env.cse_sums)
    assert np.array_equal(ok.apply_nodal_tensor_3d(n, lat.base, p("v"), p("km"), *tabs,
                                                   p("fac"), env.term_ptr, env.term_elem),
                          p("nodal"))
    u = p("v").copy()
    ok.gs_scaling_tensor_3d(n, lat.base, u, p("fv"), p("km"), p("shg"), 1.0)
    assert np.array_equal(u, p("gs_scaling"))
    u = p("v").copy()
    ok.gs_nodal_tensor_3d(n, lat.base, u, p("fv"), p("km"), *tabs, p("facg"), env.term_ptr,
                          env.term_elem, 0.9)
    assert np.array_equal(u, p("gs_nodal_w09"))


@pytest.mark.parametrize("tag,make,lvl,kname,variants", SETS[:1] + SETS[2:])
def test_oracle_tensor_operator_matches_reference(tag, make, lvl, kname, variants):
    g = golden(tag)
    grid = M.RefinedGrid(make(), lvl)
    K = TensorCoefficient(grid, _K(kname))
    vol = _vol(grid)
    for name in variants:
        hn, v = frozenset(), name
        if name.startswith("hybrid:"):
            hn, v = parse_hybrid_set(name.split(":", 1)[1]), "hybrid"
        out = CpuOperator(grid, v, K, hybrid_nodal=hn).apply(g["u"])
        want = g[f"apply_{name}"]
        if v != "hybrid":
            assert np.array_equal(out[vol], want[vol]), name
        assert np.abs(out - want).max() <= TOL_SURF * np.abs(want).max(), name
        A = assemble_global(grid, v, K, hn)
        assert rel_apply_err(want, A, g["u"], grid.dirichlet_mask) < 1e-13, name
    for var in ("scaling", "nodal"):
        u = g["u"].copy()
        CpuOperator(grid, var, K).smooth(u, g["f"], sweeps=1, omega=1.0)
        assert np.abs(u - g[f"smooth_{var}_w1"]).max() < 1e-12, var


def test_tensor_splitting_reconstructs_and_rejects():
    rng = np.random.default_rng(3)
    pts = rng.uniform(0, 1, (50, 3))
    Kfn = catalog("tensor3d_poly")
    comps = tensor_decompose_3d(Kfn)
    K = comps[0](pts)[:, None, None] * np.eye(3)
    for m in range(1, 6):
        c = np.asarray(TENSOR_DIRS_3D[m])
        K = K + comps[m](pts)[:, None, None] * np.outer(c, c)
    assert np.abs(K - Kfn(pts)).max() < 1e-13
    grid = M.RefinedGrid(M.unit_cube_6(), 1)
    tc = TensorCoefficient(grid, Kfn)
    assert tc.M == 6 and tc.packed().shape == (6, grid.lat.size, 6)
    assert np.array_equal(tc.packed()[2, :, 4], tc.fields[4].values[2])
    assert np.abs(tc.reconstruct(pts) - Kfn(pts)).max() < 1e-13

    def bad(p):
        out = np.zeros((len(p), 3, 3))
        out[:, 0, 0], out[:, 1, 1], out[:, 2, 2] = 1.0, -1.0, 1.0
        return out
    with pytest.raises(ValueError, match="positive definite"):
        TensorCoefficient(grid, bad)
    with pytest.raises(ValueError, match="safeguard"):
        Operator(M.RefinedGrid(M.unit_cube_6(), 2), "scaling_ma2",
                 TensorCoefficient(M.RefinedGrid(M.unit_cube_6(), 2), Kfn))


def test_cylinder_blend_tensor_matches_map():
    bmap, K_ref = catalog("cylinder_blend", material=False)
    rng = np.random.default_rng(5)
    ref = np.column_stack([rng.uniform(1.0, 2.0, 20), rng.uniform(0.2, 2.9, 20),
                           rng.uniform(0.0, 4.0, 20)])
    phys = bmap.inverse(ref)
    assert np.abs(bmap.phi(phys) - ref).max() < 1e-12
    assert np.abs(bmap.tensor(phys) - K_ref(ref)).max() < 1e-11


@pytest.mark.parametrize("form", ["scaling", "nodal"])
def test_tensor_surface_rows_emulated_from_partial_stencils(form):
    """numpy emulation of tensor_surface_fill_kernel + surface_csr_kernel
    from the exact host tables the device receives."""
    g = golden("tensor_cube6_l3")
    grid = M.RefinedGrid(M.unit_cube_6(), 3)
    K = TensorCoefficient(grid, _K("poly"))
    kinds = frozenset(M.PrimitiveKind) if form == "nodal" else frozenset()
    gt = GridTables(grid, tile_rows=16)
    st = SurfaceTables(grid, gt, kinds)
    env = environment(3)
    _, dir_inside = class_element_masks()
    cfs = tensor_component_coeffs(K.dirs, env.nshapes)
    parts = [[partial_stencils(grid, t, coeff=cf) for cf in cfs]
             for t in range(grid.macro.n_elements)]
    nb = st.neighbour_gids()
    lat = grid.lat
    i, j, k = st.inc_code & 1023, (st.inc_code >> 10) & 1023, (st.inc_code >> 20) & 1023
    u = g["u"]
    out = np.zeros(grid.n_nodes)
    row_of = np.repeat(np.arange(len(st.rows)), np.diff(st.inc_ptr))
    for e in range(len(st.inc_tet)):
        t, c, r = st.inc_tet[e], st.inc_cls[e], st.rows[row_of[e]]
        flat0 = lat.base[k[e], j[e]] + i[e]
        qs = {}
        for d in range(14):
            if dir_inside[c, d]:
                off = M.DIRS_3D[d]
                qs[d] = lat.base[k[e] + off[2], j[e] + off[1]] + i[e] + off[0]
        part = 0.0
        if form == "scaling":
            for d, q in qs.items():
                s = sum((K.fields[m].values[t][flat0] + K.fields[m].values[t][q])
                        * parts[t][m][0][c][d] for m in range(6))
                part += s * (u[nb[e, d]] - u[r])
        else:
            es = []
            for m in range(6):
                buf = np.zeros(55)
                kv = K.fields[m].values[t]
                buf[0] = kv[flat0]
                for d, q in qs.items():
                    buf[1 + d] = kv[q]
                for dst, a, b in env.cse_schedule:
                    buf[dst] = buf[a] + buf[b]
                es.append(buf[env.cse_sums])
            for d in qs:
                s = sum(es[m][env.term_elem[tt]] * parts[t][m][1][c][tt]
                        for tt in range(env.term_ptr[d], env.term_ptr[d + 1])
                        for m in range(6))
                part += s * (u[nb[e, d]] - u[r])
        out[r] += part
    want = g[f"apply_{form}"]
    rows = st.rows
    assert np.abs(out[rows] - want[rows]).max() <= TOL_SURF * np.abs(want).max()


# -- GPU ------------------------------------------------------------------------

def _dev(torch, a):
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda")


@pytest.mark.gpu
@pytest.mark.parametrize("n", [8, 16])
def test_gpu_tensor_element_abi_bitwise(cuda, n):
    from paper_1709_06793_b200._lib import check, lib
    torch = cuda
    g = golden("tensor_kernels")
    p = lambda k: g[f"n{n}_{k}"]
    env = environment(3)
    st = torch.cuda.current_stream().cuda_stream
    out = torch.empty(ok.nvol_of(n), dtype=torch.float64, device="cuda")
    v, km = _dev(torch, p("v")), _dev(torch, p("km"))
    check(lib.hhg_apply_scaling_tensor_3d(n, None, v.data_ptr(), km.data_ptr(), 6,
                                          _dev(torch, p("shm")).data_ptr(), out.data_ptr(),
                                          st))
    assert np.array_equal(out.cpu().numpy(), p("scaling"))
    tabs = [np.ascontiguousarray(a, dtype=np.int64) for a in
            (env.cse_schedule, env.cse_sums, env.term_ptr, env.term_elem)]
    ip = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
    check(lib.hhg_apply_nodal_tensor_3d(n, None, v.data_ptr(), km.data_ptr(), 6, ip(tabs[0]),
                                        40, ip(tabs[1]), _dev(torch, p("fac")).data_ptr(),
                                        ip(tabs[2]), ip(tabs[3]), out.data_ptr(), st))
    assert np.array_equal(out.cpu().numpy(), p("nodal"))
    fv = _dev(torch, p("fv"))
    u = _dev(torch, p("v").copy())
    check(lib.hhg_gs_scaling_tensor_3d(n, None, u.data_ptr(), fv.data_ptr(), km.data_ptr(), 6,
                                       _dev(torch, p("shg")).data_ptr(), 1.0, st))
    assert np.array_equal(u.cpu().numpy(), p("gs_scaling"))
    u = _dev(torch, p("v").copy())
    check(lib.hhg_gs_nodal_tensor_3d(n, None, u.data_ptr(), fv.data_ptr(), km.data_ptr(), 6,
                                     ip(tabs[0]), 40, ip(tabs[1]),
                                     _dev(torch, p("facg")).data_ptr(), ip(tabs[2]),
                                     ip(tabs[3]), 0.9, st))
    assert np.array_equal(u.cpu().numpy(), p("gs_nodal_w09"))
    assert lib.hhg_apply_scaling_tensor_3d(n, None, v.data_ptr(), km.data_ptr(), 5,
                                           None, out.data_ptr(), st) == -1


@pytest.mark.gpu
@pytest.mark.parametrize("tag,make,lvl,kname,variants", SETS)
def test_gpu_tensor_apply_matches_reference(cuda, tag, make, lvl, kname, variants):
    g = golden(tag)
    grid = M.RefinedGrid(make(), lvl)
    K = TensorCoefficient(grid, _K(kname))
    vol = _vol(grid)
    for name in variants:
        hn, v = frozenset(), name
        if name.startswith("hybrid:"):
            hn, v = parse_hybrid_set(name.split(":", 1)[1]), "hybrid"
        op = Operator(grid, v, K, hybrid_nodal=hn)
        out = op.apply(g["u"])
        want = g[f"apply_{name}"]
        assert np.array_equal(out[vol], want[vol]), f"{name}: volume rows not bitwise"
        assert np.array_equal(out[grid.dirichlet_mask], g["u"][grid.dirichlet_mask])
        err = np.abs(out - want).max() / np.abs(want).max()
        assert err <= TOL_SURF, f"{name}: rel err {err:.2e}"
        assert op.flops_add == 0 and op.flops_mul == 0     # no analytic tensor count


@pytest.mark.gpu
@pytest.mark.parametrize("tag,make,kname", [("tensor_cube6_l3", M.unit_cube_6, "poly"),
                                            ("tensor_cyl_l3",
                                             lambda: M.cylinder_shell_box(nr=1, na=2, nz=2),
                                             "cyl")])
def test_gpu_tensor_residual_stored_smooth(cuda, tag, make, kname):
    g = golden(tag)
    grid = M.RefinedGrid(make(), 3)
    K = TensorCoefficient(grid, _K(kname))
    vol = _vol(grid)
    for var in ("scaling", "nodal"):
        op = Operator(grid, var, K)
        r = op.residual(g["u"], g["f"])
        want = g[f"residual_{var}"]
        assert np.array_equal(r[vol], want[vol]), var
        assert np.all(r[grid.dirichlet_mask] == 0.0)
        assert np.abs(r - want).max() <= TOL_SURF * np.abs(want).max()
        stv = op.store_stencils()
        assert np.array_equal(stv.stencil_weights(1), g[f"weights_{var}_t1"]), var
        a = stv.apply(g["u"])
        assert np.array_equal(a[vol], g[f"stored_{var}"][vol]), var
        for key, sw, om in ((f"smooth_{var}_w1", 1, 1.0), (f"smooth_{var}_2sw_w08", 2, 0.8)):
            u = g["u"].copy()
            Operator(grid, var, K).smooth(u, g["f"], sweeps=sw, omega=om)
            assert np.abs(u - g[key]).max() < 1e-12, key
        u = g["u"].copy()
        stv.smooth(u, g["f"], sweeps=1, omega=1.0)
        assert np.abs(u - g[f"smooth_{var}_w1"]).max() < 1e-12


@pytest.mark.gpu
def test_gpu_tensor_vcycles_match_reference(cuda):
    from paper_1709_06793_b200.multigrid import GridHierarchy, solve
    g = golden("tensor_mg")
    hier = GridHierarchy(M.unit_cube_6(), 4, "scaling", catalog("tensor3d_poly"), tensor=True)
    u, rep = solve(hier, g["f"], stop="iters:6", pre=2, post=2)
    want = g["residuals"]
    assert len(rep.residuals) == len(want)
    assert np.allclose(rep.residuals, want, rtol=1e-8, atol=0)
    assert np.abs(u - g["u"]).max() <= 1e-9 * np.abs(g["u"]).max()
