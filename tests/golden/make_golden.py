"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py [section ...]

Every array written here is an output of `hhgscale` itself (numba kernels,
Operator, GridHierarchy, solve) on seeded inputs; the tests compare the
oracle and the CUDA path against them.  Inputs that the GPU box must
regenerate (meshes, coefficients, seeded vectors) are produced by code that
exists on both sides (numpy default_rng streams, the product's mesh
generators whose numbering tests/test_mesh_golden.py pins).
"""
from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

import hhgscale.kernels as kn                      # noqa: E402  (reference)
import hhgscale.mesh as RM                         # noqa: E402
from hhgscale.coefficients import sample_nodal as r_sample   # noqa: E402
from hhgscale.multigrid import GridHierarchy, solve          # noqa: E402
from hhgscale.operators import Operator as ROperator, parse_hybrid_set  # noqa: E402
from hhgscale.reference_stencils import environment as r_env  # noqa: E402

from paper_1709_06793_b200 import mesh as M        # noqa: E402
from tests.cases import (case_mesh, k_c1, k_c2, k_c3, k_c5, wiggle3d,  # noqa: E402
                         c4_field, checksum_weights)


def rmesh(m):
    """Reference MacroMesh with the product generator's vertices/elements."""
    return RM.MacroMesh(m.vertices.copy(), m.elements.copy())


def save(name, **arrays):
    np.savez_compressed(HERE / f"{name}.npz", **arrays)
    size = (HERE / f"{name}.npz").stat().st_size
    print(f"  wrote {name}.npz ({size / 1024:.1f} KiB)")


# ---------------------------------------------------------------------------
def sec_mesh():
    out = {}
    for tag, make, lvl in [("simplex_l3", lambda: M.reference_simplex(3), 3),
                           ("cube6_l2", M.unit_cube_6, 2), ("cube12_l2", M.unit_cube_12, 2),
                           ("kuhn48_l1", lambda: case_mesh("c3"), 1),
                           ("slab96_l1", lambda: case_mesh("c5"), 1)]:
        g = RM.RefinedGrid(rmesh(make()), lvl)
        out[f"{tag}_gidx"] = g.elem_gidx
        out[f"{tag}_dirichlet"] = g.dirichlet_mask
        out[f"{tag}_coords"] = g.node_coords
        out[f"{tag}_vol_start"] = g.vol_start
    save("mesh", **out)


def sec_kernels():
    """Kernel-level pins: the reference numba kernels on seeded lattices."""
    rng = np.random.default_rng(2024)
    env = r_env(3)
    out = {}
    for n in (8, 16):
        lat = RM.SimplexLattice(3, n)
        v = rng.uniform(-1, 1, lat.size)
        kc = rng.uniform(0.5, 3.0, lat.size)
        sh = rng.uniform(-0.3, 0.1, 14)
        fac = rng.uniform(-0.2, 0.2, 72)
        nv = (n - 1) * (n - 2) * (n - 3) // 6
        w = rng.uniform(-1, 1, (nv, 15))
        s = rng.uniform(-1, 1, 14)
        fv = rng.uniform(-1, 1, nv)
        o = {}
        o["v"], o["kc"], o["sh"], o["fac"], o["w"], o["s"], o["fv"] = v, kc, sh, fac, w, s, fv
        r = np.empty(nv); kn.apply_scaling_3d(n, lat.base, v, kc, sh, r); o["scaling"] = r
        r = np.empty(nv)
        kn.apply_nodal_3d(n, lat.base, v, kc, env.cse_schedule, env.cse_sums, fac,
                          env.term_ptr, env.term_elem, r)
        o["nodal"] = r
        r = np.empty(nv); kn.apply_const_3d(n, lat.base, v, s, -s.sum(), r); o["const"] = r
        r = np.empty(nv); kn.apply_stored_3d(n, lat.base, v, w, r); o["stored"] = r
        # GS needs a diagonally sensible stencil: negative-definite scaled rows
        shg = -np.abs(sh) - 0.05
        u = v.copy(); kn.gs_scaling_3d(n, lat.base, u, fv, kc, shg, 1.0); o["gs_scaling"] = u
        o["shg"] = shg
        u = v.copy(); kn.gs_scaling_3d(n, lat.base, u, fv, kc, shg, 0.8); o["gs_scaling_w08"] = u
        facg = -np.abs(fac) - 0.01
        u = v.copy()
        kn.gs_nodal_3d(n, lat.base, u, fv, kc, env.cse_schedule, env.cse_sums, facg,
                       env.term_ptr, env.term_elem, 1.0)
        o["gs_nodal"] = u
        o["facg"] = facg
        for key, val in o.items():
            out[f"n{n}_{key}"] = val
    # csr_gs on a small SPD matrix
    import scipy.sparse as sp
    A = sp.random(60, 60, density=0.1, random_state=3, format="csr")
    A = (A + A.T + sp.eye(60) * 8.0).tocsr()
    A.sum_duplicates()
    rows = np.arange(5, 55, dtype=np.int64)
    u = rng.normal(size=60)
    f = rng.normal(size=60)
    out["csr_indptr"], out["csr_indices"], out["csr_data"] = A.indptr, A.indices, A.data
    out["csr_rows"], out["csr_u0"], out["csr_f"] = rows, u.copy(), f
    kn.csr_gs(rows, A.indptr, A.indices, A.data, A.diagonal(), u, f, 0.9)
    out["csr_result"] = u
    save("kernels", **out)


def _apply_set(tag, mesh, level, kfn, seed, variants, extra=False):
    g = RM.RefinedGrid(rmesh(mesh), level)
    kf = r_sample(kfn, g)
    rng = np.random.default_rng(seed)
    u = rng.uniform(-1, 1, g.n_nodes)
    out = {"u": u}
    for v in variants:
        hn = frozenset()
        name = v
        if v.startswith("hybrid:"):
            hn = parse_hybrid_set(v.split(":", 1)[1])
            v = "hybrid"
        if v == "const":
            op = ROperator(g, "const", 2.5)
        else:
            op = ROperator(g, v, kf, hybrid_nodal=hn)
        out[f"apply_{name}"] = op.apply(u)
    if extra:
        f = rng.uniform(-1, 1, g.n_nodes)
        out["f"] = f
        op = ROperator(g, "scaling", kf)
        out["residual_scaling"] = op.residual(u, f)
        out["stored_scaling"] = op.store_stencils().apply(u)
        out["weights_t2"] = op.stencil_weights(2)
        for nm, var, om, sw in [("smooth_scaling_w1", "scaling", 1.0, 1),
                                ("smooth_scaling_w08", "scaling", 0.8, 1),
                                ("smooth_scaling_2sw", "scaling", 1.0, 2),
                                ("smooth_nodal_w1", "nodal", 1.0, 1)]:
            uu = u.copy()
            ROperator(g, var, kf).smooth(uu, f, sweeps=sw, omega=om)
            out[nm] = uu
    save(tag, **out)


def sec_applies():
    _apply_set("c1_simplex_l4", M.reference_simplex(3), 4, k_c1(), 0,
               ["scaling", "nodal"])
    _apply_set("cube6_l3", M.unit_cube_6(), 3, wiggle3d, 12,
               ["scaling", "nodal", "const", "hybrid:wv+we", "hybrid:w", "scaling_ma2"],
               extra=True)
    _apply_set("cube12_l3", M.unit_cube_12(), 3, wiggle3d, 13, ["scaling", "nodal"],
               extra=True)
    _apply_set("kuhn48_l3", case_mesh("c3"), 3, k_c3(), 14, ["scaling", "nodal"])
    _apply_set("cube6_l5", M.unit_cube_6(), 5, k_c2(), 15, ["scaling", "nodal"])


def sec_c3_checksums():
    """Config 3 (48 tets, L7): reference apply/residual summarised by
    size-independent checksums (the full vectors are 136 MB each)."""
    g = RM.RefinedGrid(rmesh(case_mesh("c3")), 7)
    kf = r_sample(k_c3(), g)
    rng = np.random.default_rng(3)
    u = rng.uniform(-1, 1, g.n_nodes)
    f = rng.uniform(-1, 1, g.n_nodes)
    t0 = time.time()
    op = ROperator(g, "scaling", kf)
    print("  c3 setup", time.time() - t0)
    out = {}
    w = checksum_weights(g.n_nodes)
    for nm, vec in [("apply", op.apply(u)), ("residual", op.residual(u, f))]:
        out[f"{nm}_sum"] = vec.sum()
        out[f"{nm}_sq"] = (vec * vec).sum()
        out[f"{nm}_w"] = vec @ w
        out[f"{nm}_sample"] = vec[::1009]
        out[f"{nm}_absmax"] = np.abs(vec).max()
    save("c3_checksums", **out)


def sec_c2_cg():
    """Config 2: CG to 1e-10 on unit_cube_6 L6, scaling and nodal."""
    from hhgscale import analysis as an
    import sympy as sy
    x, y, z = sy.symbols("x y z")
    u_e = sy.sin(sy.pi * x) * sy.sin(sy.pi * y) * sy.sin(sy.pi * z)
    k_e = 1 + sy.Rational(1, 2) * sy.exp(-(x ** 2 + y ** 2 + z ** 2))
    case = an._scalar_case("c2", (x, y, z), u_e, k_e, k_c2(), RM.unit_cube_6,
                           (np.zeros(3), np.ones(3)), {})
    lvl = 6
    g = RM.RefinedGrid(RM.unit_cube_6(), lvl)
    f, u0 = an.dirichlet_system(case, g, "interpolate_mass")
    out = {"f": f}
    for var in ("scaling", "nodal"):
        hier = GridHierarchy(RM.unit_cube_6(), lvl, var, k_c2(), lmin=lvl, coarse_tol=1e-10)
        op = hier.ops[lvl]
        count = {"n": 0}
        orig = op.apply

        def counted(v, _o=orig):
            count["n"] += 1
            return _o(v)
        op.apply = counted
        t0 = time.time()
        u = hier.coarse_solve(f)
        print(f"  c2 {var}: {count['n']} matvecs, {time.time() - t0:.1f}s")
        op.apply = orig
        r = f - orig(u)
        r[g.dirichlet_mask] = 0
        nr = an.error_norms(case, u, g, quad=True)
        out[f"{var}_iters"] = count["n"]
        out[f"{var}_res"] = np.linalg.norm(r[g.interior_ids])
        out[f"{var}_b"] = np.linalg.norm(f[g.interior_ids])
        out[f"{var}_l2"] = nr.l2_quad
        out[f"{var}_h1"] = nr.h1
        out[f"{var}_l2d"] = nr.l2_discrete
        out[f"{var}_u_sample"] = u[::97]
        out[f"{var}_u_norm"] = np.linalg.norm(u)
    save("c2_cg", **out)


def sec_norms():
    """analysis.error_norms (quad=True) of the config-2 manufactured case on
    a small grid, for a seeded perturbation of the exact interpolant: pins
    the test harness's restatement of the H1 / quadrature-L2 errors."""
    from hhgscale import analysis as an
    import sympy as sy
    x, y, z = sy.symbols("x y z")
    u_e = sy.sin(sy.pi * x) * sy.sin(sy.pi * y) * sy.sin(sy.pi * z)
    k_e = 1 + sy.Rational(1, 2) * sy.exp(-(x ** 2 + y ** 2 + z ** 2))
    case = an._scalar_case("c2", (x, y, z), u_e, k_e, k_c2(), RM.unit_cube_6,
                           (np.zeros(3), np.ones(3)), {})
    out = {}
    for lvl in (2, 3):
        g = RM.RefinedGrid(RM.unit_cube_6(), lvl)
        u = case.u(g.node_coords) + 1e-3 * np.random.default_rng(lvl).normal(size=g.n_nodes)
        nr = an.error_norms(case, u, g, quad=True)
        out[f"l{lvl}_u"] = u
        out[f"l{lvl}_l2"] = nr.l2_quad
        out[f"l{lvl}_h1"] = nr.h1
        out[f"l{lvl}_l2d"] = nr.l2_discrete
    save("norms", **out)


def sec_ma2_2d():
    """The reference's 2-D scaling kernels with the MA2 gray-edge selector
    (kernels.apply_scaling_2d / gs_scaling_2d): directions with g[d] set use
    the safeguarded coefficient kg instead of kc; seeded lattices, every
    gray pair."""
    out = {}
    rng = np.random.default_rng(22)
    for n in (8, 16):
        lat = RM.SimplexLattice(2, n)
        v = rng.uniform(-1, 1, lat.size)
        kc = rng.uniform(0.5, 3.0, lat.size)
        kg = rng.uniform(0.1, 1.0, lat.size)
        fv = rng.uniform(-1, 1, (n - 1) * (n - 2) // 2)
        h = rng.uniform(-1.0, 0.2, 3)
        sh = np.concatenate([h, h])
        out[f"n{n}_v"], out[f"n{n}_kc"], out[f"n{n}_kg"] = v, kc, kg
        out[f"n{n}_fv"], out[f"n{n}_sh"] = fv, sh
        for gp in (-1, 0, 1, 2):
            g = np.zeros(6, dtype=np.bool_)
            if gp >= 0:
                g[gp] = g[gp + 3] = True
            o = np.empty((n - 1) * (n - 2) // 2)
            kn.apply_scaling_2d(n, lat.base, v, kc, kg, g, sh, o)
            out[f"n{n}_g{gp}_apply"] = o
            for om in (1.0, 0.8):
                u = v.copy()
                kn.gs_scaling_2d(n, lat.base, u, fv, kc, kg, g, sh, om)
                out[f"n{n}_g{gp}_gs{int(om * 10)}"] = u
    save("ma2_2d", **out)


def sec_mg_small():
    """Multigrid V-cycles on small grids (fast pins of the solver loop)."""
    from hhgscale.coefficients import catalog
    out = {}
    cube = RM.unit_cube_6()
    for var in ("scaling", "nodal"):
        hier = GridHierarchy(cube, 4, var, catalog("cos3d", m=3))
        g = hier.grids[4]
        rng = np.random.default_rng(5)
        f = rng.normal(size=g.n_nodes)
        f[g.dirichlet_mask] = 0.0
        u, rep = solve(hier, f, stop="iters:8", pre=2, post=2)
        out[f"{var}_res"] = np.array(rep.residuals)
        out[f"{var}_u"] = u
        out[f"{var}_f"] = f
    hier = GridHierarchy(cube, 3, "scaling", catalog("cos3d", m=3), lmin=1)
    g = hier.grids[3]
    rng = np.random.default_rng(8)
    f = rng.normal(size=g.n_nodes)
    f[g.dirichlet_mask] = 0.0
    u, rep = solve(hier, f, stop="drop:1e-9", pre=3, post=3)
    out["drop_res"] = np.array(rep.residuals)
    out["drop_u"] = u
    out["drop_f"] = f
    # one V-cycle step by step for the transfer operators
    hier = GridHierarchy(cube, 3, "scaling", catalog("cos3d", m=3), lmin=2)
    r = np.random.default_rng(9).normal(size=hier.grids[3].n_nodes)
    out["restrict"] = hier.restrict(3, r)
    out["restrict_in"] = r
    ec = np.random.default_rng(10).normal(size=hier.grids[2].n_nodes)
    out["prolong"] = hier.prolongate(3, ec)
    out["prolong_in"] = ec
    save("mg_small", **out)


def sec_c4_mg():
    """Config 4: 48 tets, L6, rough k = clip(exp(g)), V(2,2) to drop 1e-8."""
    lvl = 6
    hier = GridHierarchy(rmesh(case_mesh("c3")), lvl, "scaling", c4_field())
    g = hier.grids[lvl]
    rng = np.random.default_rng(4)
    f = rng.normal(size=g.n_nodes)
    f[g.dirichlet_mask] = 0.0
    t0 = time.time()
    u, rep = solve(hier, f, stop="drop:1e-8", pre=2, post=2)
    print(f"  c4: {rep.iterations} cycles rho={rep.rho} {time.time() - t0:.1f}s")
    save("c4_mg", residuals=np.array(rep.residuals), iterations=rep.iterations,
         rho=np.nan if rep.rho is None else rep.rho, u_sample=u[::101],
         u_norm=np.linalg.norm(u))


def sec_pcg():
    """Multigrid-preconditioned CG (BASELINE config 4 names it; the
    reference has none): the flexible-beta PCG of our `multigrid.pcg`,
    written here in numpy on the REFERENCE's Operator (apply / residual) and
    `vcycle` (V(2,2) from a zero guess as the preconditioner), so the
    residual history pins our device PCG against the reference's pieces."""
    from hhgscale.multigrid import vcycle as r_vcycle
    lvl = 5
    hier = GridHierarchy(rmesh(case_mesh("c3")), lvl, "scaling", c4_field())
    g = hier.grids[lvl]
    op = hier.ops[lvl]
    rng = np.random.default_rng(4)
    f = rng.normal(size=g.n_nodes)
    f[g.dirichlet_mask] = 0.0
    hscale = 2.0 ** (-lvl * 3 / 2.0)
    x = np.zeros(g.n_nodes)
    r = op.residual(x, f)
    res = [hscale * float(np.linalg.norm(r))]
    target = 1e-8 * res[0]

    def precond(rr):
        return r_vcycle(hier, np.zeros(g.n_nodes), rr, None, 2, 2)

    z = precond(r)
    p = z.copy()
    rz = float(r @ z)
    for _ in range(200):
        Ap = op.apply(p)
        alpha = rz / float(p @ Ap)
        x = x + alpha * p
        r_new = r - alpha * Ap
        res.append(hscale * float(np.linalg.norm(r_new)))
        if res[-1] <= target:
            break
        z = precond(r_new)
        beta = float((r_new - r) @ z) / rz
        p = z + beta * p
        rz = float(r_new @ z)
        r = r_new
    print(f"  pcg: {len(res) - 1} iterations, residuals {res[0]:.3e} -> {res[-1]:.3e}")
    save("pcg_c4", residuals=np.array(res), iterations=len(res) - 1, u_sample=x[::101])


def sec_tensor():
    """Tensor-coefficient (M = 6) pins: the reference's tensor numba kernels
    on seeded lattices, tensor Operators (tensor3d_poly on the unit cube,
    cylinder_blend on the half-cylinder shell box) and a tensor V-cycle."""
    from hhgscale.coefficients import TensorCoefficient, catalog
    rng = np.random.default_rng(77)
    env = r_env(3)
    out = {}
    for n in (8, 16):
        lat = RM.SimplexLattice(3, n)
        nv = (n - 1) * (n - 2) * (n - 3) // 6
        v = rng.uniform(-1, 1, lat.size)
        km = np.ascontiguousarray(rng.uniform(0.2, 2.0, (6, lat.size)))
        shm = np.ascontiguousarray(rng.uniform(-0.3, 0.1, (6, 14)))
        fac = np.ascontiguousarray(rng.uniform(-0.2, 0.2, (6, 72)))
        fv = rng.uniform(-1, 1, nv)
        o = {"v": v, "km": km, "shm": shm, "fac": fac, "fv": fv}
        r = np.empty(nv); kn.apply_scaling_tensor_3d(n, lat.base, v, km, shm, r)
        o["scaling"] = r
        r = np.empty(nv)
        kn.apply_nodal_tensor_3d(n, lat.base, v, km, env.cse_schedule, env.cse_sums, fac,
                                 env.term_ptr, env.term_elem, r)
        o["nodal"] = r
        shg = np.ascontiguousarray(-np.abs(shm) - 0.05)
        facg = np.ascontiguousarray(-np.abs(fac) - 0.01)
        u = v.copy(); kn.gs_scaling_tensor_3d(n, lat.base, u, fv, km, shg, 1.0)
        o["gs_scaling"], o["shg"] = u, shg
        u = v.copy()
        kn.gs_nodal_tensor_3d(n, lat.base, u, fv, km, env.cse_schedule, env.cse_sums, facg,
                              env.term_ptr, env.term_elem, 0.9)
        o["gs_nodal_w09"], o["facg"] = u, facg
        for key, val in o.items():
            out[f"n{n}_{key}"] = val
    save("tensor_kernels", **out)

    def op_set(tag, mesh, level, Kfn, seed, variants, extra):
        g = RM.RefinedGrid(rmesh(mesh), level)
        K = TensorCoefficient(g, Kfn)
        r = np.random.default_rng(seed)
        u = r.uniform(-1, 1, g.n_nodes)
        f = r.uniform(-1, 1, g.n_nodes)
        res = {"u": u, "f": f}
        for v in variants:
            hn = frozenset()
            name = v
            if v.startswith("hybrid:"):
                hn = parse_hybrid_set(v.split(":", 1)[1])
                v = "hybrid"
            res[f"apply_{name}"] = ROperator(g, v, K, hybrid_nodal=hn).apply(u)
        if extra:
            for var in ("scaling", "nodal"):
                op = ROperator(g, var, K)
                res[f"residual_{var}"] = op.residual(u, f)
                res[f"stored_{var}"] = op.store_stencils().apply(u)
                res[f"weights_{var}_t1"] = op.stencil_weights(1)
                uu = u.copy()
                op.smooth(uu, f, sweeps=1, omega=1.0)
                res[f"smooth_{var}_w1"] = uu
                uu = u.copy()
                op.smooth(uu, f, sweeps=2, omega=0.8)
                res[f"smooth_{var}_2sw_w08"] = uu
        save(tag, **res)

    op_set("tensor_cube6_l3", M.unit_cube_6(), 3, catalog("tensor3d_poly"), 31,
           ["scaling", "nodal", "hybrid:wv+we"], True)
    op_set("tensor_cube6_l5", M.unit_cube_6(), 5, catalog("tensor3d_poly"), 32,
           ["scaling", "nodal"], False)
    _, K_cyl = catalog("cylinder_blend")
    op_set("tensor_cyl_l3", M.cylinder_shell_box(nr=1, na=2, nz=2), 3, K_cyl, 33,
           ["scaling", "nodal"], True)
    # tensor V(2,2) cycles (GridHierarchy(..., tensor=True), multigrid.py:117-119)
    hier = GridHierarchy(RM.unit_cube_6(), 4, "scaling", catalog("tensor3d_poly"), tensor=True)
    g = hier.grids[4]
    f = np.random.default_rng(34).normal(size=g.n_nodes)
    f[g.dirichlet_mask] = 0.0
    u, rep = solve(hier, f, stop="iters:6", pre=2, post=2)
    save("tensor_mg", f=f, residuals=np.array(rep.residuals), u=u)


def sec_coeff():
    """Coefficient sampling and the k_min safeguard field of the reference."""
    from hhgscale.coefficients import kmin_field as r_kmin
    out = {}
    for tag, mesh, lvl, kfn in [("cube6_l3", M.unit_cube_6(), 3, wiggle3d),
                                ("kuhn48_l2", case_mesh("c3"), 2, k_c3()),
                                ("simplex_l4", M.reference_simplex(3), 4, k_c1())]:
        g = RM.RefinedGrid(rmesh(mesh), lvl)
        kf = r_sample(kfn, g)
        out[f"{tag}_values"] = kf.values
        out[f"{tag}_kmin"] = r_kmin(kf).values
    save("coeff", **out)


def sec_ma2_marks():
    """The reference's 2-D scaling_ma2 set-up (operators.ma2_marks and the
    Operator's per-element selector inputs) on its two obtuse 2-D meshes
    with its 2-D catalog coefficients, plus the element kernels on those
    inputs (seeded element lattices)."""
    from hhgscale.coefficients import catalog
    from hhgscale.operators import ma2_marks as r_marks
    out = {}
    rng = np.random.default_rng(31)
    cases = [("square_sig", RM.obtuse_square(), 4, catalog("sigmoid2d")),
             ("square_sin", RM.obtuse_square(), 3, catalog("sin2d")),
             ("kite_sig", RM.obtuse_kite_band(), 4, catalog("sigmoid2d")),
             ("kite_sig5", RM.obtuse_kite_band(), 5, catalog("sigmoid2d"))]
    for tag, mesh, lvl, fn in cases:
        g = RM.RefinedGrid(mesh, lvl)
        kf = r_sample(fn, g)
        marked, gray, km = r_marks(g, kf)
        op = ROperator(g, "scaling_ma2", kf)
        assert np.array_equal(op.ma2_marked, marked)
        n = g.n
        L = (n + 1) * (n + 2) // 2
        ni = (n - 1) * (n - 2) // 2
        ne = mesh.n_elements
        u = rng.uniform(-1, 1, (ne, L))
        f = rng.uniform(-1, 1, (ne, ni))
        app = np.empty((ne, ni))
        gs = np.empty((ne, L))
        for t in range(ne):
            kn.apply_scaling_2d(n, g.lat.base, u[t], kf.values[t], op._kg[t], op._gmask[t],
                                op._sh[t], app[t])
            w = u[t].copy()
            kn.gs_scaling_2d(n, g.lat.base, w, f[t], kf.values[t], op._kg[t], op._gmask[t],
                             op._sh[t], 0.9)
            gs[t] = w
        out.update({f"{tag}_verts": mesh.vertices, f"{tag}_elems": mesh.elements,
                    f"{tag}_level": np.int64(lvl), f"{tag}_values": kf.values,
                    f"{tag}_marked": marked, f"{tag}_gray": gray, f"{tag}_kmin": km.values,
                    f"{tag}_sh": np.stack(op._sh), f"{tag}_kg": np.stack(op._kg),
                    f"{tag}_g": op._gmask, f"{tag}_u": u, f"{tag}_f": f,
                    f"{tag}_apply": app, f"{tag}_gs09": gs})
        print(f"  {tag}: marked {marked.tolist()} gray {gray.tolist()}")
    save("ma2_marks", **out)


SECTIONS = {"mesh": sec_mesh, "kernels": sec_kernels, "applies": sec_applies,
            "c3": sec_c3_checksums, "c2": sec_c2_cg, "mg": sec_mg_small, "c4": sec_c4_mg,
            "tensor": sec_tensor, "coeff": sec_coeff, "norms": sec_norms, "ma2_2d": sec_ma2_2d,
            "ma2_marks": sec_ma2_marks, "pcg": sec_pcg}

if __name__ == "__main__":
    for name in (sys.argv[1:] or list(SECTIONS)):
        print(name)
        SECTIONS[name]()
