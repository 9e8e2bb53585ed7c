"""GPU multigrid / CG against the reference's solves (golden fixtures).

Transfers must be bitwise the reference's; solves must reproduce iteration
counts and residual histories (north star: "iteration counts and final
residuals must match").
"""
import numpy as np
import pytest

from tests.conftest import golden
from paper_1709_06793_b200 import mesh as M
from paper_1709_06793_b200.coefficients import cos3d
from paper_1709_06793_b200.multigrid import GridHierarchy, prolongation_matrix, solve, vcycle
from tests.cases import c2_error_norms, case_mesh, c4_field, k_c2

pytestmark = pytest.mark.gpu


def test_transfers_bitwise(cuda):
    g = golden("mg_small")
    hier = GridHierarchy(M.unit_cube_6(), 3, "scaling", cos3d(3), lmin=2)
    assert np.array_equal(hier.restrict(3, g["restrict_in"]), g["restrict"])
    assert np.array_equal(hier.prolongate(3, g["prolong_in"]), g["prolong"])


def test_prolongation_structure():
    cube = M.unit_cube_6()
    gc, gf = M.RefinedGrid(cube, 2), M.RefinedGrid(cube, 3)
    P = prolongation_matrix(gc, gf)
    assert P.shape == (gf.n_nodes, gc.n_nodes)
    nnz = np.diff(P.indptr)
    assert nnz.min() == 1 and nnz.max() == 2
    assert np.abs(P @ np.ones(gc.n_nodes) - 1.0).max() == 0.0
    aff = lambda x: 2.0 * x[:, 0] - 0.7 * x[:, 1] + 0.3 * x[:, 2] + 1.0
    assert np.abs(P @ aff(gc.node_coords) - aff(gf.node_coords)).max() < 1e-13


@pytest.mark.parametrize("variant", ["scaling", "nodal"])
def test_vcycle_solve_matches_reference(cuda, variant):
    g = golden("mg_small")
    hier = GridHierarchy(M.unit_cube_6(), 4, variant, cos3d(3))
    u, rep = solve(hier, g[f"{variant}_f"], stop="iters:8", pre=2, post=2)
    want = g[f"{variant}_res"]
    assert rep.iterations == len(want) - 1
    assert np.allclose(rep.residuals, want, rtol=1e-8, atol=0)
    assert np.abs(u - g[f"{variant}_u"]).max() <= 1e-9 * np.abs(u).max()
    assert rep.flops_add > 0


def test_drop_mode_with_coarse_lmin(cuda):
    g = golden("mg_small")
    hier = GridHierarchy(M.unit_cube_6(), 3, "scaling", cos3d(3), lmin=1)
    u, rep = solve(hier, g["drop_f"], stop="drop:1e-9", pre=3, post=3)
    want = g["drop_res"]
    assert rep.iterations == len(want) - 1
    assert rep.residuals[-1] <= 1e-9 * rep.residuals[0]
    assert np.allclose(rep.residuals, want, rtol=1e-7)
    assert not rep.diverged


def test_solver_edge_cases(cuda):
    cube = M.unit_cube_6()
    hier = GridHierarchy(cube, 3, "const")
    z = np.zeros(hier.grids[3].n_nodes)
    u = vcycle(hier, z.copy(), z)
    assert np.all(u == 0.0)
    with pytest.raises(ValueError, match="stop"):
        solve(hier, z, stop="until:tuesday")
    with pytest.raises(ValueError, match="coefficient"):
        GridHierarchy(cube, 2, "scaling")
    # over-relaxation beyond 2 diverges and is aborted
    hier = GridHierarchy(cube, 3, "const", omega=2.2)
    g = hier.grids[3]
    f = np.random.default_rng(1).normal(size=g.n_nodes)
    f[g.dirichlet_mask] = 0.0
    _, rep = solve(hier, f, stop="iters:50")
    assert rep.diverged and rep.iterations < 10


@pytest.mark.parametrize("variant", ["scaling", "nodal"])
def test_config2_cg_matches_reference(cuda, variant):
    """Config 2: unit cube (6 tets) level 6, CG to 1e-10 relative."""
    g = golden("c2_cg")
    lvl = 6
    hier = GridHierarchy(M.unit_cube_6(), lvl, variant, k_c2(), lmin=lvl, coarse_tol=1e-10)
    f = hier.torch.as_tensor(g["f"], device="cuda")
    rep = {}
    u = hier._cg_device(hier.ops[lvl], f, report=rep).cpu().numpy()
    assert rep["iterations"] == int(g[f"{variant}_iters"])
    grid = hier.grids[lvl]
    r = g["f"] - hier.ops[lvl].apply(u)
    r[grid.dirichlet_mask] = 0.0
    res = np.linalg.norm(r[grid.interior_ids])
    assert res <= 1.5e-10 * g[f"{variant}_b"]
    # final true residual: the iterates differ from the reference's only by
    # the summation order of surface rows / dots (1e-13 per apply); after
    # 292 iterations the measured final residuals agree to 0.13%
    # (tools/c2_probe.py: ratios 1.0013 scaling, 0.9992 nodal)
    assert abs(res - g[f"{variant}_res"]) <= 0.01 * g[f"{variant}_res"]
    assert np.abs(u[::97] - g[f"{variant}_u_sample"]).max() <= 1e-8 * np.abs(u).max()
    # discretisation errors against the reference's analysis.error_norms
    # (restated in tests/cases.py, pinned by tests/test_norms_golden.py)
    l2d, l2q, h1 = c2_error_norms(u, grid)
    assert abs(l2d - g[f"{variant}_l2d"]) <= 1e-6 * g[f"{variant}_l2d"]
    assert abs(l2q - g[f"{variant}_l2"]) <= 1e-6 * g[f"{variant}_l2"]
    assert abs(h1 - g[f"{variant}_h1"]) <= 1e-6 * g[f"{variant}_h1"]


@pytest.mark.slow
def test_config4_multigrid_matches_reference(cuda):
    """Config 4: 48 tets level 6, rough k, V(2,2) to a 1e-8 drop."""
    g = golden("c4_mg")
    lvl = 6
    hier = GridHierarchy(case_mesh("c4"), lvl, "scaling", c4_field())
    grid = hier.grids[lvl]
    f = np.random.default_rng(4).normal(size=grid.n_nodes)
    f[grid.dirichlet_mask] = 0.0
    u, rep = solve(hier, f, stop="drop:1e-8", pre=2, post=2)
    assert rep.iterations == int(g["iterations"])
    assert np.allclose(rep.residuals, g["residuals"], rtol=1e-6)
    assert abs(rep.rho - float(g["rho"])) <= 1e-6
    assert np.abs(u[::101] - g["u_sample"]).max() <= 1e-7 * np.abs(u).max()


def test_mg_preconditioned_cg_config4_like(cuda):
    """BASELINE config 4 names V(2,2)-preconditioned CG; the reference has
    none, so this pins the extension by its own contract:
    the true residual of the returned solution drops by 1e-8, faster than
    the stationary V-cycle the reference uses, from the same rough field."""
    from paper_1709_06793_b200.multigrid import pcg
    lvl = 5
    hier = GridHierarchy(case_mesh("c4"), lvl, "scaling", c4_field())
    grid = hier.grids[lvl]
    f = np.random.default_rng(4).normal(size=grid.n_nodes)
    f[grid.dirichlet_mask] = 0.0
    u, rep = pcg(hier, f, stop="drop:1e-8", pre=2, post=2)
    _, rep_mg = solve(hier, f, stop="drop:1e-8", pre=2, post=2)
    op = hier.ops[lvl]
    r = op.residual(u, f)
    r0 = op.residual(np.zeros_like(f), f)
    assert np.linalg.norm(r) <= 1.05e-8 * np.linalg.norm(r0)
    assert rep.iterations < rep_mg.iterations
    assert rep.residuals[-1] <= 1e-8 * rep.residuals[0]


def test_pcg_matches_reference_components(cuda):
    """PCG pinned against the same flexible-beta PCG written in numpy on the
    REFERENCE's Operator and vcycle (tests/golden/make_golden.py sec_pcg,
    config-4 mesh and field at L5): same iteration count, residual history
    within rtol 1e-6, solution samples within 1e-7."""
    from paper_1709_06793_b200.multigrid import pcg
    g = golden("pcg_c4")
    lvl = 5
    hier = GridHierarchy(case_mesh("c3"), lvl, "scaling", c4_field())
    grid = hier.grids[lvl]
    f = np.random.default_rng(4).normal(size=grid.n_nodes)
    f[grid.dirichlet_mask] = 0.0
    u, rep = pcg(hier, f, stop="drop:1e-8", pre=2, post=2)
    assert rep.iterations == int(g["iterations"])
    assert np.allclose(rep.residuals, g["residuals"], rtol=1e-6, atol=0)
    assert np.abs(u[::101] - g["u_sample"]).max() <= 1e-7 * np.abs(u).max()


@pytest.mark.parametrize("variant", ["scaling", "nodal"])
def test_vcycle_fixed_point(cuda, variant):
    """The discrete solution is a fixed point of the V-cycle (the reference's
    tests/test_multigrid.py:184-197 property): with f = A u*, one cycle from
    u* changes it by at most 1e-12."""
    hier = GridHierarchy(M.unit_cube_6(), 4, variant, cos3d(3))
    grid = hier.grids[4]
    op = hier.ops[4]
    rng = np.random.default_rng(11)
    ustar = rng.uniform(-1, 1, grid.n_nodes)
    ustar[grid.dirichlet_mask] = 0.0
    f = op.apply(ustar)
    u = ustar.copy()
    vcycle(hier, u, f, pre=2, post=2)
    assert np.abs(u - ustar).max() <= 1e-12 * np.abs(ustar).max()


def test_sharded_cg_device_path_world1(cuda):
    """sharded_cg on CUDA vectors (fused update kernel, owner-masked device
    dots, all-reduce of device scalars) on a world-1 group: the same
    iterates as the single-domain device CG, hence the same iteration
    count and solution."""
    import socket
    import torch.distributed as dist
    from paper_1709_06793_b200.shard import InterfaceMap, ShardedOperator, sharded_cg
    torch = cuda
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                            world_size=1)
    try:
        lvl = 4
        hier = GridHierarchy(M.unit_cube_6(), lvl, "scaling", k_c2(), lmin=lvl, coarse_tol=1e-10)
        grid = hier.grids[lvl]
        op = hier.ops[lvl]
        f = np.random.default_rng(3).normal(size=grid.n_nodes)
        f[grid.dirichlet_mask] = 0.0
        fd = torch.as_tensor(f, device="cuda")
        rep = {}
        want = hier._cg_device(op, fd, report=rep, graphs=False)
        sop = ShardedOperator(op, InterfaceMap(grid, 0, 1, 1.0), dist, grid.dirichlet_mask)
        x, its, res = sharded_cg(sop, fd, tol=1e-10)
        assert its == rep["iterations"]
        assert torch.equal(x, want)
    finally:
        dist.destroy_process_group()
