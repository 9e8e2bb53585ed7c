"""Edge cases of the drop-in API: grids without volume rows (levels 0-3 of
small meshes: the reference's `test_apply_no_volume_nodes`), a single macro
element, the maximum supported level, argument errors, and zero-diagonal
Gauss-Seidel rows.  CPU parts check the host logic; GPU parts compare the
CUDA path with the CPU oracle on the same inputs."""
import types

import numpy as np
import pytest

from oracle.assemble import CpuOperator
from paper_1709_06793_b200 import mesh as M
from paper_1709_06793_b200.coefficients import sample_nodal
from paper_1709_06793_b200.operators import MAX_LEVEL, Operator
from tests.cases import wiggle3d


def test_level_limit_is_reported():
    fake = types.SimpleNamespace(dim=3, level=MAX_LEVEL + 1)
    with pytest.raises(ValueError, match="maximum"):
        Operator(fake, "const")


def test_argument_errors_match_reference_messages():
    grid = M.RefinedGrid(M.unit_cube_6(), 2)
    kf = sample_nodal(wiggle3d, grid)
    with pytest.raises(ValueError, match="unknown variant"):
        Operator(grid, "bogus", kf)
    with pytest.raises(ValueError, match="store_stencils"):
        Operator(grid, "stored", kf)
    with pytest.raises(ValueError, match="positive"):
        Operator(grid, "const", -1.0)
    with pytest.raises(ValueError, match="sampled coefficient"):
        Operator(grid, "scaling", None)
    other = M.RefinedGrid(M.unit_cube_6(), 2)
    with pytest.raises(ValueError, match="different grid"):
        Operator(other, "scaling", kf)


CASES = [(M.unit_cube_6, 0), (M.unit_cube_6, 1), (M.unit_cube_6, 2),
         (lambda: M.reference_simplex(3), 2), (lambda: M.reference_simplex(3), 3),
         (M.unit_cube_12, 2)]


@pytest.mark.gpu
@pytest.mark.parametrize("make,lvl", CASES)
def test_gpu_small_grids_match_oracle(cuda, make, lvl):
    grid = M.RefinedGrid(make(), lvl)
    kf = sample_nodal(wiggle3d, grid)
    rng = np.random.default_rng(lvl)
    u = rng.uniform(-1, 1, grid.n_nodes)
    f = rng.uniform(-1, 1, grid.n_nodes)
    for var in ("scaling", "nodal"):
        op = Operator(grid, var, kf)
        ref = CpuOperator(grid, var, kf)
        want = ref.apply(u)
        out = op.apply(u)
        scale = max(np.abs(want).max(), 1e-300)
        assert np.abs(out - want).max() <= 1e-13 * scale, (var, lvl)
        r = op.residual(u, f)
        assert np.abs(r - ref.residual(u, f)).max() <= 1e-13 * max(np.abs(f).max(), scale)
        u1, u2 = u.copy(), u.copy()
        op.smooth(u1, f, sweeps=2, omega=0.9)
        ref.smooth(u2, f, sweeps=2, omega=0.9)
        assert np.abs(u1 - u2).max() <= 1e-12 * max(np.abs(u2).max(), 1.0), (var, lvl)
        w = op.stencil_weights(0)
        assert w.shape == (grid.nodes_per_volume, 15)


@pytest.mark.gpu
def test_gpu_zero_diagonal_raises(cuda):
    # k == 0 on one element makes its volume rows' diagonal vanish
    grid = M.RefinedGrid(M.unit_cube_6(), 4)
    vals = sample_nodal(wiggle3d, grid).values.copy()
    vals[2] = 0.0
    from paper_1709_06793_b200.coefficients import CoefficientField
    op = Operator(grid, "scaling", CoefficientField(grid, vals))
    u = np.zeros(grid.n_nodes)
    with pytest.raises(ValueError, match="zero central stencil entry"):
        op.smooth(u, np.ones(grid.n_nodes))


@pytest.mark.gpu
def test_gpu_single_element_level_limit(cuda):
    # the largest level the build supports on one macro element (n = 512:
    # 22.5 M lattice points) against the oracle's C kernel on a few rows
    from oracle import kernels as ok
    import torch
    from paper_1709_06793_b200._lib import check, lib
    n = 512
    lat = M.SimplexLattice(3, n)
    rng = np.random.default_rng(9)
    v = rng.uniform(-1, 1, lat.size)
    kc = rng.uniform(0.5, 2.0, lat.size)
    sh = rng.uniform(-0.3, 0.1, 14)
    dv, dk, ds = (torch.as_tensor(a, device="cuda") for a in (v, kc, sh))
    out = torch.empty(ok.nvol_of(n), dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    check(lib.hhg_apply_scaling_3d(n, None, dv.data_ptr(), dk.data_ptr(), ds.data_ptr(),
                                   out.data_ptr(), st))
    got = out.cpu().numpy()
    # every row against the oracle on the same lattice
    want = ok.apply_scaling_3d(n, lat.base, v, kc, sh)
    assert np.array_equal(got, want)
    assert lib.hhg_apply_scaling_3d(1024, None, dv.data_ptr(), dk.data_ptr(), ds.data_ptr(),
                                    out.data_ptr(), st) == -1
