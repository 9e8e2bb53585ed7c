"""Smoother over more meshes, levels and variants than the golden cases:
GPU `Operator.smooth` (slot surface kernels, hyperplane-major whole-lattice
volume sweep from level 5, later sweeps reusing the skewed copies) against
the C oracle's lexicographic Gauss-Seidel (oracle/assemble.py: surface rows
from the independently assembled CSR, volume rows by the C restatement of
kernels.gs_scaling_3d / gs_nodal_3d), 1e-12 relative."""
import numpy as np
import pytest

from oracle.assemble import CpuOperator
from paper_1709_06793_b200 import mesh as M
from paper_1709_06793_b200 import Operator, RefinedGrid, sample_nodal
from tests.cases import k_c3

pytestmark = pytest.mark.gpu

CASES = [("cube6", lambda: M.unit_cube_6(), 6),
         ("blocks112", lambda: M.unit_cube_blocks(1, 1, 2), 5),
         ("blocks221", lambda: M.unit_cube_blocks(2, 2, 1), 5),
         ("simplex", lambda: M.reference_simplex(3), 7),
         ("kuhn48", lambda: M.unit_cube_blocks(2, 2, 2), 6)]


@pytest.mark.parametrize("tag,make,level", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("variant", ["scaling", "nodal"])
def test_smooth_matches_oracle(cuda, tag, make, level, variant):
    grid = RefinedGrid(make(), level)
    kf = sample_nodal(k_c3(), grid)
    rng = np.random.default_rng(level * 7 + len(tag))
    u0 = rng.uniform(-1, 1, grid.n_nodes)
    f = rng.uniform(-1, 1, grid.n_nodes)
    op = Operator(grid, variant, kf)
    assert op._skew_workspace() is not None
    sweeps, omega = (3, 1.0) if level == 6 else (2, 0.9)
    got = op.smooth(u0.copy(), f, sweeps=sweeps, omega=omega)
    want = CpuOperator(grid, variant, kf).smooth(u0.copy(), f, sweeps=sweeps, omega=omega)
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
