"""Cost model: analytic counts, traffic table and the host replay of single
volume rows (the reference's costmodel.py:116-258 and its
tests/test_costmodel.py:60-80 - replayed values bitwise the kernels, every
row costs the analytic count)."""
import numpy as np
import pytest

from oracle.assemble import CpuOperator
from paper_1709_06793_b200 import Operator, RefinedGrid, sample_nodal
from paper_1709_06793_b200 import costmodel as cm
from tests.cases import case_mesh, k_c1, k_c3


@pytest.mark.parametrize("variant", ["scaling", "nodal", "hybrid", "scaling_ma2"])
def test_measured_count_equals_analytic(variant):
    grid = RefinedGrid(case_mesh("c1"), 4)
    op = Operator(grid, variant, sample_nodal(k_c1(), grid))
    base = {"hybrid": "scaling", "scaling_ma2": "scaling"}.get(variant, variant)
    assert cm.measured_count(op) == cm.analytic_count(base, 3)


def test_const_count_and_traffic_table():
    grid = RefinedGrid(case_mesh("c1"), 4)
    assert cm.measured_count(Operator(grid, "const", 2.0)) == cm.analytic_count("const", 3)
    rows = {r["variant"]: r for r in cm.traffic_table(1000)}
    assert rows["stored"]["bytes_optimistic"] == 120_000
    assert rows["scaling"]["bytes_optimistic"] == 112 + 8_000
    assert rows["nodal"]["bytes_pessimistic"] == 768 + 120_000


@pytest.mark.parametrize("variant", ["scaling", "nodal"])
def test_replay_bitwise_the_oracle_rows(variant):
    """Replayed rows of every element equal the pinned C oracle's rows (which
    are bitwise the reference's numba kernels, tests/test_oracle_golden.py)."""
    grid = RefinedGrid(case_mesh("c3"), 4)
    kf = sample_nodal(k_c3(), grid)
    u = np.random.default_rng(2).uniform(-1, 1, grid.n_nodes)
    op = Operator(grid, variant, kf)
    want = CpuOperator(grid, variant, kf).apply(u)
    rng = np.random.default_rng(3)
    for t in range(grid.macro.n_elements):
        for c in rng.choice(op._nvol, size=3, replace=False):
            val, cnt = cm.replay_node(op, u, t, int(c))
            assert val == want[grid.vol_start[t] + c], (t, c)


def test_replay_errors():
    grid = RefinedGrid(case_mesh("c1"), 1)
    op = Operator(grid, "scaling", sample_nodal(k_c1(), grid))
    with pytest.raises(ValueError, match="refine"):
        cm.measured_count(op)


@pytest.mark.gpu
def test_replay_bitwise_the_gpu_kernels(cuda):
    grid = RefinedGrid(case_mesh("c3"), 5)
    kf = sample_nodal(k_c3(), grid)
    u = np.random.default_rng(4).uniform(-1, 1, grid.n_nodes)
    rng = np.random.default_rng(5)
    for variant in ("scaling", "nodal"):
        op = Operator(grid, variant, kf)
        got = op.apply(u)
        for t in range(grid.macro.n_elements):
            for c in rng.choice(op._nvol, size=2, replace=False):
                assert cm.replay_node(op, u, t, int(c))[0] == got[grid.vol_start[t] + c]
