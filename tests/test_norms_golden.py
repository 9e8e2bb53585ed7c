"""The harness's error-norm restatement (tests/cases.c2_error_norms) against
the reference's analysis.error_norms on the config-2 manufactured case."""
import numpy as np
import pytest

from paper_1709_06793_b200 import mesh as M
from tests.cases import c2_error_norms
from tests.conftest import golden


@pytest.mark.parametrize("lvl", [2, 3])
def test_c2_error_norms_match_reference(lvl):
    g = golden("norms")
    grid = M.RefinedGrid(M.unit_cube_6(), lvl)
    l2d, l2, h1 = c2_error_norms(g[f"l{lvl}_u"], grid)
    assert l2d == pytest.approx(float(g[f"l{lvl}_l2d"]), rel=1e-13)
    assert l2 == pytest.approx(float(g[f"l{lvl}_l2"]), rel=1e-12)
    assert h1 == pytest.approx(float(g[f"l{lvl}_h1"]), rel=1e-12)
