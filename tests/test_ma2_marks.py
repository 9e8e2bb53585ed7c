"""2-D MA2 safeguard set-up (ma2.py) against the reference's own outputs
(tests/golden/ma2_marks.npz, make_golden.py sec_ma2_marks): the marking
(operators.py:88-129), the k_min field (coefficients.py:78-92) and the
per-element selector inputs of the reference Operator (operators.py:201-
220, reference_stencil / s/2 in 2-D) - all bitwise; and, on the GPU, the
element kernels fed with OUR inputs reproduce the reference kernels' rows
and Gauss-Seidel sweeps bitwise."""
import numpy as np
import pytest

from tests.conftest import golden
from paper_1709_06793_b200.mesh import MacroMesh
from paper_1709_06793_b200.ma2 import (Ma2Grid, apply_ma2_elements, classify_edge_types_2d,
                                       lambda_min, ma2_inputs, ma2_marks)

TAGS = ("square_sig", "square_sin", "kite_sig", "kite_sig5")


def _case(tag):
    g = golden("ma2_marks")
    p = lambda k: g[f"{tag}_{k}"]   # noqa: E731
    grid = Ma2Grid(MacroMesh(p("verts"), p("elems")), int(p("level")))
    return grid, p


@pytest.mark.parametrize("tag", TAGS)
def test_marks_kmin_and_selector_inputs_bitwise(tag):
    grid, p = _case(tag)
    marked, gray, km = ma2_marks(grid, p("values"))
    assert np.array_equal(marked, p("marked"))
    assert np.array_equal(gray, p("gray"))
    assert np.array_equal(km, p("kmin"))
    sh, kc, kg, g, _ = ma2_inputs(grid, p("values"))
    assert np.array_equal(sh, p("sh"))
    assert np.array_equal(kg, p("kg"))
    assert np.array_equal(g, p("g"))


def test_fixtures_cover_marked_unmarked_and_plain_elements():
    seen = set()
    for tag in TAGS:
        _, p = _case(tag)
        for m, gr in zip(p("marked"), p("gray")):
            seen.add(("marked" if m else "gray") if gr >= 0 else "plain")
    assert seen == {"marked", "gray", "plain"}


def test_obtuse_geometry_helpers():
    grid, _ = _case("square_sig")
    for t in range(grid.macro.n_elements):
        colors, s = classify_edge_types_2d(grid.macro, t, grid.level)
        # mirror pairs carry equal entries; gray iff positive
        assert np.array_equal(s[:3], s[3:])
        lam, _ = lambda_min(grid.macro.vertices[grid.macro.elements[t]])
        assert lam > 0
    with pytest.raises(ValueError, match="2D"):
        from paper_1709_06793_b200.mesh import reference_simplex
        Ma2Grid(reference_simplex(3), 2)


@pytest.mark.gpu
@pytest.mark.parametrize("tag", TAGS)
def test_ma2_element_kernels_on_our_inputs_bitwise(cuda, tag):
    grid, p = _case(tag)
    got = apply_ma2_elements(grid, p("values"), p("u"))
    assert np.array_equal(got, p("apply"))
    got = apply_ma2_elements(grid, p("values"), p("u"), omega=0.9, f_elem=p("f"))
    assert np.array_equal(got, p("gs09"))
