"""Host numbering layer pinned to the reference (golden mesh.npz) and the
lattice/shell/tile bookkeeping the device kernels rely on."""
import numpy as np
import pytest

from tests.conftest import golden
from paper_1709_06793_b200 import mesh as M
from paper_1709_06793_b200.device import shell_layout, volume_tiles
from tests.cases import case_mesh

GRIDS = [("simplex_l3", lambda: M.reference_simplex(3), 3),
         ("cube6_l2", M.unit_cube_6, 2), ("cube12_l2", M.unit_cube_12, 2),
         ("kuhn48_l1", lambda: case_mesh("c3"), 1), ("slab96_l1", lambda: case_mesh("c5"), 1)]


@pytest.mark.parametrize("tag,make,lvl", GRIDS)
def test_numbering_matches_reference(tag, make, lvl):
    g = golden("mesh")
    grid = M.RefinedGrid(make(), lvl)
    assert np.array_equal(grid.elem_gidx, g[f"{tag}_gidx"])
    assert np.array_equal(grid.dirichlet_mask, g[f"{tag}_dirichlet"])
    assert np.array_equal(grid.node_coords, g[f"{tag}_coords"])     # bitwise
    assert np.array_equal(grid.vol_start, g[f"{tag}_vol_start"])


@pytest.mark.parametrize("n", [1, 2, 4, 8, 16, 32])
def test_lattice_base_closed_form(n):
    lat = M.SimplexLattice(3, n)
    for k in range(n + 1):
        for j in range(n + 1 - k):
            assert lat.base[k, j] == M.lattice_base(n, k, j)
    assert lat.size == M.lattice_size(n)
    assert np.array_equal(lat.index(lat.coords), np.arange(lat.size))


@pytest.mark.parametrize("n", [2, 4, 8, 16])
def test_shell_layout_covers_boundary_once(n):
    srow, pos, S = shell_layout(n)
    lat = M.SimplexLattice(3, n)
    c = lat.coords
    bary_zero = (c == 0).any(axis=1) | (c.sum(axis=1) == n)
    assert S == len(pos) == bary_zero.sum()
    assert set(pos.tolist()) == set(np.nonzero(bary_zero)[0].tolist())
    # srow addresses the first shell point of every row
    for k in range(n + 1):
        for j in range(n + 1 - k):
            assert pos[srow[k * (n + 1) + j]] == lat.base[k, j]


@pytest.mark.parametrize("n,rows", [(4, 16), (8, 16), (16, 16), (32, 16), (64, 4)])
def test_tiles_partition_volume_rows(n, rows):
    tiles = volume_tiles(n, 2, rows)
    seen = np.zeros((2, n, n, n), dtype=np.int64)
    for t, i0, j0, kmax in tiles:
        for k in range(1, kmax + 1):
            for j in range(j0, min(j0 + rows, n)):
                for i in range(i0, i0 + 32):
                    if i + j + k <= n - 1 and i >= 1 and j >= 1:
                        seen[t, i, j, k] += 1
    want = np.zeros_like(seen)
    for k in range(1, n):
        for j in range(1, n):
            for i in range(1, n):
                if i + j + k <= n - 1:
                    want[:, i, j, k] = 1
    assert np.array_equal(seen, want)
    for t in range(2):                                 # deep j-bands first
        assert np.all(np.diff(tiles[tiles[:, 0] == t, 2]) >= 0)


def test_volume_block_is_lattice_interior():
    g = M.RefinedGrid(M.unit_cube_6(), 3)
    n = g.n
    inner = M.SimplexLattice(3, n - 4).coords + 1
    pos = g.lat.index(inner)
    for t in range(g.macro.n_elements):
        assert np.array_equal(g.elem_gidx[t][pos],
                              g.vol_start[t] + np.arange(g.nodes_per_volume))


def test_orientation_and_errors():
    m = M.MacroMesh([(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)], [(1, 0, 2, 3)])
    assert np.all(m.signed_volumes() > 0)
    with pytest.raises(M.MeshFormatError, match="degenerate"):
        M.MacroMesh([(0, 0, 0), (1, 0, 0), (2, 0, 0), (0, 0, 1)], [(0, 1, 2, 3)])
    with pytest.raises(M.MeshFormatError, match="repeats"):
        M.MacroMesh([(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)], [(0, 1, 1, 3)])
    with pytest.raises(M.MeshFormatError, match="out of range"):
        M.MacroMesh([(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)], [(0, 1, 2, 7)])


def test_loader_roundtrip(tmp_path):
    text = "DIM 3\nVERTICES 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nELEMENTS 1\n0 1 2 3  # tet\n"
    m = M.load_macro_mesh(text)
    assert m.n_elements == 1 and m.boundary_face.all()
    with pytest.raises(M.MeshFormatError, match="trailing"):
        M.load_macro_mesh(text + "junk\n")


def test_generators():
    assert M.unit_cube_6().n_elements == 6
    assert M.unit_cube_12().n_elements == 12
    c3 = case_mesh("c3")
    assert c3.n_elements == 48 and len(c3.vertices) == 27
    assert np.isclose(c3.signed_volumes().sum(), 1.0)
    c5 = case_mesh("c5")
    assert c5.n_elements == 96
    g = M.RefinedGrid(M.unit_cube_12(), 0)
    assert (~g.dirichlet_mask).sum() == 1      # one interior macro vertex


@pytest.mark.parametrize("tag,make,lvl,kname", [
    ("cube6_l3", "unit_cube_6", 3, "wiggle"),
    ("kuhn48_l2", "c3", 2, "c3"),
    ("simplex_l4", "simplex", 4, "c1")])
def test_coefficient_sampling_and_kmin_bitwise(tag, make, lvl, kname):
    """sample_nodal and kmin_field (coefficients.py:47-92) reproduce the
    reference's lattice arrays bit for bit."""
    from paper_1709_06793_b200.coefficients import kmin_field, sample_nodal
    from tests.cases import case_mesh, k_c1, k_c3, wiggle3d
    g = golden("coeff")
    mesh = {"unit_cube_6": M.unit_cube_6, "c3": lambda: case_mesh("c3"),
            "simplex": lambda: M.reference_simplex(3)}[make]()
    kfn = {"wiggle": wiggle3d, "c3": k_c3(), "c1": k_c1()}[kname]
    grid = M.RefinedGrid(mesh, lvl)
    kf = sample_nodal(kfn, grid)
    assert np.array_equal(kf.values, g[f"{tag}_values"])
    assert np.array_equal(kmin_field(kf).values, g[f"{tag}_kmin"])


def test_classify_primitives_and_neighborhood():
    """mesh.classify_primitives / neighborhood (reference mesh.py:748-765):
    node counts per owner kind follow the refinement formulas; the stencil
    offsets of an interior node are the lattice directions through the
    element's edge vectors, mirror pairs opposite."""
    from paper_1709_06793_b200 import mesh as Mm
    grid = Mm.RefinedGrid(Mm.unit_cube_6(), 3)
    n, mm = grid.n, grid.macro
    counts = Mm.classify_primitives(grid)
    ne = len(np.unique(np.sort(np.asarray(mm.elements)[:, [[0, 1], [0, 2], [0, 3], [1, 2], [1, 3], [2, 3]]], axis=2).reshape(-1, 2), axis=0))
    assert counts["vertex"] == len(mm.vertices)
    assert counts["edge"] == ne * (n - 1)
    assert counts["volume"] == mm.n_elements * (n - 1) * (n - 2) * (n - 3) // 6
    assert sum(counts.values()) == grid.n_nodes
    for t in range(mm.n_elements):
        off = Mm.neighborhood(grid, t)
        assert off.shape == (14, 3)
        assert np.array_equal(off[:7], -off[7:])
        V = np.asarray(mm.vertices, dtype=float)[np.asarray(mm.elements[t])]
        assert np.allclose(off[0], (V[1] - V[0]) / n)
