"""GPU parity of the drop-in Operator and of the per-element C ABI.

Volume rows must be BITWISE the reference's (the kernels reproduce the
numba operation order with explicit round-to-nearest fp64 ops); surface rows
(matrix-free one-sided stencils, a different summation order than the
reference's scipy CSR) within 1e-13 relative; everything within the
north-star tolerance 1e-12 relative.
"""
import ctypes

import numpy as np
import pytest

from tests.conftest import golden
from oracle import kernels as ok
from oracle.assemble import CpuOperator
from paper_1709_06793_b200 import mesh as M
from paper_1709_06793_b200 import Operator, parse_hybrid_set
from paper_1709_06793_b200._lib import lib, check
from paper_1709_06793_b200.coefficients import sample_nodal
from paper_1709_06793_b200.reference_stencils import environment
from tests.cases import case_mesh, checksum_weights, k_c1, k_c2, k_c3, wiggle3d

pytestmark = pytest.mark.gpu

TOL_SURF = 1e-13


def _dev(torch, a):
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda")


def _vol_mask(grid):
    return np.arange(grid.n_nodes) >= grid.n_surface_nodes


# -- per-element ABI (kernels.py signatures) ---------------------------------

@pytest.mark.parametrize("n", [8, 16])
def test_element_abi_bitwise(cuda, n):
    torch = cuda
    g = golden("kernels")
    p = lambda k: g[f"n{n}_{k}"]
    nv = ok.nvol_of(n)
    st = torch.cuda.current_stream().cuda_stream
    env = environment(3)
    out = torch.empty(nv, dtype=torch.float64, device="cuda")
    v, kc = _dev(torch, p("v")), _dev(torch, p("kc"))
    check(lib.hhg_apply_scaling_3d(n, None, v.data_ptr(), kc.data_ptr(),
                                   _dev(torch, p("sh")).data_ptr(), out.data_ptr(), st))
    assert np.array_equal(out.cpu().numpy(), p("scaling"))
    tabs = [np.ascontiguousarray(a, dtype=np.int64) for a in
            (env.cse_schedule, env.cse_sums, env.term_ptr, env.term_elem)]
    ip = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
    fac = _dev(torch, p("fac"))
    check(lib.hhg_apply_nodal_3d(n, None, v.data_ptr(), kc.data_ptr(), ip(tabs[0]), 40,
                                 ip(tabs[1]), fac.data_ptr(), ip(tabs[2]), ip(tabs[3]),
                                 out.data_ptr(), st))
    assert np.array_equal(out.cpu().numpy(), p("nodal"))
    s = p("s")
    s14 = _dev(torch, np.ascontiguousarray(s))          # 14 weights + c0 by value
    check(lib.hhg_apply_const_3d(n, None, v.data_ptr(), s14.data_ptr(), -s.sum(),
                                 out.data_ptr(), st))
    assert np.array_equal(out.cpu().numpy(), p("const"))
    # the c0 argument is the diagonal weight (not read from the array)
    check(lib.hhg_apply_const_3d(n, None, v.data_ptr(), s14.data_ptr(), 0.0,
                                 out.data_ptr(), st))
    assert np.array_equal(out.cpu().numpy(), ok.apply_const_3d(n, M.SimplexLattice(3, n).base,
                                                               p("v"), s, 0.0))
    w = _dev(torch, p("w"))
    check(lib.hhg_apply_stored_3d(n, None, v.data_ptr(), w.data_ptr(), out.data_ptr(), st))
    assert np.array_equal(out.cpu().numpy(), p("stored"))
    fv = _dev(torch, p("fv"))
    for key, om in (("gs_scaling", 1.0), ("gs_scaling_w08", 0.8)):
        u = _dev(torch, p("v").copy())
        check(lib.hhg_gs_scaling_3d(n, None, u.data_ptr(), fv.data_ptr(), kc.data_ptr(),
                                    _dev(torch, p("shg")).data_ptr(), om, st))
        assert np.array_equal(u.cpu().numpy(), p(key)), key
    u = _dev(torch, p("v").copy())
    check(lib.hhg_gs_nodal_3d(n, None, u.data_ptr(), fv.data_ptr(), kc.data_ptr(),
                              ip(tabs[0]), 40, ip(tabs[1]), _dev(torch, p("facg")).data_ptr(),
                              ip(tabs[2]), ip(tabs[3]), 1.0, st))
    assert np.array_equal(u.cpu().numpy(), p("gs_nodal"))
    bad = np.ascontiguousarray(tabs[0].copy())
    bad[0, 0] = 99
    assert lib.hhg_apply_nodal_3d(n, None, v.data_ptr(), kc.data_ptr(), ip(bad), 40,
                                  ip(tabs[1]), fac.data_ptr(), ip(tabs[2]), ip(tabs[3]),
                                  out.data_ptr(), st) == -4


# -- drop-in Operator vs the reference ------------------------------------------

APPLY_SETS = [
    ("c1_simplex_l4", lambda: M.reference_simplex(3), 4, k_c1(), ["scaling", "nodal"]),
    ("cube6_l3", M.unit_cube_6, 3, wiggle3d,
     ["scaling", "nodal", "const", "hybrid:wv+we", "hybrid:w", "scaling_ma2"]),
    ("cube12_l3", M.unit_cube_12, 3, wiggle3d, ["scaling", "nodal"]),
    ("kuhn48_l3", lambda: case_mesh("c3"), 3, k_c3(), ["scaling", "nodal"]),
    ("cube6_l5", M.unit_cube_6, 5, k_c2(), ["scaling", "nodal"]),
]


def _op(grid, kf, name):
    if name == "const":
        return Operator(grid, "const", 2.5)
    hn = frozenset()
    v = name
    if name.startswith("hybrid:"):
        hn, v = parse_hybrid_set(name.split(":", 1)[1]), "hybrid"
    if v == "scaling_ma2":
        with pytest.warns(RuntimeWarning, match="safeguard"):
            return Operator(grid, v, kf)
    return Operator(grid, v, kf, hybrid_nodal=hn)


@pytest.mark.parametrize("tag,make,lvl,kfn,variants", APPLY_SETS)
def test_apply_matches_reference(cuda, tag, make, lvl, kfn, variants):
    g = golden(tag)
    grid = M.RefinedGrid(make(), lvl)
    kf = sample_nodal(kfn, grid)
    u = g["u"]
    vol = _vol_mask(grid)
    for name in variants:
        out = _op(grid, kf, name).apply(u)
        want = g[f"apply_{name}"]
        assert np.array_equal(out[vol], want[vol]), f"{name}: volume rows not bitwise"
        assert np.array_equal(out[grid.dirichlet_mask], u[grid.dirichlet_mask])
        err = np.abs(out - want).max() / np.abs(want).max()
        assert err <= TOL_SURF, f"{name}: rel err {err:.2e}"


@pytest.mark.parametrize("tag,make", [("cube6_l3", M.unit_cube_6),
                                      ("cube12_l3", M.unit_cube_12)])
def test_residual_stored_smooth_match_reference(cuda, tag, make):
    g = golden(tag)
    grid = M.RefinedGrid(make(), 3)
    kf = sample_nodal(wiggle3d, grid)
    op = Operator(grid, "scaling", kf)
    r = op.residual(g["u"], g["f"])
    want = g["residual_scaling"]
    vol = _vol_mask(grid)
    assert np.array_equal(r[vol], want[vol])
    assert np.all(r[grid.dirichlet_mask] == 0.0)
    assert np.abs(r - want).max() <= TOL_SURF * np.abs(want).max()
    st = op.store_stencils()
    assert st.variant == "stored" and st.source_variant == "scaling"
    assert np.array_equal(st.stencil_weights(2), g["weights_t2"])
    a = st.apply(g["u"])
    assert np.array_equal(a[vol], g["stored_scaling"][vol])
    assert np.abs(a - g["stored_scaling"]).max() <= TOL_SURF * np.abs(a).max()
    for nm, var, om, sw in [("smooth_scaling_w1", "scaling", 1.0, 1),
                            ("smooth_scaling_w08", "scaling", 0.8, 1),
                            ("smooth_scaling_2sw", "scaling", 1.0, 2),
                            ("smooth_nodal_w1", "nodal", 1.0, 1)]:
        u = g["u"].copy()
        ret = Operator(grid, var, kf).smooth(u, g["f"], sweeps=sw, omega=om)
        assert ret is u
        assert np.abs(u - g[nm]).max() < 1e-12, nm


def test_smooth_equals_oracle_gs_bitwise_on_volume(cuda):
    # with identical surface values the volume wavefront is bitwise the
    # lexicographic sweep: compare one sweep against the C oracle started
    # from the GPU's own post-surface state
    grid = M.RefinedGrid(case_mesh("c3"), 4)
    kf = sample_nodal(k_c3(), grid)
    rng = np.random.default_rng(1)
    u0 = rng.uniform(-1, 1, grid.n_nodes)
    f = rng.uniform(-1, 1, grid.n_nodes)
    u_gpu = Operator(grid, "scaling", kf).smooth(u0.copy(), f)
    cpu = CpuOperator(grid, "scaling", kf)
    u_cpu = cpu.smooth(u0.copy(), f)
    assert np.abs(u_gpu - u_cpu).max() < 1e-12
    # volume GS from identical shells is bitwise
    u_mix = u0.copy()
    surf = np.arange(grid.n_nodes) < grid.n_surface_nodes
    u_mix[surf] = u_gpu[surf]
    n = grid.n
    for t in range(grid.macro.n_elements):
        uloc = np.ascontiguousarray(u_mix[grid.elem_gidx[t]])
        s0 = grid.vol_start[t]
        ok.gs_scaling_3d(n, grid.lat.base, uloc, f[s0:s0 + grid.nodes_per_volume],
                         kf.values[t], cpu.sh[t], 1.0)
        u_mix[s0:s0 + grid.nodes_per_volume] = uloc[cpu.vol_pos]
    vol = ~surf
    assert np.array_equal(u_gpu[vol], u_mix[vol])


def test_device_tensor_path_and_errors(cuda):
    torch = cuda
    grid = M.RefinedGrid(M.unit_cube_6(), 4)
    kf = sample_nodal(wiggle3d, grid)
    op = Operator(grid, "scaling", kf)
    u = np.random.default_rng(3).normal(size=grid.n_nodes)
    host = op.apply(u)
    du = torch.as_tensor(u, device="cuda")
    dev = op.apply(du)
    assert isinstance(dev, torch.Tensor) and dev.is_cuda
    assert np.array_equal(dev.cpu().numpy(), host)
    with pytest.raises(ValueError, match="length"):
        op.apply(np.zeros(grid.n_nodes + 1))
    with pytest.raises(ValueError, match="unknown variant"):
        Operator(grid, "magic", kf)
    with pytest.raises(ValueError, match="positive"):
        Operator(grid, "const", -1.0)
    with pytest.raises(ValueError, match="sampled coefficient"):
        Operator(grid, "scaling", 3.0)
    with pytest.raises(ValueError, match="store_stencils"):
        Operator(grid, "stored", kf)
    op.apply(u)
    nvol = grid.nodes_per_volume * grid.macro.n_elements
    assert op.flops_add == 3 * 41 * nvol and op.flops_mul == 3 * 28 * nvol


@pytest.mark.parametrize("variant", ["scaling", "nodal"])
def test_fast_mode_within_tolerance(cuda, variant):
    """fast=True (FMA edge-flux scaling rows / FMA term sums of the nodal
    rows) stays within 1e-12 (max-norm relative) of the reference order,
    for apply and residual."""
    grid = M.RefinedGrid(case_mesh("c3"), 5)
    kf = sample_nodal(k_c3(), grid)
    rng = np.random.default_rng(4)
    u = rng.uniform(-1, 1, grid.n_nodes)
    f = rng.uniform(-1, 1, grid.n_nodes)
    ex, fa = Operator(grid, variant, kf), Operator(grid, variant, kf, fast=True)
    exact, fast = ex.apply(u), fa.apply(u)
    assert not np.array_equal(fast, exact)          # the FMA path really ran
    assert np.abs(fast - exact).max() <= 1e-12 * np.abs(exact).max()
    re, rf = ex.residual(u, f), fa.residual(u, f)
    assert np.abs(rf - re).max() <= 1e-12 * np.abs(re).max()


# -- config 3 at full size (48 macro elements, level 7, 1.7e7 nodes) -----------

@pytest.mark.slow
def test_config3_full_size_checksums(cuda):
    g = golden("c3_checksums")
    grid = M.RefinedGrid(case_mesh("c3"), 7)
    kf = sample_nodal(k_c3(), grid)
    rng = np.random.default_rng(3)
    u = rng.uniform(-1, 1, grid.n_nodes)
    f = rng.uniform(-1, 1, grid.n_nodes)
    op = Operator(grid, "scaling", kf)
    w = checksum_weights(grid.n_nodes)
    for nm, vec in (("apply", op.apply(u)), ("residual", op.residual(u, f))):
        scale = g[f"{nm}_absmax"]
        assert np.abs(vec[::1009] - g[f"{nm}_sample"]).max() <= 1e-13 * scale
        assert abs(vec @ w - g[f"{nm}_w"]) <= 1e-12 * scale * np.sqrt(grid.n_nodes)
        assert abs(vec.sum() - g[f"{nm}_sum"]) <= 1e-12 * scale * np.sqrt(grid.n_nodes)
    # volume rows of every macro element bitwise against the C oracle
    out = op.apply(u)
    n = grid.n
    sh = op._sh
    nvol = grid.nodes_per_volume
    for t in range(grid.macro.n_elements):
        want = ok.apply_scaling_3d(n, grid.lat.base, u[grid.elem_gidx[t]], kf.values[t], sh[t])
        s0 = grid.vol_start[t]
        assert np.array_equal(out[s0:s0 + nvol], want), t


@pytest.mark.slow
def test_large_grid_algebraic_properties(cuda):
    """Size-independent properties at the per-GPU size of config 5 (96
    macro elements, level 8 would be 2.7e8 rows; level 7 keeps host setup
    short): constants in the kernel, linearity, symmetry on free nodes."""
    torch = cuda
    grid = M.RefinedGrid(case_mesh("c5"), 7)
    kf = sample_nodal(k_c1(), grid)
    op = Operator(grid, "scaling", kf)
    free = torch.as_tensor(~grid.dirichlet_mask, device="cuda")
    ones = torch.ones(grid.n_nodes, dtype=torch.float64, device="cuda")
    r = op.apply(ones)
    assert torch.where(free, r, 0).abs().max().item() < 1e-11
    gen = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand(grid.n_nodes, dtype=torch.float64, device="cuda", generator=gen) * free
    y = torch.rand(grid.n_nodes, dtype=torch.float64, device="cuda", generator=gen) * free
    Ax, Ay = op.apply(x), op.apply(y)
    Axy = op.apply(2.0 * x - 3.0 * y)
    assert (Axy - (2.0 * Ax - 3.0 * Ay)).abs().max().item() <= 1e-12 * Ax.abs().max().item()
    s1 = torch.dot(y, Ax * free).item()
    s2 = torch.dot(x, Ay * free).item()
    assert abs(s1 - s2) <= 1e-10 * abs(s1)
    # the smoother at full size (hyperplane-major whole-lattice sweep, one
    # wave of clusters, grid surface sweep): two sweeps, then the volume
    # rows of three elements re-swept by the C oracle from the GPU's own
    # state after the second surface sweep are bitwise the GPU's
    rng = np.random.default_rng(5)
    u = rng.uniform(-1, 1, grid.n_nodes)
    f = rng.uniform(-1, 1, grid.n_nodes)
    nvol = grid.nodes_per_volume
    df = torch.as_tensor(f, device="cuda")
    du = torch.as_tensor(u, device="cuda")
    op.smooth_device(du, df, sweeps=1)
    mid = du.clone()
    op.smooth_device(du, df, sweeps=1)
    after = du.cpu().numpy()
    surf = np.arange(grid.n_nodes) < grid.n_surface_nodes
    u_mix = mid.cpu().numpy()
    u_mix[surf] = after[surf]
    vol_pos = grid.lat.index(M.SimplexLattice(3, grid.n - 4).coords + 1)
    for t in (0, 47, 95):
        uloc = np.ascontiguousarray(u_mix[grid.elem_gidx[t]])
        s0 = int(grid.vol_start[t])
        ok.gs_scaling_3d(grid.n, grid.lat.base, uloc, f[s0:s0 + nvol], kf.values[t], op._sh[t],
                         1.0)
        assert np.array_equal(after[s0:s0 + nvol], uloc[vol_pos]), t


@pytest.mark.parametrize("name", ["scaling", "nodal", "hybrid:wv+we", "hybrid:wf"])
@pytest.mark.parametrize("cfg", ["c3", "c5"])
def test_surface_modes_agree_bitwise(cuda, name, cfg):
    """The three executions of the surface rows - face-tiled (default: face
    rows per macro face from static face-major layers, edge / vertex rows
    from the precomputed rows), precomputed rows for every row, and the
    matrix-free two-pass kernels - perform the same IEEE operations in the
    same order."""
    grid = M.RefinedGrid(case_mesh(cfg), 4)
    kf = sample_nodal(k_c3(), grid)
    hn, v = frozenset(), name
    if name.startswith("hybrid:"):
        hn, v = parse_hybrid_set(name.split(":", 1)[1]), "hybrid"
    u = np.random.default_rng(9).uniform(-1, 1, grid.n_nodes)
    f = np.random.default_rng(10).uniform(-1, 1, grid.n_nodes)
    a = Operator(grid, v, kf, hybrid_nodal=hn)                      # default: face-tiled
    ds = a._device()["surf"]
    assert ds.desc.nfaces > 0 and ds.desc.nsub < len(ds.st.rows)
    b = Operator(grid, v, kf, hybrid_nodal=hn, surface_mode="matrix-free")
    c = Operator(grid, v, kf, hybrid_nodal=hn, surface_mode="csr")  # every row precomputed
    assert c._device()["surf"].desc.nfaces == 0
    for x in (b, c):
        assert np.array_equal(a.apply(u), x.apply(u))
        assert np.array_equal(a.residual(u, f), x.residual(u, f))


def test_surface_first_side_stream_path(cuda):
    """The N > 1 path (ShardedOperator / bench.py): surface rows and the
    interface hook on a side stream concurrently with the volume kernel must
    give the same rows as the default order, for apply and residual."""
    torch = cuda
    grid = M.RefinedGrid(case_mesh("c3"), 4)
    kf = sample_nodal(k_c3(), grid)
    op = Operator(grid, "scaling", kf)
    rng = np.random.default_rng(3)
    u = torch.as_tensor(rng.uniform(-1, 1, grid.n_nodes), device="cuda")
    f = torch.as_tensor(rng.uniform(-1, 1, grid.n_nodes), device="cuda")
    calls = []

    def hook(out):
        calls.append(torch.cuda.current_stream().cuda_stream)
        out.mul_(1.0)                      # a device op on the hook's stream
    ref = op.apply_device(u).cpu().numpy()
    got = op.apply_device(u, after_surface=hook).cpu().numpy()
    assert np.array_equal(got, ref)
    assert calls and calls[0] != torch.cuda.current_stream().cuda_stream
    ref_r = op.apply_device(u, f=f).cpu().numpy()
    got_r = op.apply_device(u, f=f, after_surface=hook).cpu().numpy()
    assert np.array_equal(got_r, ref_r)


@pytest.mark.slow
def test_config5_full_size(cuda):
    """BASELINE config 5 at its full per-GPU size (96 macro elements, level 8,
    2.7e8 unknowns): constants are annihilated exactly on free rows, three
    elements' volume rows are bitwise the C oracle's, the operator is
    linear and symmetric on the free nodes, and the smoother's volume rows
    of three elements are bitwise the oracle's sweep from the same state."""
    from tests.cases import k_c5
    torch = cuda
    grid = M.RefinedGrid(case_mesh("c5"), 8)
    kf = sample_nodal(k_c5(), grid)
    op = Operator(grid, "scaling", kf)
    free = torch.as_tensor(~grid.dirichlet_mask, device="cuda")
    ones = torch.ones(grid.n_nodes, dtype=torch.float64, device="cuda")
    assert torch.where(free, op.apply(ones), 0).abs().max().item() == 0.0
    rng = np.random.default_rng(5)
    u = rng.uniform(-1, 1, grid.n_nodes)
    du = torch.as_tensor(u, device="cuda")
    out = op.apply(du)
    nvol = grid.nodes_per_volume
    for t in (0, 47, 95):
        want = ok.apply_scaling_3d(grid.n, grid.lat.base, u[grid.elem_gidx[t]], kf.values[t],
                                   op._sh[t])
        s0 = int(grid.vol_start[t])
        assert np.array_equal(out[s0:s0 + nvol].cpu().numpy(), want), t
    gen = torch.Generator(device="cuda").manual_seed(1)
    y = torch.rand(grid.n_nodes, dtype=torch.float64, device="cuda", generator=gen) * free
    x = du * free
    Ax, Ay = op.apply(x), op.apply(y)
    Axy = op.apply(2.0 * x - 3.0 * y)
    assert (Axy - (2.0 * Ax - 3.0 * Ay)).abs().max().item() <= 1e-12 * Ax.abs().max().item()
    s1 = torch.dot(y, Ax * free).item()
    s2 = torch.dot(x, Ay * free).item()
    assert abs(s1 - s2) <= 1e-10 * abs(s1)
    # the smoother at full size (hyperplane-major whole-lattice sweep, one
    # wave of clusters, grid surface sweep): two sweeps, then the volume
    # rows of three elements re-swept by the C oracle from the GPU's own
    # state after the second surface sweep are bitwise the GPU's
    rng = np.random.default_rng(5)
    u = rng.uniform(-1, 1, grid.n_nodes)
    f = rng.uniform(-1, 1, grid.n_nodes)
    nvol = grid.nodes_per_volume
    df = torch.as_tensor(f, device="cuda")
    du = torch.as_tensor(u, device="cuda")
    op.smooth_device(du, df, sweeps=1)
    mid = du.clone()
    op.smooth_device(du, df, sweeps=1)
    after = du.cpu().numpy()
    surf = np.arange(grid.n_nodes) < grid.n_surface_nodes
    u_mix = mid.cpu().numpy()
    u_mix[surf] = after[surf]
    vol_pos = grid.lat.index(M.SimplexLattice(3, grid.n - 4).coords + 1)
    for t in (0, 47, 95):
        uloc = np.ascontiguousarray(u_mix[grid.elem_gidx[t]])
        s0 = int(grid.vol_start[t])
        ok.gs_scaling_3d(grid.n, grid.lat.base, uloc, f[s0:s0 + nvol], kf.values[t], op._sh[t],
                         1.0)
        assert np.array_equal(after[s0:s0 + nvol], uloc[vol_pos]), t


@pytest.mark.parametrize("name", ["scaling", "nodal", "const", "hybrid:wv+we", "stored"])
def test_pinned_host_pipeline_equals_device_apply(cuda, name):
    """Operator.apply on a pinned CPU tensor runs the overlapped H2D /
    per-group volume kernels / D2H pipeline (the bench's e2e path); it must
    return exactly the device-resident apply."""
    torch = cuda
    grid = M.RefinedGrid(case_mesh("c3"), 4)
    kf = sample_nodal(k_c3(), grid)
    op = _op(grid, kf, "scaling" if name == "stored" else name)
    if name == "stored":
        op = op.store_stencils()
    u = np.random.default_rng(21).uniform(-1, 1, grid.n_nodes)
    host = torch.from_numpy(u).pin_memory()
    got = op.apply(host)
    assert got.device.type == "cpu" and got.is_pinned()
    want = op.apply_device(torch.as_tensor(u, device="cuda")).cpu().numpy()
    assert np.array_equal(got.numpy(), want)
    assert np.array_equal(op.apply(u), want)           # numpy in, numpy out
    # every call returns a fresh buffer (the pinned output was
    # recycled, so a second apply overwrote the first result)
    first = op.apply(u)
    second = op.apply(2.0 * u)
    assert np.array_equal(first, want)
    assert np.array_equal(second, op.apply_device(torch.as_tensor(2.0 * u, device="cuda"))
                          .cpu().numpy())
    # numpy residual through the same pipeline
    f = np.random.default_rng(22).uniform(-1, 1, grid.n_nodes)
    rw = op.apply_device(torch.as_tensor(u, device="cuda"),
                         f=torch.as_tensor(f, device="cuda")).cpu().numpy()
    assert np.array_equal(op.residual(u, f), rw)
    assert np.array_equal(op.residual(host, torch.from_numpy(f).pin_memory()).numpy(), rw)


@pytest.mark.parametrize("variant", ["scaling", "nodal", "hybrid:wv"])
def test_surface_matrix_S_matches_oracle(cuda, variant):
    """Operator._S (the reference's surface CSR, operators.py:329-365),
    built from the device-filled rows, equals the independently assembled
    shell-element matrix entrywise to 1e-13 and reproduces the surface rows
    of apply."""
    grid = M.RefinedGrid(case_mesh("c3"), 3)
    kf = sample_nodal(k_c3(), grid)
    op = _op(grid, kf, variant)
    want = CpuOperator(grid, op.variant, kf, hybrid_nodal=op.hybrid_nodal).S.tocsr()
    S = op._S
    assert S.shape == (grid.n_nodes, grid.n_nodes)
    diff = abs(S - want)
    assert diff.max() <= 1e-13 * abs(want).max()
    u = np.random.default_rng(5).uniform(-1, 1, grid.n_nodes)
    rows = np.nonzero(np.diff(S.indptr))[0]
    assert np.abs(S.dot(u)[rows] - op.apply(u)[rows]).max() <= 1e-13 * np.abs(u).max() * \
        abs(want).max() * 30


def test_constant_field_collapses_variants(cuda):
    """k = const makes scaling, nodal and scaling_ma2 the constant-coefficient
    operator (the reference's tests/test_oracle.py:37-43, in 3-D)."""
    grid = M.RefinedGrid(M.unit_cube_6(), 4)
    cval = 2.5
    kf = sample_nodal(lambda x: np.full(len(x), cval), grid)
    u = np.random.default_rng(8).normal(size=grid.n_nodes)
    ref = Operator(grid, "const", cval).apply(u)
    scale = np.abs(ref).max()
    for variant in ("scaling", "nodal", "scaling_ma2"):
        out = Operator(grid, variant, kf).apply(u)
        assert np.abs(out - ref).max() <= 1e-13 * scale, variant


@pytest.mark.parametrize("variant,lvl", [("nodal", 6), ("scaling", 6)])
def test_every_element_bitwise_against_oracle(cuda, variant, lvl):
    """Volume rows of all 48 elements of the config-3/4 mesh (several element
    orientations and shapes) against the C oracle, bitwise, and the
    residual's volume rows likewise."""
    grid = M.RefinedGrid(case_mesh("c3"), lvl)
    kf = sample_nodal(k_c3(), grid)
    op = Operator(grid, variant, kf)
    rng = np.random.default_rng(lvl)
    u = rng.uniform(-1, 1, grid.n_nodes)
    f = rng.uniform(-1, 1, grid.n_nodes)
    out = op.apply(u)
    res = op.residual(u, f)
    env = environment(3)
    nvol = grid.nodes_per_volume
    for t in range(grid.macro.n_elements):
        uloc = u[grid.elem_gidx[t]]
        if variant == "nodal":
            want = ok.apply_nodal_3d(grid.n, grid.lat.base, uloc, kf.values[t], env.cse_schedule,
                                     env.cse_sums, op._fac[t], env.term_ptr, env.term_elem)
        else:
            want = ok.apply_scaling_3d(grid.n, grid.lat.base, uloc, kf.values[t], op._sh[t])
        s0 = grid.vol_start[t]
        assert np.array_equal(out[s0:s0 + nvol], want), t
        assert np.array_equal(res[s0:s0 + nvol], f[s0:s0 + nvol] - want), t


def test_csr_gs_abi_bitwise(cuda):
    """hhg_csr_gs against the reference's kernels.csr_gs output (golden)."""
    torch = cuda
    g = golden("kernels")
    import scipy.sparse as sp
    A = sp.csr_matrix((g["csr_data"], g["csr_indices"], g["csr_indptr"]), shape=(60, 60))
    d = lambda a, dt=None: torch.as_tensor(np.ascontiguousarray(a, dtype=dt), device="cuda")
    # device copies kept alive until the kernels have run
    rows, ptr, idx = (d(g["csr_rows"], np.int64), d(A.indptr, np.int64),
                      d(A.indices, np.int64))
    data, diag, f = d(A.data), d(A.diagonal()), d(g["csr_f"])
    u = d(g["csr_u0"].copy())
    st = torch.cuda.current_stream().cuda_stream
    nr = len(g["csr_rows"])
    check(lib.hhg_csr_gs(nr, rows.data_ptr(), ptr.data_ptr(), idx.data_ptr(), data.data_ptr(),
                         diag.data_ptr(), u.data_ptr(), f.data_ptr(), 0.9, st))
    assert np.array_equal(u.cpu().numpy(), g["csr_result"])
    # a zero diagonal stops the sweep at that row and is reported
    zd = A.diagonal().copy()
    zd[g["csr_rows"][3]] = 0.0
    zdiag = d(zd)
    u = d(g["csr_u0"].copy())
    lib.hhg_status_reset()
    check(lib.hhg_csr_gs(nr, rows.data_ptr(), ptr.data_ptr(), idx.data_ptr(), data.data_ptr(),
                         zdiag.data_ptr(), u.data_ptr(), f.data_ptr(), 0.9, st))
    torch.cuda.synchronize()
    with pytest.raises(ValueError, match="zero central stencil entry"):
        check(lib.hhg_status())
    lib.hhg_status_reset()
    got = u.cpu().numpy()
    want = g["csr_u0"].copy()
    rows = g["csr_rows"][:3]
    ok.csr_gs(rows, A.indptr, A.indices, A.data, A.diagonal(), want, g["csr_f"], 0.9)
    assert np.array_equal(got, want)


# -- the FMA edge-flux path (fast=True: the bench's default arithmetic) ----
# Contract (BASELINE north star): within 1e-12 relative of the reference
# order, measured against max |A u| of the bitwise result.
TOL_FAST = 1e-12


def _fast_vs(exact, fast):
    return np.abs(fast - exact).max() / np.abs(exact).max()


def test_fast_config1_against_oracle(cuda):
    grid = M.RefinedGrid(case_mesh("c1"), 4)
    kf = sample_nodal(k_c1(), grid)
    u = np.random.default_rng(0).uniform(-1, 1, grid.n_nodes)
    want = CpuOperator(grid, "scaling", kf).apply(u)
    op = Operator(grid, "scaling", kf, fast=True)
    assert op._vol_flags() & 6 == 6            # the FMA mirror kernel
    assert _fast_vs(want, op.apply(u)) <= TOL_FAST
    f = np.random.default_rng(1).uniform(-1, 1, grid.n_nodes)
    assert _fast_vs(CpuOperator(grid, "scaling", kf).residual(u, f),
                    op.residual(u, f)) <= TOL_FAST


@pytest.mark.slow
@pytest.mark.parametrize("variant", ["scaling", "nodal"])
def test_fast_config3_full_size(cuda, variant):
    """Config 3 at full size (48 elements, level 7): the FMA path against
    the bitwise path (itself pinned by test_config3_full_size_checksums and
    the per-element oracle tests), apply and residual."""
    torch = cuda
    grid = M.RefinedGrid(case_mesh("c3"), 7)
    kf = sample_nodal(k_c3(), grid)
    rng = np.random.default_rng(17)
    u = torch.as_tensor(rng.uniform(-1, 1, grid.n_nodes), device="cuda")
    f = torch.as_tensor(rng.uniform(-1, 1, grid.n_nodes), device="cuda")
    exact, fast = Operator(grid, variant, kf), Operator(grid, variant, kf, fast=True)
    a, b = exact.apply(u), fast.apply(u)
    assert ((a - b).abs().max() / a.abs().max()).item() <= TOL_FAST
    a, b = exact.residual(u, f), fast.residual(u, f)
    assert ((a - b).abs().max() / a.abs().max()).item() <= TOL_FAST


@pytest.mark.slow
def test_fast_config5_elements(cuda):
    """Config 5 (96 elements, level 8): three elements' volume rows of the
    FMA path against the C oracle of the reference kernel."""
    from tests.cases import k_c5
    torch = cuda
    grid = M.RefinedGrid(case_mesh("c5"), 8)
    kf = sample_nodal(k_c5(), grid)
    op = Operator(grid, "scaling", kf, fast=True)
    u = np.random.default_rng(5).uniform(-1, 1, grid.n_nodes)
    out = op.apply(torch.as_tensor(u, device="cuda"))
    nvol = grid.nodes_per_volume
    for t in (0, 47, 95):
        want = ok.apply_scaling_3d(grid.n, grid.lat.base, u[grid.elem_gidx[t]], kf.values[t],
                                   op._sh[t])
        s0 = int(grid.vol_start[t])
        assert _fast_vs(want, out[s0:s0 + nvol].cpu().numpy()) <= TOL_FAST, t


@pytest.mark.parametrize("fast", [False, True])
def test_config5_slab_whole_vector_against_oracle(cuda, fast):
    """The config-5 mesh (96-element slab) at a reduced level, whole vector
    against the CPU operator (reference algorithm, independent assembly of
    the surface rows): volume rows bitwise (fast: 1e-12), surface rows
    1e-13, Dirichlet rows exact — apply and residual."""
    from tests.cases import k_c5
    grid = M.RefinedGrid(case_mesh("c5"), 5)
    kf = sample_nodal(k_c5(), grid)
    rng = np.random.default_rng(55)
    u = rng.uniform(-1, 1, grid.n_nodes)
    f = rng.uniform(-1, 1, grid.n_nodes)
    cpu = CpuOperator(grid, "scaling", kf)
    op = Operator(grid, "scaling", kf, fast=fast)
    vol = _vol_mask(grid)
    for got, want in ((op.apply(u), cpu.apply(u)), (op.residual(u, f), cpu.residual(u, f))):
        scale = np.abs(want).max()
        if fast:
            assert np.abs(got[vol] - want[vol]).max() <= TOL_FAST * scale
        else:
            assert np.array_equal(got[vol], want[vol])
        assert np.abs(got[~vol] - want[~vol]).max() <= TOL_SURF * scale
        d = grid.dirichlet_mask
        assert np.array_equal(got[d], want[d])


@pytest.mark.parametrize("cfg,variant,kw", [("c3", "scaling", {}), ("c3", "scaling", {"fast": True}),
                                            ("c5", "scaling", {"surface_mode": "csr"}),
                                            ("c3", "nodal", {}),
                                            ("c3", "scaling", {"surface_mode": "matrix-free"})])
def test_no_writes_outside_the_output(cuda, cfg, variant, kw):
    """Canary check in place of compute-sanitizer (closed on this GPU pool):
    the output vector is a view into a larger buffer whose guard bands hold
    NaN sentinels; apply, residual and a smoothing sweep must leave them
    untouched (and write every row: no NaN inside)."""
    torch = cuda
    grid = M.RefinedGrid(case_mesh(cfg), 4)
    kf = sample_nodal(k_c3(), grid)
    op = Operator(grid, variant, kf, **kw)
    n, pad = grid.n_nodes, 4096
    rng = np.random.default_rng(12)
    u = torch.as_tensor(rng.uniform(-1, 1, n), device="cuda")
    f = torch.as_tensor(rng.uniform(-1, 1, n), device="cuda")
    buf = torch.full((n + 2 * pad,), float("nan"), dtype=torch.float64, device="cuda")
    out = buf[pad:pad + n]
    for call in (lambda: op.apply_device(u, out=out), lambda: op.apply_device(u, out=out, f=f)):
        out.fill_(float("nan"))
        call()
        torch.cuda.synchronize()
        assert torch.isnan(buf[:pad]).all() and torch.isnan(buf[pad + n:]).all()
        assert not torch.isnan(out).any()
    ubuf = torch.full((n + 2 * pad,), float("nan"), dtype=torch.float64, device="cuda")
    uu = ubuf[pad:pad + n]
    uu.copy_(u)
    op.smooth_device(uu, f, sweeps=1)
    torch.cuda.synchronize()
    assert torch.isnan(ubuf[:pad]).all() and torch.isnan(ubuf[pad + n:]).all()
    assert not torch.isnan(uu).any()


def test_ma2_2d_kernels_bitwise(cuda):
    """The 2-D scaling kernels with the MA2 gray-edge selector
    (kernels.apply_scaling_2d / gs_scaling_2d) through the C ABI, against
    the reference's own outputs, for every gray pair."""
    torch = cuda
    g = golden("ma2_2d")
    st = torch.cuda.current_stream().cuda_stream
    for n in (8, 16):
        p = lambda k: g[f"n{n}_{k}"]
        v, kc, kg, sh, fv = (_dev(torch, p(k)) for k in ("v", "kc", "kg", "sh", "fv"))
        out = torch.empty((n - 1) * (n - 2) // 2, dtype=torch.float64, device="cuda")
        for gp in (-1, 0, 1, 2):
            sel = np.zeros(6, dtype=np.uint8)
            if gp >= 0:
                sel[gp] = sel[gp + 3] = 1
            check(lib.hhg_apply_scaling_2d(n, None, v.data_ptr(), kc.data_ptr(), kg.data_ptr(),
                                           sel.ctypes.data, sh.data_ptr(), out.data_ptr(), st))
            assert np.array_equal(out.cpu().numpy(), p(f"g{gp}_apply")), (n, gp)
            for om in (1.0, 0.8):
                u = _dev(torch, p("v").copy())
                check(lib.hhg_gs_scaling_2d(n, None, u.data_ptr(), fv.data_ptr(), kc.data_ptr(),
                                            kg.data_ptr(), sel.ctypes.data, sh.data_ptr(), om,
                                            st))
                assert np.array_equal(u.cpu().numpy(), p(f"g{gp}_gs{int(om * 10)}")), (n, gp)


@pytest.mark.parametrize("variant", ["scaling", "nodal"])
def test_device_stencil_dump_matches_host_restatement(cuda, variant):
    """store_stencils dumps every element's (centre, s_0..s_13) table on the
    device (hhg_dump_stencils); each equals the host restatement of the
    reference's dump kernel bitwise, and the stored twin applies exactly
    like the source operator's stencils."""
    grid = M.RefinedGrid(case_mesh("c3"), 4)
    kf = sample_nodal(k_c3(), grid)
    op = Operator(grid, variant, kf)
    st = op.store_stencils()
    assert st.bytes_required == grid.macro.n_elements * grid.nodes_per_volume * 15 * 8
    for t in (0, 17, 47):
        assert np.array_equal(st.stencil_weights(t), op.stencil_weights(t)), t
    u = np.random.default_rng(6).uniform(-1, 1, grid.n_nodes)
    vol = _vol_mask(grid)
    ref = np.empty(grid.nodes_per_volume * grid.macro.n_elements)
    out = st.apply(u)
    for t in range(grid.macro.n_elements):
        w = op.stencil_weights(t)
        uloc = u[grid.elem_gidx[t]]
        want = ok.apply_stored_3d(grid.n, grid.lat.base, uloc, w)
        s0 = grid.vol_start[t]
        assert np.array_equal(out[s0:s0 + grid.nodes_per_volume], want), t
