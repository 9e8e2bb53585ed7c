"""Launch-shape variants of the Gauss-Seidel kernels are the same sweep.

* hyperplane-major volume sweep (gs_volume_skew_kernel, level >= 7): bitwise
  the C oracle's lexicographic sweep (kernels.py:510-600) from the GPU's own
  post-surface state, at the automatic CTAs-per-element choice and at forced
  ones (HHG_GS_CLUSTER_N, read once per process -> subprocesses);
* several sweeps in one call (later sweeps reuse the skewed f and interior)
  equal the same number of one-sweep calls, bitwise;
* surface rows: the level sweep from the level-ordered slots on one
  cluster or on a cooperative grid (gs_surface_slots_kernel) and the
  round-1 grid kernel give bitwise equal results.
"""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def check_skew_volume(variant: str, omega: float) -> None:
    from oracle import kernels as ok
    from oracle.assemble import CpuOperator
    from paper_1709_06793_b200 import Operator, RefinedGrid, sample_nodal
    from paper_1709_06793_b200.reference_stencils import environment
    from tests.cases import case_mesh, k_c1
    grid = RefinedGrid(case_mesh("c1"), 7)
    kf = sample_nodal(k_c1(), grid)
    rng = np.random.default_rng(7)
    u0 = rng.uniform(-1, 1, grid.n_nodes)
    f = rng.uniform(-1, 1, grid.n_nodes)
    op = Operator(grid, variant, kf)
    assert op._skew_workspace() is not None          # the hyperplane-major path
    u_gpu = op.smooth(u0.copy(), f, omega=omega)
    cpu = CpuOperator(grid, variant, kf)
    env = environment(3)
    u_mix = u0.copy()
    surf = np.arange(grid.n_nodes) < grid.n_surface_nodes
    u_mix[surf] = u_gpu[surf]
    n = grid.n
    for t in range(grid.macro.n_elements):
        uloc = np.ascontiguousarray(u_mix[grid.elem_gidx[t]])
        s0 = grid.vol_start[t]
        fv = f[s0:s0 + grid.nodes_per_volume]
        if variant == "scaling":
            ok.gs_scaling_3d(n, grid.lat.base, uloc, fv, kf.values[t], cpu.sh[t], omega)
        else:
            ok.gs_nodal_3d(n, grid.lat.base, uloc, fv, kf.values[t], env.cse_schedule,
                           env.cse_sums, cpu.fac[t], env.term_ptr, env.term_elem, omega)
        u_mix[s0:s0 + grid.nodes_per_volume] = uloc[cpu.vol_pos]
    vol = ~surf
    assert np.array_equal(u_gpu[vol], u_mix[vol])


def smooth_c3(out: str) -> None:
    from paper_1709_06793_b200 import Operator, RefinedGrid, sample_nodal
    from tests.cases import case_mesh, k_c3
    grid = RefinedGrid(case_mesh("c3"), 6)
    kf = sample_nodal(k_c3(), grid)
    rng = np.random.default_rng(3)
    u = rng.uniform(-1, 1, grid.n_nodes)
    f = rng.uniform(-1, 1, grid.n_nodes)
    Operator(grid, "scaling", kf).smooth(u, f, sweeps=2)
    np.save(out, u)


def _sub(code: str, **env) -> None:
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", f"import sys; sys.path.insert(0, {str(ROOT)!r}); "
                        + code], env=e, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]


@pytest.mark.parametrize("variant,omega", [("scaling", 1.0), ("nodal", 0.8)])
def test_skew_volume_sweep_bitwise_oracle(cuda, variant, omega):
    check_skew_volume(variant, omega)


@pytest.mark.parametrize("ctas", ["4", "5", "8"])
def test_skew_volume_sweep_cluster_sizes(cuda, ctas):
    _sub("from tests.test_gpu_gs_kernels import check_skew_volume; "
         "check_skew_volume('scaling', 0.9)", HHG_GS_CLUSTER_N=ctas)


def test_surface_sweep_forms_agree(cuda, tmp_path):
    # automatic choice, one cluster of 8 / 16 CTAs, grid, round-1 grid kernel
    outs = []
    for cl, legacy in (("-1", "0"), ("0", "0"), ("8", "0"), ("16", "0"), ("0", "1")):
        p = str(tmp_path / f"u{cl}{legacy}.npy")
        _sub(f"from tests.test_gpu_gs_kernels import smooth_c3; smooth_c3({p!r})",
             HHG_SURF_CLUSTER=cl, HHG_SURF_LEGACY=legacy)
        outs.append(np.load(p))
    for o in outs[1:]:
        assert np.array_equal(outs[0], o)


@pytest.mark.parametrize("variant", ["scaling", "nodal"])
def test_skew_multi_sweep_equals_single_sweeps(cuda, variant):
    from paper_1709_06793_b200 import Operator, RefinedGrid, sample_nodal
    from tests.cases import case_mesh, k_c3
    grid = RefinedGrid(case_mesh("c3"), 7)
    kf = sample_nodal(k_c3(), grid)
    op = Operator(grid, variant, kf)
    assert op._skew_workspace() is not None
    rng = np.random.default_rng(11)
    u0 = rng.uniform(-1, 1, grid.n_nodes)
    f = rng.uniform(-1, 1, grid.n_nodes)
    a = op.smooth(u0.copy(), f, sweeps=3, omega=0.9)
    b = u0.copy()
    for _ in range(3):
        op.smooth(b, f, sweeps=1, omega=0.9)
    assert np.array_equal(a, b)
