"""Wall time of the config-2 CG and config-4 multigrid solves on the GPU
(device-resident vectors; setup excluded), next to the reference numbers
recorded in the golden fixtures' generation log (SURVEY/BASELINE)."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1709_06793_b200 import mesh as M  # noqa: E402
from paper_1709_06793_b200.multigrid import GridHierarchy, solve  # noqa: E402
from tests.cases import c4_field, case_mesh, k_c2  # noqa: E402

out = {}
g = np.load(ROOT / "tests/golden/c2_cg.npz")
for var in ("scaling", "nodal"):
    hier = GridHierarchy(M.unit_cube_6(), 6, var, k_c2(), lmin=6, coarse_tol=1e-10)
    f = torch.as_tensor(g["f"], device="cuda")
    rep = {}
    hier._cg_device(hier.ops[6], f, max_iter=5)          # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hier._cg_device(hier.ops[6], f, report=rep)
    torch.cuda.synchronize()
    out[f"c2_cg_{var}"] = {"iters": rep["iterations"], "s": time.perf_counter() - t0}
    print(var, out[f"c2_cg_{var}"], flush=True)
t0 = time.perf_counter()
hier = GridHierarchy(case_mesh("c4"), 6, "scaling", c4_field())
setup = time.perf_counter() - t0
grid = hier.grids[6]
f = np.random.default_rng(4).normal(size=grid.n_nodes)
f[grid.dirichlet_mask] = 0.0
solve(hier, f, stop="iters:1", pre=2, post=2)           # warm (levels, coarse inverse)
torch.cuda.synchronize()
t0 = time.perf_counter()
u, rep = solve(hier, f, stop="drop:1e-8", pre=2, post=2)
torch.cuda.synchronize()
out["c4_mg"] = {"cycles": rep.iterations, "rho": rep.rho, "s": time.perf_counter() - t0,
                "setup_s": setup}
print(out["c4_mg"], flush=True)
# smoother sweep cost at the finest level
op = hier.ops[6]
du = torch.as_tensor(u, device="cuda")
df = torch.as_tensor(f, device="cuda")
op.smooth_device(du, df, 1)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    op.smooth_device(du, df, 1)
torch.cuda.synchronize()
out["c4_smooth_sweep_ms"] = (time.perf_counter() - t0) / 5 * 1e3
nlev = op._device()["surf"].gs_tables(op._device()["grid"])["nlev"]
out["c4_surface_gs_levels"] = nlev
print(json.dumps(out))
