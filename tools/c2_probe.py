"""Config-2 CG (unit cube, level 6, tol 1e-10): final true residual of the
device CG against the reference's (golden), to size the test tolerance."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1709_06793_b200 import mesh as M  # noqa: E402
from paper_1709_06793_b200.multigrid import GridHierarchy  # noqa: E402
from tests.cases import k_c2  # noqa: E402
from tests.conftest import golden  # noqa: E402

g = golden("c2_cg")
lvl = 6
for variant in ("scaling", "nodal"):
    hier = GridHierarchy(M.unit_cube_6(), lvl, variant, k_c2(), lmin=lvl, coarse_tol=1e-10)
    f = hier.torch.as_tensor(g["f"], device="cuda")
    rep = {}
    u = hier._cg_device(hier.ops[lvl], f, report=rep).cpu().numpy()
    grid = hier.grids[lvl]
    r = g["f"] - hier.ops[lvl].apply(u)
    r[grid.dirichlet_mask] = 0.0
    res = np.linalg.norm(r[grid.interior_ids])
    print(f"{variant}: iters {rep['iterations']} (ref {int(g[f'{variant}_iters'])}) "
          f"res {res:.6e} ref {float(g[f'{variant}_res']):.6e} ratio {res / g[f'{variant}_res']:.4f} "
          f"b {float(g[f'{variant}_b']):.6e}", flush=True)
