"""Relative time-to-solution scaling / nodal (the paper's Table 6/7 metric,
PAPER.md:1659-1707): V(3,3) multigrid to a 1e-8 residual drop on the 48-tet
Kuhn cube at level 6 with k = exp(x+y+z)/e, on one GPU (setup excluded)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1709_06793_b200.multigrid import GridHierarchy, solve  # noqa: E402
from tests.cases import case_mesh, k_c3  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 6
res = {}
for var in ("scaling", "nodal"):
    hier = GridHierarchy(case_mesh("c3"), level, var, k_c3())
    g = hier.grids[level]
    f = np.random.default_rng(6).normal(size=g.n_nodes)
    f[g.dirichlet_mask] = 0.0
    solve(hier, f, stop="iters:1", pre=3, post=3)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    u, rep = solve(hier, f, stop="drop:1e-8", pre=3, post=3)
    torch.cuda.synchronize()
    res[var] = (time.perf_counter() - t0, rep.iterations)
    print(var, f"{res[var][0]:.3f} s", rep.iterations, "cycles", flush=True)
print("relative tts scaling/nodal:", round(res["scaling"][0] / res["nodal"][0], 3))
