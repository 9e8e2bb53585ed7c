"""Kernel-time breakdown of one config-4 V(2,2) cycle (run under
`ncu --metrics gpu__time_duration.sum`): which kernels the multigrid solve
spends its device time in."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1709_06793_b200.multigrid import GridHierarchy, solve  # noqa: E402
from tests.cases import c4_field, case_mesh  # noqa: E402

hier = GridHierarchy(case_mesh("c4"), 6, "scaling", c4_field())
g = hier.grids[6]
f = np.random.default_rng(4).normal(size=g.n_nodes)
f[g.dirichlet_mask] = 0.0
solve(hier, f, stop="iters:1", pre=2, post=2)      # warm (tables, coarse inverse)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
solve(hier, f, stop="iters:1", pre=2, post=2)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("lmin", hier.lmin, "levels", sorted(hier.grids))
