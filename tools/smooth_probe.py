import sys, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1709_06793_b200 import Operator, RefinedGrid, sample_nodal
from tests.cases import case_mesh, k_c3
g = RefinedGrid(case_mesh("c4"), 6)
kf = sample_nodal(k_c3(), g)
op = Operator(g, "scaling", kf)
u = torch.rand(g.n_nodes, dtype=torch.float64, device="cuda"); f = torch.rand_like(u)
op.smooth_device(u, f, 1); torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5): op.smooth_device(u, f, 1)
torch.cuda.synchronize(); print("sweep ms", (time.perf_counter() - t0) / 5 * 1e3)
