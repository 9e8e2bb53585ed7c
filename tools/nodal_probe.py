"""Time the nodal-integration volume kernel on a small workload."""
import sys, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1709_06793_b200 import Operator, RefinedGrid, sample_nodal, unit_cube_6
from tests.cases import k_c2
g = RefinedGrid(unit_cube_6(), 6)
kf = sample_nodal(k_c2(), g)
for var in ("scaling", "nodal"):
    op = Operator(g, var, kf)
    u = torch.rand(g.n_nodes, dtype=torch.float64, device="cuda")
    op.apply_device(u); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        op.apply_device(u)
    torch.cuda.synchronize()
    print(var, (time.perf_counter() - t0) / 20 * 1e3, "ms/apply")
