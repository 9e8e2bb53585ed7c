"""Host-buffer apply (Operator.apply on a pinned CPU tensor, the e2e leg of
bench.py) for several element-group counts of the H2D / kernel / D2H
pipeline on the config-5 workload."""
import sys, time, statistics
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1709_06793_b200 import RefinedGrid, sample_nodal, Operator
from paper_1709_06793_b200.shard import slab_mesh
from tests.cases import k_c5
g = RefinedGrid(slab_mesh(0, 1), 8)
op = Operator(g, "scaling", sample_nodal(k_c5(), g))
u = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, g.n_nodes)).pin_memory()
for groups in (4, 8, 16, 32, 48):
    op._pipe = None
    op._pipeline(groups=groups)
    op.apply(u); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); op.apply(u); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print(groups, "groups: e2e ms", round(statistics.median(ts) * 1e3, 2), flush=True)
