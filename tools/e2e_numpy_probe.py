"""End-to-end Operator.apply on host inputs at config 5: numpy in / numpy
out (staged through pinned buffers by host threads, pipelined with the
copies) against a pinned torch tensor in / pinned tensor out."""
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1709_06793_b200 import Operator, RefinedGrid, sample_nodal  # noqa: E402
from paper_1709_06793_b200.shard import slab_mesh  # noqa: E402
from tests.cases import k_c5  # noqa: E402

grid = RefinedGrid(slab_mesh(0, 1), int(sys.argv[1]) if len(sys.argv) > 1 else 8)
op = Operator(grid, "scaling", sample_nodal(k_c5(), grid), fast=True)
u = np.random.default_rng(0).uniform(-1, 1, grid.n_nodes)
pinned = torch.from_numpy(u).pin_memory()
for name, x in (("pinned tensor", pinned), ("numpy", u)):
    ts = []
    for i in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        y = op.apply(x)
        torch.cuda.synchronize()
        if i:
            ts.append((time.perf_counter() - t0) * 1e3)
        del y
    print(f"{name:14s} e2e {statistics.median(ts):8.2f} ms", flush=True)
