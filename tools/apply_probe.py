"""Full device-resident apply on the config-5 workload (FMA default),
CUDA events over 30 applies after 5 warm-up: the bench step without the
rest of bench.py (quick A/B of launch-level changes)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1709_06793_b200 import Operator, RefinedGrid, sample_nodal  # noqa: E402
from paper_1709_06793_b200.shard import slab_mesh  # noqa: E402
from tests.cases import k_c5  # noqa: E402

grid = RefinedGrid(slab_mesh(0, 1), 8)
op = Operator(grid, "scaling", sample_nodal(k_c5(), grid), fast=True)
u = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, grid.n_nodes), device="cuda")
out = torch.empty_like(u)
for rep in range(3):
    for _ in range(5):
        op.apply_device(u, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(30):
        op.apply_device(u, out=out)
    e1.record()
    torch.cuda.synchronize()
    print(f"apply {e0.elapsed_time(e1) / 30:.4f} ms", flush=True)
