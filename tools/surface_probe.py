"""Time the surface + Dirichlet rows of one apply on the config-5 workload:
face-tiled (default), precomputed rows for every row, matrix-free two-pass."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1709_06793_b200 import Operator, RefinedGrid, sample_nodal  # noqa: E402
from paper_1709_06793_b200._lib import check, lib  # noqa: E402
from paper_1709_06793_b200.shard import slab_mesh  # noqa: E402
from tests.cases import k_c5  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 8
grid = RefinedGrid(slab_mesh(0, 1), level)
kf = sample_nodal(k_c5(), grid)
u = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, grid.n_nodes), device="cuda")
for mode in ("face-tiled", "csr", "matrix-free"):
    op = Operator(grid, "scaling", kf, surface_mode="face" if mode == "face-tiled" else mode)
    D = op._device()
    out = op.apply_device(u)
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        op._surface(D["grid"], D["surf"], 0, u, None, out, st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        op._surface(D["grid"], D["surf"], 0, u, None, out, st)
    e1.record()
    torch.cuda.synchronize()
    print(f"{mode:12s} surface + Dirichlet rows: {e0.elapsed_time(e1) / 20:.3f} ms "
          f"({len(D['surf'].st.rows)} rows, {D['surf'].st.inc_ptr[-1]} incidences)", flush=True)
    del op, D
    torch.cuda.empty_cache()
