"""Kernel breakdown of one config-5 smoothing call (one sweep): run under
`ncu --metrics gpu__time_duration.sum` - the second call is the measured
one (the first builds the skewed k copy and the slot tables).

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        python tools/gs_breakdown.py [level]
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1709_06793_b200 import Operator, RefinedGrid, sample_nodal  # noqa: E402
from paper_1709_06793_b200.shard import slab_mesh  # noqa: E402
from tests.cases import k_c5  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 8
g = RefinedGrid(slab_mesh(0, 1), level)
op = Operator(g, "scaling", sample_nodal(k_c5(), g))
u = torch.rand(g.n_nodes, dtype=torch.float64, device="cuda")
f = torch.rand_like(u)
op.smooth_device(u, f, 1)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("measured")
op.smooth_device(u, f, 1)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("done")
