"""Time one forward Gauss-Seidel sweep (surface levels + ghost refresh +
volume hyperplane wavefronts) and one apply on a given workload, with the
split between the surface and volume parts (CUDA events).

    python tools/smooth_probe.py [c4|c5] [level]
"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1709_06793_b200 import Operator, RefinedGrid, sample_nodal  # noqa: E402
from paper_1709_06793_b200._lib import check, lib  # noqa: E402
from paper_1709_06793_b200.shard import slab_mesh  # noqa: E402
from tests.cases import case_mesh, k_c3, k_c5  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "c4"
level = int(sys.argv[2]) if len(sys.argv) > 2 else 6
mesh = slab_mesh(0, 1) if case == "c5" else case_mesh("c3")
g = RefinedGrid(mesh, level)
kf = sample_nodal(k_c5() if case == "c5" else k_c3(), g)
op = Operator(g, "scaling", kf)
u = torch.rand(g.n_nodes, dtype=torch.float64, device="cuda")
f = torch.rand_like(u)
op.smooth_device(u, f, 1)
torch.cuda.synchronize()
reps = 3
t0 = time.perf_counter()
for _ in range(reps):
    op.smooth_device(u, f, 1)
torch.cuda.synchronize()
sweep = (time.perf_counter() - t0) / reps * 1e3
# split: surface part alone
D = op._device()
dg, ds = D["grid"], D["surf"]
gs = ds.gs_tables(dg)
st = torch.cuda.current_stream().cuda_stream
e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
e0.record()
check(lib.hhg_smooth_surface_all(dg.ref, ds.ref, gs["ref"], 1.0, u.data_ptr(), f.data_ptr(), st))
e1.record()
ws = op._skew_workspace()
if ws is None:
    check(lib.hhg_smooth_volume(dg.ref, 0, D["sh"].data_ptr(), 1.0, u.data_ptr(), f.data_ptr(),
                                st))
else:
    check(lib.hhg_smooth_volume_skew(dg.ref, 0, D["sh"].data_ptr(), 1.0, u.data_ptr(),
                                     f.data_ptr(), *(x.data_ptr() for x in ws), 0, st))
e2.record()
torch.cuda.synchronize()
out = op.apply_device(u)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(reps):
    op.apply_device(u, out=out)
torch.cuda.synchronize()
app = (time.perf_counter() - t0) / reps * 1e3
print(f"{case} L{level}: {g.n_nodes} nodes, {g.macro.n_elements} elements, surface levels {gs['nlev']}")
print(f"GS sweep {sweep:.2f} ms (surface {e0.elapsed_time(e1):.2f} ms, volume {e1.elapsed_time(e2):.2f} ms); "
      f"apply {app:.2f} ms")
