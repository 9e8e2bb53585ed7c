"""Volume-kernel throughput of every operator variant on the config-5 workload
(96 macro elements, level 8, one GPU): the paper's Table 5 / §7.4 comparison
(stored stencils vs on-the-fly scaling vs nodal integration vs constant)
plus the tensor (M = 6) kernels.  Kernel-only, inputs resident, CUDA events,
L2 flushed by the 4.3 GB streams themselves.  Synthetic values where the
timing does not depend on them (stored weights, tensor components).

    python tools/variant_bench.py [--level 8] [--reps 10] [--json out.json]
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1709_06793_b200 import RefinedGrid, sample_nodal  # noqa: E402
from paper_1709_06793_b200._lib import FLAG_FAST, FLAG_MIRROR, VAR, check, lib  # noqa: E402
from paper_1709_06793_b200.coefficients import TENSOR_DIRS_3D  # noqa: E402
from paper_1709_06793_b200.device import DeviceGrid, GridTables  # noqa: E402
from paper_1709_06793_b200.reference_stencils import (nodal_factors,  # noqa: E402
                                                     reference_stencil, tensor_tables)
from paper_1709_06793_b200.shard import slab_mesh  # noqa: E402
from tests.cases import k_c5  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--level", type=int, default=8)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--json", default=None)
ap.add_argument("--skip", default="")
args = ap.parse_args()

grid = RefinedGrid(slab_mesh(0, 1), args.level)
ne = grid.macro.n_elements
kf = sample_nodal(k_c5(), grid)
gt = GridTables(grid)
dg = DeviceGrid(gt, kf.values)
st = torch.cuda.current_stream().cuda_stream
dev = "cuda"
u = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, grid.n_nodes), device=dev)
out = torch.empty_like(u)
check(lib.hhg_ghost_update(dg.ref, u.data_ptr(), st))
nrows = grid.nodes_per_volume * ne
L = gt.L
sh = torch.as_tensor(np.stack([reference_stencil(grid, t)[1] / 2 for t in range(ne)]),
                     device=dev).reshape(-1)
fac = torch.as_tensor(np.stack([nodal_factors(grid, t) for t in range(ne)]),
                      device=dev).reshape(-1)
c15 = []
for t in range(ne):
    s = 2.0 * reference_stencil(grid, t)[1] / 2
    c15.append(np.append(s, -s.sum()))
c15 = torch.as_tensor(np.stack(c15), device=dev).reshape(-1)
tt = [tensor_tables(grid, t, TENSOR_DIRS_3D) for t in range(ne)]
shm = torch.as_tensor(np.stack([a for a, _ in tt]), device=dev).reshape(-1)
facm = torch.as_tensor(np.stack([b for _, b in tt]), device=dev).reshape(-1)


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / args.reps


def vol(var, flags, coef, w=None):
    return lambda: check(lib.hhg_volume_apply(dg.ref, var, flags, coef.data_ptr() if coef is not None
                                              else None, w.data_ptr() if w is not None else None,
                                              u.data_ptr(), None, out.data_ptr(), st))


# algorithmic bytes per launch: read u and k lattices once,
# write the rows; stored reads u + 15 weights per row; tensor reads M k's
per_lat = 8 * L * ne
rows_b = 8 * nrows
cases = [
    ("scaling (bitwise, mirror reuse)", vol(VAR["scaling"], FLAG_MIRROR, sh), 2 * per_lat + rows_b, 69),
    ("scaling (bitwise, generic)", vol(VAR["scaling"], 0, sh), 2 * per_lat + rows_b, 69),
    ("scaling (fast: FMA, mirror-folded)", vol(VAR["scaling"], FLAG_FAST, sh), 2 * per_lat + rows_b, 69),
    ("nodal integration", vol(VAR["nodal"], 0, fac), 2 * per_lat + rows_b, 211),
    ("const (15-point, constant k)", vol(VAR["const"], 0, c15), per_lat + rows_b, 29),
]
results = []
skip = set(args.skip.split(",")) if args.skip else set()
for name, fn, nbytes, flops in cases:
    ms = timed(fn)
    results.append((name, ms, nbytes, flops))
    print(f"{name:40s} {ms:8.3f} ms {nrows / ms / 1e6:8.1f} GDoF/s "
          f"{nbytes / ms / 1e6:8.1f} GB/s {flops * nrows / ms / 1e9:8.2f} TFLOP/s", flush=True)

if "stored" not in skip:
    w = torch.empty(nrows * 15, dtype=torch.float64, device=dev).uniform_(-1, 1)
    nb = per_lat + rows_b + 120 * nrows
    ms = timed(vol(VAR["stored"], 0, None, w))
    results.append(("stored stencils (15 weights/row)", ms, nb, 29))
    print(f"{'stored stencils (15 weights/row)':40s} {ms:8.3f} ms {nrows / ms / 1e6:8.1f} GDoF/s "
          f"{nb / ms / 1e6:8.1f} GB/s", flush=True)
    del w
    torch.cuda.empty_cache()

if "tensor" not in skip:
    km = torch.empty(ne * 6 * L, dtype=torch.float64, device=dev).uniform_(0.5, 2.0)
    work = torch.empty(ne * L, dtype=torch.float64, device=dev)
    for name, var, coef, flops in (("tensor scaling (M=6)", VAR["scaling"], shm, 14 * 20),
                                   ("tensor nodal (M=6)", VAR["nodal"], facm, 6 * 40 + 72 * 12 + 42)):
        nb = 7 * per_lat + rows_b
        ms = timed(lambda: check(lib.hhg_tensor_volume_apply(
            dg.ref, var, 0, 6, km.data_ptr(), coef.data_ptr(), u.data_ptr(), None,
            out.data_ptr(), work.data_ptr(), st)))
        results.append((name, ms, nb, flops))
        print(f"{name:40s} {ms:8.3f} ms {nrows / ms / 1e6:8.1f} GDoF/s "
              f"{nb / ms / 1e6:8.1f} GB/s {flops * nrows / ms / 1e9:8.2f} TFLOP/s", flush=True)

if args.json:
    Path(args.json).write_text(json.dumps({
        "workload": f"config 5 per GPU: {ne} macro elements, level {args.level}, {nrows} volume rows",
        "results": [{"variant": n, "ms": ms, "gdofs": nrows / ms / 1e6,
                     "algorithmic_gbs": b / ms / 1e6, "flop_per_row": f}
                    for n, ms, b, f in results]}, indent=1))
