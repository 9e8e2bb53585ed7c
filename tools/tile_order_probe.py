"""Does DRAM locality across co-running CTAs matter?  Times the volume
kernel (full and data-movement-only builds) with the default tile order
(element group, band, element, i), a random order, and (band, i, element)."""
import ctypes
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1709_06793_b200 import RefinedGrid, sample_nodal  # noqa: E402
from paper_1709_06793_b200._lib import EXPORTS  # noqa: E402
from paper_1709_06793_b200.device import DeviceGrid, GridTables  # noqa: E402
from paper_1709_06793_b200.reference_stencils import reference_stencil  # noqa: E402
from paper_1709_06793_b200.shard import slab_mesh  # noqa: E402
from tests.cases import k_c5  # noqa: E402

grid = RefinedGrid(slab_mesh(0, 1), 8)
kf = sample_nodal(k_c5(), grid)
u = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, grid.n_nodes), device="cuda")
out = torch.empty_like(u)
sh = torch.as_tensor(np.stack([reference_stencil(grid, t)[1] / 2 for t in range(grid.macro.n_elements)]),
                     device="cuda").reshape(-1)
gt = GridTables(grid, tile_rows=12)
base = gt.tiles.copy()
rng = np.random.default_rng(0)
orders = {"default": base,
          "random": base[rng.permutation(len(base))],
          "band_i_elem": base[np.lexsort((base[:, 0], base[:, 1], base[:, 2]))]}
for expt in (0, 1):
    so = f"/tmp/hhg_order_{expt}.so"
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                    "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-shared",
                    "-DHHG_SCALING_ONLY", f"-DHHG_VOL_EXPT={expt}", "-o", so,
                    str(ROOT / "paper_1709_06793_b200/csrc/hhg_b200.cu")], check=True)
    h = ctypes.CDLL(so)
    for name, (res, args) in EXPORTS.items():
        if hasattr(h, name):
            getattr(h, name).restype = res
            getattr(h, name).argtypes = args
    for name, tl in orders.items():
        gt.tiles = np.ascontiguousarray(tl)
        dg = DeviceGrid(gt, kf.values)
        st = torch.cuda.current_stream().cuda_stream
        h.hhg_ghost_update(dg.ref, u.data_ptr(), st)
        for _ in range(3):
            h.hhg_volume_apply(dg.ref, 0, 4, sh.data_ptr(), None, u.data_ptr(), None, out.data_ptr(), st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            h.hhg_volume_apply(dg.ref, 0, 4, sh.data_ptr(), None, u.data_ptr(), None, out.data_ptr(), st)
        e1.record()
        torch.cuda.synchronize()
        print(f"EXPT={expt} order={name:12s} {e0.elapsed_time(e1) / 20:.3f} ms", flush=True)
        del dg
