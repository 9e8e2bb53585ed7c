"""Build the data-movement-only volume kernel (HHG_VOL_EXPT=1) and run it
on the config-5 workload, for an ncu capture of the staging path alone."""
import ctypes, subprocess, sys
from pathlib import Path
import numpy as np, torch
ROOT = Path("/root/repo"); sys.path.insert(0, str(ROOT))
from paper_1709_06793_b200 import RefinedGrid, sample_nodal
from paper_1709_06793_b200._lib import EXPORTS
from paper_1709_06793_b200.device import DeviceGrid, GridTables
from paper_1709_06793_b200.reference_stencils import reference_stencil
from paper_1709_06793_b200.shard import slab_mesh
from tests.cases import k_c5
so = "/tmp/hhg_memonly.so"
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "--expt-relaxed-constexpr",
                "-Xcompiler", "-fPIC", "-shared", "-DHHG_SCALING_ONLY", "-DHHG_VOL_EXPT=1", "-lineinfo", "-o", so,
                str(ROOT / "paper_1709_06793_b200/csrc/hhg_b200.cu")], check=True)
h = ctypes.CDLL(so)
for name, (res, args) in EXPORTS.items():
    if hasattr(h, name):
        getattr(h, name).restype = res; getattr(h, name).argtypes = args
grid = RefinedGrid(slab_mesh(0, 1), 8)
kf = sample_nodal(k_c5(), grid)
u = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, grid.n_nodes), device="cuda")
out = torch.empty_like(u)
sh = torch.as_tensor(np.stack([reference_stencil(grid, t)[1] / 2 for t in range(grid.macro.n_elements)]), device="cuda").reshape(-1)
gt = GridTables(grid, tile_rows=12, mirror_cols=32)
dg = DeviceGrid(gt, kf.values)
st = torch.cuda.current_stream().cuda_stream
h.hhg_ghost_update(dg.ref, u.data_ptr(), st)
for _ in range(3):
    h.hhg_volume_apply(dg.ref, 0, 4, sh.data_ptr(), None, u.data_ptr(), None, out.data_ptr(), st)
torch.cuda.synchronize(); print("ok")
