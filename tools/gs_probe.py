"""Volume Gauss-Seidel sweep variants on the config-5 workload: builds
libhhg_b200 variants (-D macros, BUILD_ONLY=1 cross-compiles them here into
tools/_so), times hhg_smooth_volume with CUDA events and checks each
variant's result bitwise against the first one.

    VARIANTS="HHG_GS_CLUSTER=0 HHG_GS_CLUSTER=8" python tools/gs_probe.py
"""
import ctypes
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1709_06793_b200 import Operator, RefinedGrid, sample_nodal  # noqa: E402
from paper_1709_06793_b200._lib import EXPORTS  # noqa: E402
from paper_1709_06793_b200.device import DeviceGrid, GridTables  # noqa: E402
from paper_1709_06793_b200.shard import slab_mesh  # noqa: E402
from tests.cases import k_c5  # noqa: E402

level = int(os.environ.get("LEVEL", "8"))
variants = os.environ.get("VARIANTS", "HHG_GS_CLUSTER=0 HHG_GS_CLUSTER=8").split()


def tag_of(var):
    defs = [d for d in var.split("+") if d]
    return defs, "gs_" + ("_".join(d.replace("=", "") for d in defs) or "default")


def nvcc_cmd(defs, out):
    return ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
            "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-shared",
            *[f"-D{d}" for d in defs], "-Xptxas", "-v", "-o", str(out),
            str(ROOT / "paper_1709_06793_b200/csrc/hhg_b200.cu")]


if os.environ.get("BUILD_ONLY"):
    (ROOT / "tools" / "_so").mkdir(exist_ok=True)
    procs = []
    for var in variants:
        defs, tag = tag_of(var)
        so = ROOT / "tools" / "_so" / f"{tag}.so"
        procs.append((var, so, subprocess.Popen(nvcc_cmd(defs, so), stdout=subprocess.PIPE,
                                                stderr=subprocess.PIPE, text=True)))
    for var, so, pr in procs:
        _, err = pr.communicate()
        print(var, "built" if pr.returncode == 0 else err[-800:], flush=True)
    sys.exit(0)

grid = RefinedGrid(slab_mesh(0, 1), level)
kf = sample_nodal(k_c5(), grid)
op = Operator(grid, "scaling", kf)
sh = torch.as_tensor(np.stack(op._sh), device="cuda").reshape(-1)
rng = np.random.default_rng(0)
u0 = torch.as_tensor(rng.uniform(-1, 1, grid.n_nodes), device="cuda")
f = torch.as_tensor(rng.uniform(-1, 1, grid.n_nodes), device="cuda")
ref = None
nv = grid.nodes_per_volume * grid.macro.n_elements
ws = None
for var in variants:
    skew = var.endswith(":skew")
    var = var.replace(":skew", "")
    defs, tag = tag_of(var)
    so = ROOT / "tools" / "_so" / f"{tag}.so"
    h = ctypes.CDLL(str(so))
    for nm, (res, args) in EXPORTS.items():
        if hasattr(h, nm):
            getattr(h, nm).restype = res
            getattr(h, nm).argtypes = args
    gt = GridTables(grid, tile_rows=int(h.hhg_volume_tile_rows()),
                    mirror_cols=int(h.hhg_volume_tile_cols_mirror()))
    dg = DeviceGrid(gt, kf.values)
    st = torch.cuda.current_stream().cuda_stream
    u = u0.clone()
    h.hhg_ghost_update(dg.ref, u.data_ptr(), st)
    if skew:
        if ws is None:
            nl = gt.ntets * gt.L
            ws = torch.empty(2 * nl + nv, dtype=torch.float64, device="cuda")   # us, ks, fs
        h.hhg_skew_coefficient(dg.ref, ws[nl:].data_ptr(), st)

    def sweep():
        if skew:
            return h.hhg_smooth_volume_skew(dg.ref, 0, sh.data_ptr(), 1.0, u.data_ptr(),
                                            f.data_ptr(), ws.data_ptr(), ws[2 * nl:].data_ptr(),
                                            ws[nl:].data_ptr(), 0, st)
        return h.hhg_smooth_volume(dg.ref, 0, sh.data_ptr(), 1.0, u.data_ptr(), f.data_ptr(),
                                   st)
    rc = sweep()
    torch.cuda.synchronize()
    if rc:
        print(var, "rc", rc, flush=True)
        continue
    res = u.clone()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        sweep()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    if ref is None:
        ref = res
    print(f"{var + (' skewed' if skew else ''):50s} volume GS sweep {ms:8.3f} ms  bitwise={bool(torch.equal(res, ref))}",
          flush=True)
    del dg
