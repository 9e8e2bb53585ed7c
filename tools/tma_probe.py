"""Volume-kernel variant probe on the GPU box: builds scaling-only variants of
libhhg_b200 (extra -D macros per variant), times hhg_volume_apply with CUDA
events on the config-5 workload and checks every variant against the first
one (bitwise for the reference-order kernels, max relative error for the FMA
ones).

    VARIANTS="HHG_VOLUME_TMA=0 HHG_VOLUME_TMA=1 HHG_VOLUME_TMA=1+HHG_TMA_NS=8" \\
        python tools/tma_probe.py
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
from paper_1709_06793_b200 import RefinedGrid, sample_nodal  # noqa: E402
from paper_1709_06793_b200._lib import EXPORTS  # noqa: E402
from paper_1709_06793_b200.device import DeviceGrid, GridTables  # noqa: E402
from paper_1709_06793_b200.reference_stencils import reference_stencil  # noqa: E402
from paper_1709_06793_b200.shard import slab_mesh  # noqa: E402
from tests.cases import k_c5  # noqa: E402

level = int(os.environ.get("LEVEL", "8"))
reps = int(os.environ.get("REPS", "20"))
variants = os.environ.get("VARIANTS", "HHG_VOLUME_TMA=0 HHG_VOLUME_TMA=1").split()
flag_sets = [int(x) for x in os.environ.get("FLAGS", "4 6").split()]   # 4 mirror, 6 mirror+fast



def nvcc_cmd(defs, out):
    return ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
            "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-shared", "-DHHG_SCALING_ONLY",
            *[f"-D{d}" for d in defs], "-Xptxas", "-v", "-o", str(out),
            str(ROOT / "paper_1709_06793_b200/csrc/hhg_b200.cu")]


def tag_of(var):
    defs = [d for d in var.split("+") if d]
    return defs, "_".join(d.replace("=", "") for d in defs) or "default"


if os.environ.get("BUILD_ONLY"):      # cross-compile the variants here, in parallel
    (ROOT / "tools" / "_so").mkdir(exist_ok=True)
    procs = []
    for var in variants:
        defs, tag = tag_of(var)
        pre = ROOT / "tools" / "_so" / f"hhg_probe_{tag}.so"
        procs.append((var, pre, subprocess.Popen(nvcc_cmd(defs, pre), stdout=subprocess.PIPE,
                                                 stderr=subprocess.PIPE, text=True)))
    for var, pre, pr in procs:
        _, err = pr.communicate()
        pre.with_suffix(".log").write_text(err)
        print(var, "built" if pr.returncode == 0 else err[-800:], flush=True)
    sys.exit(0)

grid = RefinedGrid(slab_mesh(0, 1), level)
kf = sample_nodal(k_c5(), grid)
u = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, grid.n_nodes), device="cuda")
out = torch.zeros_like(u)
sh = torch.as_tensor(np.stack([reference_stencil(grid, t)[1] / 2
                               for t in range(grid.macro.n_elements)]), device="cuda").reshape(-1)
nvol = grid.nodes_per_volume * grid.macro.n_elements
vol = slice(grid.n_surface_nodes, grid.n_nodes)
ref = None
for var in variants:
    defs, tag = tag_of(var)
    so = f"/tmp/hhg_probe_{tag}.so"
    pre = ROOT / "tools" / "_so" / f"hhg_probe_{tag}.so"     # BUILD_ONLY=1 cross-compiles these
    cmd = nvcc_cmd(defs, so)
    if pre.exists():
        so = str(pre)
        r = subprocess.CompletedProcess(cmd, 0, "", (pre.with_suffix(".log")).read_text()
                                        if pre.with_suffix(".log").exists() else "")
    else:
        r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        print(var, "build failed", r.stderr[-800:], flush=True)
        continue
    regs = {}
    name = None
    for line in r.stderr.splitlines():
        if "Compiling entry function" in line:
            name = line.split("'")[1]
        elif "registers" in line and name and ("volume_kernel_tma" in name or "mirror" in name):
            regs[name[:40]] = line.split("Used")[1].split(",")[0].strip()
    h = ctypes.CDLL(so)
    for nm, (res, args) in EXPORTS.items():
        if hasattr(h, nm):
            getattr(h, nm).restype = res
            getattr(h, nm).argtypes = args
    gt = GridTables(grid, tile_rows=int(h.hhg_volume_tile_rows()),
                    mirror_cols=int(h.hhg_volume_tile_cols_mirror()))
    dg = DeviceGrid(gt, kf.values)
    st = torch.cuda.current_stream().cuda_stream
    h.hhg_ghost_update(dg.ref, u.data_ptr(), st)
    for fl in flag_sets:
        out.zero_()
        rc = h.hhg_volume_apply(dg.ref, 0, fl, sh.data_ptr(), None, u.data_ptr(), None,
                                out.data_ptr(), st)
        torch.cuda.synchronize()
        if rc:
            print(var, fl, "rc", rc, flush=True)
            continue
        res_v = out[vol].clone()
        for _ in range(3):
            h.hhg_volume_apply(dg.ref, 0, fl, sh.data_ptr(), None, u.data_ptr(), None,
                               out.data_ptr(), st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            h.hhg_volume_apply(dg.ref, 0, fl, sh.data_ptr(), None, u.data_ptr(), None,
                               out.data_ptr(), st)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        if ref is None:
            ref = res_v
        same = bool(torch.equal(res_v, ref))
        rel = float((res_v - ref).abs().max() / ref.abs().max())
        print(f"{var:40s} flags={fl} {ms:.4f} ms {nvol / ms / 1e6:7.1f} GDoF/s "
              f"frac={6.4939e9 / (ms * 1e-3) / 6544.3e9:.3f} bitwise={same} rel={rel:.2e} "
              f"regs={regs}", flush=True)
    del dg
    torch.cuda.synchronize()
