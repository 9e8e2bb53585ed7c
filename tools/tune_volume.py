"""Sweep the volume-kernel tile configuration (B rows per thread, W warps,
NS ring stages) on the GPU box: builds scaling-only variants of
libhhg_b200 with nvcc there, times hhg_volume_apply with CUDA events on the
config-5 workload, prints one line per variant."""
import ctypes
import itertools
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1709_06793_b200 import RefinedGrid, sample_nodal  # noqa: E402
from paper_1709_06793_b200._lib import EXPORTS, HhgGrid  # noqa: E402
from paper_1709_06793_b200.device import DeviceGrid, GridTables  # noqa: E402
from paper_1709_06793_b200.reference_stencils import reference_stencil  # noqa: E402
from paper_1709_06793_b200.shard import slab_mesh  # noqa: E402
from tests.cases import k_c5  # noqa: E402

level = int(os.environ.get("LEVEL", "8"))
# CONFIGS items: "B,W,NS[,MINB[,EXPT]][:DEF=1+DEF2=0]" (extra -D macros)
configs = []
for c in os.environ.get("CONFIGS", "2,8,6 1,8,6 2,4,6 3,4,6 1,16,6 2,8,4 2,8,8").split():
    nums, _, extra = c.partition(":")
    configs.append(tuple(int(x) for x in (nums + ",2,0,0").split(",")[:5]) +
                   (tuple(e for e in extra.split("+") if e),))
grid = RefinedGrid(slab_mesh(0, 1), level)
kf = sample_nodal(k_c5(), grid)
u = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, grid.n_nodes), device="cuda")
out = torch.empty_like(u)
sh = torch.as_tensor(np.stack([reference_stencil(grid, t)[1] / 2 for t in range(grid.macro.n_elements)]),
                     device="cuda").reshape(-1)
nvol = grid.nodes_per_volume * grid.macro.n_elements
ref = None
for B, W, NS, MINB, EXPT, EXTRA in configs:
    tag = "".join(ch if ch.isalnum() else "_" for ch in "_".join(EXTRA))
    so = f"/tmp/hhg_tune_{B}_{W}_{NS}_{MINB}_{EXPT}_{tag}.so"
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
           "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-shared", "-DHHG_SCALING_ONLY",
           f"-DHHG_VOL_B={B}", f"-DHHG_VOL_W={W}", f"-DHHG_VOL_NS={NS}", f"-DHHG_VOL_MINB={MINB}", f"-DHHG_MIRROR_MINB={MINB}", f"-DHHG_VOL_EXPT={EXPT}", *[f"-D{e}" for e in EXTRA], "-Xptxas", "-v",
           "-o", so, str(ROOT / "paper_1709_06793_b200/csrc/hhg_b200.cu")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        print(B, W, NS, "build failed", r.stderr[-500:]); continue
    regs = [l for l in r.stderr.splitlines() if "registers" in l]
    h = ctypes.CDLL(so)
    for name, (res, args) in EXPORTS.items():
        if hasattr(h, name):
            getattr(h, name).restype = res
            getattr(h, name).argtypes = args
    gt = GridTables(grid, tile_rows=W * B, mirror_cols=int(h.hhg_volume_tile_cols_mirror()))
    dg = DeviceGrid(gt, kf.values)
    st = torch.cuda.current_stream().cuda_stream
    h.hhg_ghost_update(dg.ref, u.data_ptr(), st)
    for fast in (int(x) for x in os.environ.get("FLAGS", "0 2 4 6").split()):
        for _ in range(3):
            h.hhg_volume_apply(dg.ref, 0, fast, sh.data_ptr(), None, u.data_ptr(), None, out.data_ptr(), st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            h.hhg_volume_apply(dg.ref, 0, fast, sh.data_ptr(), None, u.data_ptr(), None, out.data_ptr(), st)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        chk = float(out[grid.n_surface_nodes:].abs().sum())
        if ref is None and EXPT == 0: ref = chk
        print(f"B={B} W={W} NS={NS} MINB={MINB} EXPT={EXPT} {'+'.join(EXTRA)} flags={fast} {ms:.3f} ms {nvol/ms/1e6:.1f} GDoF/s "
              f"regs={regs[0].split('Used')[1].split(',')[0].strip() if regs else '?'} chk_ok={ref is not None and abs(chk-ref)<=1e-9*ref}", flush=True)
    del dg
