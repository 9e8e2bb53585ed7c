"""Full-apply timing on the config-5 workload with the surface rows either
after the volume kernel on the main stream (N = 1 default) or on a side
stream concurrently with it (the N > 1 path), for library variants built
with extra -D macros (BUILD_ONLY=1 cross-compiles them into tools/_so).

    VARIANTS="default HHG_FACE_TB=4" python tools/overlap_probe.py
"""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
variants = os.environ.get("VARIANTS", "default").split()


def so_of(var):
    tag = "ovl_" + var.replace("=", "").replace("+", "_")
    return ROOT / "tools" / "_so" / f"{tag}.so"


if os.environ.get("BUILD_ONLY"):
    (ROOT / "tools" / "_so").mkdir(exist_ok=True)
    procs = []
    for var in variants:
        defs = [] if var == "default" else var.split("+")
        cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
               "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-shared",
               *[f"-D{d}" for d in defs], "-o", str(so_of(var)),
               str(ROOT / "paper_1709_06793_b200/csrc/hhg_b200.cu")]
        procs.append((var, subprocess.Popen(cmd, stderr=subprocess.PIPE, text=True)))
    for var, pr in procs:
        _, err = pr.communicate()
        print(var, "built" if pr.returncode == 0 else err[-600:], flush=True)
    sys.exit(0)

var = variants[0]
from paper_1709_06793_b200 import _lib  # noqa: E402
_lib.LIB_PATH = so_of(var)
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1709_06793_b200 import Operator, RefinedGrid, sample_nodal  # noqa: E402
from paper_1709_06793_b200.shard import slab_mesh  # noqa: E402
from tests.cases import k_c5  # noqa: E402

grid = RefinedGrid(slab_mesh(0, 1), int(os.environ.get("LEVEL", "8")))
kf = sample_nodal(k_c5(), grid)
op = Operator(grid, "scaling", kf, fast=True)
u = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, grid.n_nodes), device="cuda")
out = torch.empty_like(u)
ref = None
for mode in ("sequential", "concurrent"):
    hook = (lambda o: None) if mode == "concurrent" else None
    for _ in range(5):
        op.apply_device(u, out=out, after_surface=hook)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        op.apply_device(u, out=out, after_surface=hook)
    e1.record()
    torch.cuda.synchronize()
    if ref is None:
        ref = out.clone()
    print(f"{var:20s} {mode:11s} {e0.elapsed_time(e1) / 20:.4f} ms/apply  "
          f"same={bool(torch.equal(out, ref))}", flush=True)
