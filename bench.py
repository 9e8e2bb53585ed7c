"""Benchmark: GDoF/s of the scaled-stencil operator apply (fp64) on B200.

Workload (BASELINE.json config 5, per GPU): a 4 x 4 x 1 slab of Kuhn cubes =
96 macro tetrahedra refined to level 8 (2.7e8 unknowns per GPU), k = 2 +
sin(2 pi x) sin(2 pi y) sin(2 pi z), u uniform[-1, 1] from a seed.  With N
GPUs the slabs stack in z (weak scaling); interface rows are completed by
the NCCL partial-sum exchange.

One step = one full Operator.apply on device-resident data: ghost-layer
update, batched volume stencil kernel, matrix-free surface rows + Dirichlet
rows, and (N > 1) the interface exchange.  `value` counts volume unknowns
(the paper's residual-benchmark convention) over all
ranks; `e2e` times the public call with host numpy buffers.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

With --gpus N > 1 and no torchrun environment the script re-launches itself
under `torch.distributed.run` with N local ranks (127.0.0.1 rendezvous) and
exits with its status; under torchrun it checks WORLD_SIZE == N.
`--dry-run` runs the same multi-rank plumbing on CPU (gloo, no kernels): the
interface partial-sum exchange of every rank's slab at a tiny level.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="own", choices=["own", "reference"])
    ap.add_argument("--level", type=int, default=8)
    ap.add_argument("--nx", type=int, default=4)
    ap.add_argument("--variant", default="scaling", choices=["scaling", "nodal"])
    ap.add_argument("--fast", action="store_true",
                    help="FMA / mirror-pair arithmetic (default: bitwise reference order)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                    help="N > 1 interface exchange: peer-memory push fused into the "
                         "surface-row kernel (CUDA IPC over NVLink) or NCCL send/recv")
    ap.add_argument("--cpu-tets", type=int, default=16,
                    help="macro elements per CPU-baseline step (bounded sample)")
    ap.add_argument("--bitwise", action="store_true",
                    help="reference-order arithmetic (bitwise the CPU kernel); default "
                         "is the FMA edge-flux form, within 1e-12 of it")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU/gloo multi-rank plumbing check (no GPU work)")
    a = ap.parse_args()
    if a.gpus < 1:
        ap.error("--gpus must be >= 1")
    a.fast = not a.bitwise          # --fast kept for compatibility (it is the default)
    return a


def relaunch(args):
    """--gpus N > 1 outside torchrun: run N local ranks under
    torch.distributed.run (one process per GPU) and return its status."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def dist_env(args=None):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args is not None and "WORLD_SIZE" in os.environ and world != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}\n")
        sys.exit(2)
    return world, rank, local


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout
                self.rows.append([x.strip() for x in out.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


SETUP = {}


def build_workload(rank, world, level, nx, variant, fast):
    from paper_1709_06793_b200 import Operator, RefinedGrid, sample_nodal
    from paper_1709_06793_b200.shard import InterfaceMap, slab_mesh
    from tests.cases import k_c5
    t0 = time.time()
    grid = RefinedGrid(slab_mesh(rank, world, nx, nx), level)
    t1 = time.time()
    kf = sample_nodal(k_c5(), grid)     # the synthetic coefficient (numpy, host)
    t2 = time.time()
    op = Operator(grid, variant, kf, fast=fast)
    SETUP.update(grid_s=round(t1 - t0, 2), coefficient_s=round(t2 - t1, 2),
                 operator_s=round(time.time() - t2, 2))
    u = np.random.default_rng(1234 + rank).uniform(-1.0, 1.0, grid.n_nodes)
    imap = InterfaceMap(grid, rank, world, 1.0 / nx) if world > 1 else None
    if imap is not None:   # interface copies must agree across ranks
        X = grid.node_coords
        for ids in imap.neighbours.values():
            u[ids] = np.sin(17.3 * X[ids, 0] + 29.1 * X[ids, 1])
    return grid, kf, op, u, imap


def run_own(args):
    import torch
    world, rank, local = dist_env(args)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if torch.cuda.device_count() < world:
            sys.stderr.write(f"bench.py: {world} ranks but {torch.cuda.device_count()} GPUs\n")
            sys.exit(2)
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    from paper_1709_06793_b200._lib import lib
    from paper_1709_06793_b200.costmodel import volume_apply_bytes, apply_step_bytes
    from paper_1709_06793_b200.shard import exchange_partials

    t_setup = time.time()
    grid, kf, op, u, imap = build_workload(rank, world, args.level, args.nx, args.variant,
                                           args.fast)
    # the CPU baseline runs before any GPU work of this process (after the
    # GPU work the host measured up to 1.5x slower in round 1)
    cpu = None
    if rank == 0 and world == 1:
        t_cpu = time.time()
        cpu = cpu_baseline(grid, kf, op, u, args.cpu_tets, reps=3)
        t_setup += time.time() - t_cpu        # not part of the set-up
    t_dev = time.time()
    D = op._device()
    du = torch.as_tensor(u, device="cuda")
    out = torch.empty_like(du)
    idx_t = sop = None
    if imap is not None:
        from paper_1709_06793_b200.shard import ShardedOperator
        idx_t = {k: torch.as_tensor(v, device="cuda") for k, v in imap.neighbours.items()}
        from paper_1709_06793_b200.shard import PeerUnavailable
        try:
            sop = ShardedOperator(op, imap, dist, grid.dirichlet_mask, transport=args.exchange)
        except PeerUnavailable as exc:     # agreed on every rank: fall back to NCCL
            if rank == 0:
                print(f"bench: p2p exchange unavailable ({exc}); using nccl", file=sys.stderr)
            args.exchange = "nccl"
            sop = ShardedOperator(op, imap, dist, grid.dirichlet_mask, transport="nccl")
    torch.cuda.synchronize()
    SETUP["device_s"] = round(time.time() - t_dev, 2)
    t_setup = time.time() - t_setup

    vol_ev = []

    def step(record=False):
        # the product's Operator.apply_device (surface rows + the N>1
        # interface exchange on a side stream, concurrent with the ghost
        # update and the volume kernel), with CUDA events around the volume
        # kernel on the launching stream
        ev = None
        if record:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            vol_ev.append(ev)
        if sop is not None and sop.peer is not None:
            sop.peer.apply(du, out=out, volume_events=ev)
            return
        hook = None
        if imap is not None:
            hook = lambda o: exchange_partials(o, imap, dist, idx_t)  # noqa: E731
        op.apply_device(du, out=out, after_surface=hook, volume_events=ev)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if sop is not None:
        sop.check()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = lib.hhg_launch_count()
    with ClockSampler(local) as clk:
        ev0.record()
        for _ in range(args.steps):
            step(record=True)
        ev1.record()
        torch.cuda.synchronize()
    launches = lib.hhg_launch_count() - launches0
    if sop is not None:
        sop.check()                       # a lost peer signal invalidates the run
    ms = ev0.elapsed_time(ev1) / args.steps
    vol_ms = sum(a.elapsed_time(b) for a, b in vol_ev) / len(vol_ev)
    per_rank = [{"rank": rank, "step_ms": round(ms, 4), "volume_kernel_ms": round(vol_ms, 4),
                 "other_ms": round(ms - vol_ms, 4)}]
    if dist:
        dist.barrier()
        t = torch.tensor([ms, vol_ms], dtype=torch.float64, device="cuda")
        allt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        per_rank = [{"rank": r, "step_ms": round(float(x[0]), 4),
                     "volume_kernel_ms": round(float(x[1]), 4),
                     "other_ms": round(float(x[0] - x[1]), 4)} for r, x in enumerate(allt)]
        ms = max(float(x[0]) for x in allt)         # max over ranks
        vol_ms = max(float(x[1]) for x in allt)

    ntets = grid.macro.n_elements
    nvol_rank = grid.nodes_per_volume * ntets
    total_dofs = nvol_rank * world
    value = total_dofs / (ms * 1e-3) / 1e9
    hbm, hbm_kind = peaks()
    bytes_launch = volume_apply_bytes(args.level, ntets)
    achieved = bytes_launch / (vol_ms * 1e-3) / 1e9
    step_bytes = apply_step_bytes(grid, op)

    # end to end through the public API with HOST buffers: pinned CPU tensor
    # in, Operator.apply (H2D, kernels, D2H into pinned memory) out
    u_host = torch.from_numpy(u).pin_memory()
    e2e_ms = []
    for i in range(args.e2e_steps + 1):
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if imap is None:
            res = op.apply(u_host)
        else:
            dd = u_host.to("cuda", non_blocking=True)
            o = sop.apply(dd)
            res = torch.empty(o.shape, dtype=o.dtype, pin_memory=True)
            res.copy_(o, non_blocking=True)
        torch.cuda.synchronize()
        if i:
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
        del res
    e2e = statistics.median(e2e_ms) if e2e_ms else float("nan")
    if dist:
        t = torch.tensor([e2e], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = t.item()

    traffic = None
    tp = ROOT / "profiles" / "volume_traffic.json"
    if tp.exists():
        for tj in json.loads(tp.read_text()).get("entries", []):
            if tj.get("level") == args.level and tj.get("ntets") == ntets and \
                    tj.get("arithmetic") == ("fma" if args.fast else "bitwise"):
                traffic = tj.get("dram_bytes_per_launch")

    if rank == 0:
        flags = op._vol_flags()
        if args.variant == "nodal":
            arith = ("fma term sums (<= 1e-12 of the reference order)" if flags & 2
                     else "bitwise-reference-order")
        else:
            arith = ("fma edge-flux, mirror edge reuse (<= 1e-12 of the reference order)"
                     if flags & 2 else "bitwise-reference-order, mirror edge reuse")
        line = {
            "metric": "GDoF/s of scaled-stencil apply (fp64)",
            "value": round(value, 3), "unit": "GDoF/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded u, analytic k)",
            "config": workload_config(args, grid, world),
            "arithmetic": arith,
            "exchange": args.exchange if world > 1 else None,
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm,
                         "unit": "GB/s", "frac": round(achieved / hbm, 4),
                         "traffic": traffic, "peak_kind": hbm_kind,
                         "kernel": "volume_kernel_mirror", "kernel_ms": round(vol_ms, 4),
                         "algorithmic_bytes_per_launch": bytes_launch,
                         "step": {"algorithmic_bytes": step_bytes,
                                  "achieved": round(step_bytes / (ms * 1e-3) / 1e9, 1),
                                  "frac": round(step_bytes / (ms * 1e-3) / 1e9 / hbm, 4)}},
            "e2e": ({"value": round(total_dofs / (e2e * 1e-3) / 1e9, 4), "unit": "GDoF/s",
                     "ms_per_step": round(e2e, 2), "h2d_bytes_per_step": 8 * grid.n_nodes,
                     "d2h_bytes_per_step": 8 * grid.n_nodes} if e2e_ms else None),
            "gpu_launches": int(launches),
            "per_rank": per_rank,
            "all_rows_gdofs": round(grid.n_nodes * world / (ms * 1e-3) / 1e9, 3),
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "setup_s": round(t_setup, 1), "setup": dict(SETUP),
            "build": lib.hhg_build_info().decode(),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def run_dry(args):
    """--dry-run: the multi-rank plumbing of the bench on CPU (gloo): every
    rank builds its slab at --level, exchanges and completes its interface
    partial sums with the neighbours, times the steps on the host and takes
    the max over ranks; no GPU work, no measured value."""
    import torch
    import torch.distributed as dist
    from paper_1709_06793_b200 import RefinedGrid
    from paper_1709_06793_b200.shard import InterfaceMap, exchange_partials, slab_mesh
    world, rank, _ = dist_env(args)
    if world > 1:
        dist.init_process_group("gloo")
    grid = RefinedGrid(slab_mesh(rank, world, args.nx, args.nx), args.level)
    imap = InterfaceMap(grid, rank, world, 1.0 / args.nx) if world > 1 else None
    vec = torch.as_tensor(np.random.default_rng(rank).uniform(-1, 1, grid.n_nodes))
    idx = {k: torch.as_tensor(v) for k, v in imap.neighbours.items()} if imap else None
    for _ in range(args.warmup):
        if imap:
            exchange_partials(vec.clone(), imap, dist, idx)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        if imap:
            exchange_partials(vec.clone(), imap, dist, idx)
    ms = (time.perf_counter() - t0) * 1e3 / args.steps
    ranks = [rank]
    if world > 1:
        t = torch.tensor([ms])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t)
        allr = [None] * world
        dist.all_gather_object(allr, rank)
        ranks = allr
    if rank == 0:
        print(json.dumps({"metric": "GDoF/s of scaled-stencil apply (fp64)", "dry_run": True,
                          "value": None, "unit": "GDoF/s", "n_gpus": world,
                          "ranks_seen": ranks, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": round(ms, 4), "scaling": "weak",
                          "config": {"workload": f"dry run: slab of {grid.macro.n_elements} "
                                                 f"macro tets per rank, level {args.level}",
                                     "parallelism": f"macro-tet slabs x{world}"}}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(grid, kf, op, u, ntets_sample, reps=2):
    """Oracle port (C restatement of kernels.apply_scaling_3d) on the host
    cores over a bounded sample of macro elements of the same workload."""
    from oracle import kernels as ok
    n = grid.n
    T = min(ntets_sample, grid.macro.n_elements)
    v = np.ascontiguousarray(np.stack([u[grid.elem_gidx[t]] for t in range(T)]))
    kc = np.ascontiguousarray(kf.values[:T])
    sh = np.ascontiguousarray(np.stack(op._sh[:T]))
    threads = ok.num_threads()
    ok.apply_scaling_3d_batch(n, grid.lat.base, v, kc, sh, threads)     # warm
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        ok.apply_scaling_3d_batch(n, grid.lat.base, v, kc, sh, threads)
        ts.append(time.perf_counter() - t0)
    t = min(ts)
    return {"value": round(T * grid.nodes_per_volume / t / 1e9, 4), "unit": "GDoF/s",
            "cores": threads, "kind": "port", "cpu_model": cpu_model(),
            "host_cpus": os.cpu_count(),
            "sample": f"{T} of {grid.macro.n_elements} macro tets (level {grid.level}) "
                      f"per step, best of {reps}, volume rows, all host threads"}


def workload_config(args, grid, world):
    """The workload both arms (own / --impl reference) report: identical
    dicts for the same flags (the arithmetic mode is a separate key)."""
    ntets = grid.macro.n_elements
    return {"workload": f"config 5 per GPU: 4x4x1 Kuhn-cube slab, {ntets} macro tets, "
                        f"level {args.level}", "level": args.level,
            "macro_tets_per_gpu": ntets, "dofs_per_gpu": int(grid.n_nodes),
            "volume_dofs_per_gpu": int(grid.nodes_per_volume * ntets), "variant": args.variant,
            "parallelism": f"macro-tet slabs x{world}",
            "l2": "inputs larger than L2 (2.2 GB per vector)"}


def run_reference(args):
    """--impl reference: the reference's CPU algorithm for this path (the C
    restatement of its numba kernel — the reference itself is Python/numba
    and is not importable on the GPU box) on all host cores, same config,
    metric and units; rank 0 only."""
    world, rank, _ = dist_env()
    world = max(world, args.gpus)
    if rank != 0:
        return
    from oracle import kernels as ok
    from paper_1709_06793_b200 import RefinedGrid, sample_nodal
    from paper_1709_06793_b200.reference_stencils import reference_stencil
    from paper_1709_06793_b200.shard import slab_mesh
    from tests.cases import k_c5
    grid = RefinedGrid(slab_mesh(0, 1, args.nx, args.nx), args.level)
    kf = sample_nodal(k_c5(), grid)
    u = np.random.default_rng(1234).uniform(-1.0, 1.0, grid.n_nodes)
    T = min(args.cpu_tets, grid.macro.n_elements)
    v = np.ascontiguousarray(np.stack([u[grid.elem_gidx[t]] for t in range(T)]))
    kc = np.ascontiguousarray(kf.values[:T])
    sh = np.ascontiguousarray(np.stack([reference_stencil(grid, t)[1] / 2.0 for t in range(T)]))
    threads = ok.num_threads()
    for _ in range(args.warmup):
        ok.apply_scaling_3d_batch(grid.n, grid.lat.base, v, kc, sh, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ok.apply_scaling_3d_batch(grid.n, grid.lat.base, v, kc, sh, threads)
    dt = (time.perf_counter() - t0) / args.steps
    val = T * grid.nodes_per_volume / dt / 1e9
    line = {"impl": "reference", "metric": "GDoF/s of scaled-stencil apply (fp64)",
            "value": round(val, 4), "unit": "GDoF/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded u, analytic k)",
            "config": workload_config(args, grid, world),
            "arithmetic": "bitwise reference order (C restatement of kernels.apply_scaling_3d)",
            "cpu_baseline": {"value": round(val, 4), "unit": "GDoF/s", "cores": threads,
                             "kind": "port", "cpu_model": cpu_model(),
                             "host_cpus": os.cpu_count(),
                             "sample": f"{T} macro tets of level {args.level} per step "
                                       "(volume rows), C restatement of "
                                       "kernels.apply_scaling_3d, one thread per core"},
            "e2e": {"value": round(val, 4), "unit": "GDoF/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)          # rank 0 of N (or a plain process): host cores only
    elif a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(a))
    elif a.dry_run:
        run_dry(a)
    else:
        run_own(a)
