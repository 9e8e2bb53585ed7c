"""Drop-in `Operator` with the reference signature, executed on the B200.

Mirrors `pkg/src/hhgscale/operators.py:142-561`:

    Operator(grid, variant, coeff=None, hybrid_nodal=frozenset())
    .apply(u) -> A u              (Dirichlet rows: identity)
    .residual(u, f) -> f - A u    (Dirichlet rows: 0)
    .smooth(u, f, sweeps=1, omega=1.0)   forward Gauss-Seidel in global order
    .stencil_weights(t), .store_stencils()
    .flops_add / .flops_mul       analytic counters (costmodel.py:36-55)

Inputs may be numpy arrays (copied to the device and back, the reference
contract) or CUDA float64 torch tensors (device-resident, no copies).  Volume
rows run through the batched sm_100a stencil kernels; surface rows through
the matrix-free partial-stencil kernel; there is no host arithmetic on any
apply, residual or smoothing path.
"""
from __future__ import annotations

import warnings

import numpy as np

from . import _lib
from ._lib import check, lib
from .coefficients import CoefficientField, TensorCoefficient
from .costmodel import analytic_count
from .device import (DeviceGrid, DeviceSurface, FaceTables, GridTables, SurfaceTables,
                     require_cuda)
from .mesh import PrimitiveKind
from .reference_stencils import (classify_edge_types, environment,
                                 nodal_factors, partial_stencils,
                                 reference_stencil, tensor_component_coeffs,
                                 tensor_tables)

__all__ = ["Operator", "VARIANTS", "parse_hybrid_set"]

VARIANTS = ("const", "nodal", "scaling", "scaling_ma2", "hybrid", "stored")
MAX_LEVEL = 9     # include/hhg_b200.h HHG_MAX_N = 512

_KIND_NAMES = {"wv": PrimitiveKind.VERTEX, "we": PrimitiveKind.EDGE,
               "wf": PrimitiveKind.FACE}


def parse_hybrid_set(spec: str):
    """'wv+we' style row-class spec -> frozenset of PrimitiveKind."""
    s = spec.strip().lower()
    if s in ("w", "all"):
        return frozenset(_KIND_NAMES.values())
    if not s:
        return frozenset()
    out = set()
    for tok in s.replace(",", "+").split("+"):
        if tok not in _KIND_NAMES:
            raise ValueError(f"unknown primitive class {tok!r} in {spec!r}")
        out.add(_KIND_NAMES[tok])
    return frozenset(out)


class _StoredWeights:
    """Device-resident stencil tables of a stored-variant operator:
    [ntets * nvol * 15] on the GPU; item t is element t's (nvol, 15) table
    copied to the host (numpy)."""

    def __init__(self, dev, ntets, nvol):
        self.device, self.ntets, self.nvol = dev, ntets, nvol

    def __len__(self):
        return self.ntets

    def __getitem__(self, t):
        if not 0 <= t < self.ntets:
            raise IndexError(t)
        a = t * self.nvol * 15
        return self.device[a:a + self.nvol * 15].reshape(self.nvol, 15).cpu().numpy()


class Operator:
    """One operator variant bound to a grid and coefficient, on the GPU."""

    def __init__(self, grid, variant: str, coeff=None, hybrid_nodal=frozenset(),
                 fast=False, surface_mode="face"):
        if variant not in VARIANTS:
            raise ValueError(f"unknown variant {variant!r}")
        if variant == "stored":
            raise ValueError("build the stored variant via store_stencils()")
        self.grid = grid
        self.variant = variant
        self.coeff = coeff
        self.hybrid_nodal = frozenset(hybrid_nodal)
        self.dim = grid.dim
        self.is_tensor = isinstance(coeff, TensorCoefficient)
        self.flops_add = 0
        self.flops_mul = 0
        self.ma2_marked = None
        self._stored = None
        self.fast = bool(fast)
        if surface_mode not in ("csr", "face", "matrix-free"):
            raise ValueError("surface_mode must be 'csr', 'face' or 'matrix-free'")
        self.surface_mode = surface_mode
        if variant == "const":
            self.const_value = 1.0 if coeff is None else float(coeff)
            if self.const_value <= 0:
                raise ValueError("constant coefficient must be positive")
        elif self.is_tensor:
            if variant == "scaling_ma2":
                raise ValueError("the safeguard is defined for scalar "
                                 "coefficients only")
            if coeff.grid is not grid:
                raise ValueError("coefficient sampled on a different grid")
            if surface_mode not in ("csr", "face"):
                raise ValueError("tensor operators use the precomputed surface rows")
        else:
            if not isinstance(coeff, CoefficientField) and not (
                    hasattr(coeff, "values") and hasattr(coeff, "grid")):
                raise ValueError("variant needs a sampled coefficient field")
            if coeff.grid is not grid:
                raise ValueError("coefficient sampled on a different grid")
        if grid.dim != 3:
            raise ValueError("the B200 operators are tetrahedral (dim 3)")
        if grid.level > MAX_LEVEL:
            raise ValueError(f"refinement level {grid.level} exceeds the B200 build's "
                             f"maximum {MAX_LEVEL} (n = 2^level <= 512: 32-bit lattice "
                             "offsets, 10-bit point codes)")
        self._env = environment(3)
        self._nvol = grid.nodes_per_volume
        self._setup_tables()
        self._dev = None

    # -- host setup (tables only; no operator arithmetic) --------------------
    def _setup_tensor_tables(self):
        """Per element and component: half stencils shm (M, 14), nodal
        factors facm (M, 72) (operators.py:221-238), and the one-sided
        partial stencils of the surface rows, [element][M][class][...]."""
        grid = self.grid
        ne = grid.macro.n_elements
        self._sh, self._fac = [], []
        for t in range(ne):
            shm, facm = tensor_tables(grid, t, self.coeff.dirs)
            self._sh.append(shm)
            self._fac.append(facm)
        cfs = tensor_component_coeffs(self.coeff.dirs, self._env.nshapes)
        psh = np.zeros((ne, len(cfs), 14, 14))
        pfac = np.zeros((ne, len(cfs), 14, 72))
        for t in range(ne):
            for m, cf in enumerate(cfs):
                psh[t, m], pfac[t, m] = partial_stencils(grid, t, coeff=cf)
        self._psh, self._pfac = psh, pfac
        stack = self._fac if self.variant == "nodal" else self._sh
        self._coef = np.ascontiguousarray(np.stack(stack)) if ne else np.zeros((0, 6, 14))
        self._mirror = False
        if self.variant == "nodal":
            self._nodal_kinds = frozenset(PrimitiveKind)
        elif self.variant == "hybrid":
            self._nodal_kinds = self.hybrid_nodal
        else:
            self._nodal_kinds = frozenset()

    def _setup_tables(self):
        grid = self.grid
        ne = grid.macro.n_elements
        if self.is_tensor:
            return self._setup_tensor_tables()
        self._sh, self._fac = [], []
        if self.variant == "scaling_ma2":
            self._warn_3d_safeguard()
        for t in range(ne):
            _, s = reference_stencil(grid, t)
            self._sh.append(s / 2.0)
            self._fac.append(nodal_factors(grid, t) if self.variant == "nodal" else None)
        parts = [partial_stencils(grid, t) for t in range(ne)]
        self._psh = np.ascontiguousarray(np.stack([p for p, _ in parts])) if ne else \
            np.zeros((0, 14, 14))
        need_fac = self.variant in ("nodal", "hybrid")
        self._pfac = np.ascontiguousarray(np.stack([f for _, f in parts])) \
            if (need_fac and ne) else None
        if self.variant == "const":
            # element rows c * A_hat == scaling rows with k == c
            coef = []
            for t in range(ne):
                s = self.const_value * 2.0 * self._sh[t]
                coef.append(np.append(s, -s.sum()))
            self._coef = np.ascontiguousarray(np.stack(coef)) if ne else np.zeros((0, 15))
        elif self.variant == "nodal":
            self._coef = np.ascontiguousarray(np.stack(self._fac)) if ne else np.zeros((0, 72))
        else:
            self._coef = np.ascontiguousarray(np.stack(self._sh)) if ne else np.zeros((0, 14))
        # sh[d] == sh[d+7] bitwise for every element -> edge-term reuse in
        # the volume kernel gives bitwise the same rows with fewer FP64 ops
        self._mirror = bool(ne) and all(np.array_equal(h[:7], h[7:]) for h in self._sh)
        if self.variant == "nodal":
            self._nodal_kinds = frozenset(PrimitiveKind)
        elif self.variant == "hybrid":
            self._nodal_kinds = self.hybrid_nodal
        else:
            self._nodal_kinds = frozenset()

    def _warn_3d_safeguard(self):
        """3-D MA2 is a diagnostic only (operators.py:257-275)."""
        grid = self.grid
        hits = []
        for t in range(grid.macro.n_elements):
            _, s, _ = classify_edge_types(grid, t)
            if not np.any(s > 0):
                continue
            kv = self.coeff.values[t]
            if kv.max() / kv.min() > 2.0:
                hits.append(t)
        if hits:
            warnings.warn(
                "3D safeguard not implemented: macro elements "
                f"{hits} have positive stencil directions and strong "
                "coefficient variation; using plain scaling rows",
                RuntimeWarning, stacklevel=3)

    # -- device state ------------------------------------------------------
    def _device(self):
        if self._dev is None:
            torch = require_cuda()
            grid = self.grid
            gt = GridTables(grid)
            km = None
            if self.variant == "const":
                kc = np.full((gt.ntets, gt.L), self.const_value)
            elif self.is_tensor:
                kc = self.coeff.fields[0].values
                km = torch.as_tensor(self.coeff.packed(), device="cuda").reshape(-1)
            else:
                kc = self.coeff.values
            dg = DeviceGrid(gt, kc)
            st = SurfaceTables(grid, gt, self._nodal_kinds)
            faces = FaceTables(grid, gt, st, kc) if (self.surface_mode == "face" and
                                                     not self.is_tensor) else None
            ds = DeviceSurface(st, self._psh, self._pfac,
                               tensor=(self.coeff.M, km) if self.is_tensor else None,
                               faces=faces)
            coef = torch.as_tensor(self._coef, device="cuda").reshape(-1)
            w = None
            if self._stored is not None:
                w = self._stored.device
            sh = torch.as_tensor(np.ascontiguousarray(np.stack(self._sh)) if self._sh
                                 else np.zeros((0, 14)), device="cuda").reshape(-1)
            fac = None
            if self._fac and self._fac[0] is not None:
                fac = torch.as_tensor(np.ascontiguousarray(np.stack(self._fac)),
                                      device="cuda").reshape(-1)
            self._dev = {"grid": dg, "surf": ds, "coef": coef, "w": w, "torch": torch,
                         "sh": sh, "fac": fac, "km": km}
        return self._dev

    def _lattice_work(self):
        """Element-lattice scratch of the tensor kernels ([elements * L])."""
        D = self._device()
        if D.get("work") is None:
            gt = D["grid"].gt
            D["work"] = D["torch"].empty(max(gt.ntets * gt.L, 1), dtype=D["torch"].float64,
                                         device="cuda")
        return D["work"]

    def _vol_flags(self, residual=False):
        f = _lib.FLAG_RESIDUAL if residual else 0
        if self.is_tensor and self._stored is None:
            return f
        # mirror-symmetric stencils: edge terms shared by two rows of a thread
        # are evaluated once (bitwise); with fast=True the FMA edge-flux form
        # of the same kernel (hhg_volume.cuh fma_step, <= 1e-12 of the
        # reference order)
        if self._mirror and self._vol_variant() == _lib.VAR["scaling"]:
            f |= _lib.FLAG_MIRROR
        if self.fast and self._vol_variant() in (_lib.VAR["scaling"], _lib.VAR["nodal"]):
            f |= _lib.FLAG_FAST
        return f

    def _vol_variant(self):
        if self._stored is not None:
            return _lib.VAR["stored"]
        if self.variant == "nodal":
            return _lib.VAR["nodal"]
        if self.variant == "const":
            return _lib.VAR["const"]
        return _lib.VAR["scaling"]

    def _to_dev(self, x, name="grid function"):
        """(device tensor, kind) with kind 'cuda' (device input, no copy),
        'host' (CPU torch tensor: pinned-friendly non-blocking copy) or
        'numpy' (reference contract: numpy in, numpy out)."""
        D = self._device()
        torch = D["torch"]
        if isinstance(x, torch.Tensor):
            if x.shape != (self.grid.n_nodes,):
                raise ValueError(f"{name} has wrong length")
            if x.is_cuda:
                return x.to(dtype=torch.float64).contiguous(), "cuda"
            return x.to(device="cuda", dtype=torch.float64, non_blocking=True), "host"
        a = np.asarray(x, dtype=np.float64)
        if a.shape != (self.grid.n_nodes,):
            raise ValueError(f"{name} has wrong length")
        return torch.from_numpy(np.ascontiguousarray(a)).to("cuda"), "numpy"

    def _from_dev(self, out, kind):
        if kind == "cuda":
            return out
        torch = self._device()["torch"]
        if kind == "host":
            host = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
            host.copy_(out, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            return host
        return out.cpu().numpy()

    def _stream(self):
        return self._device()["torch"].cuda.current_stream().cuda_stream

    def apply_device(self, du, out=None, f=None, after_surface=None, volume_events=None,
                     push=None):
        """Device-resident A u (or f - A u when f is given), torch tensors.

        Order: ghost update, volume rows, surface + Dirichlet rows.  With
        ``after_surface(out)`` (the sharded operator's interface exchange)
        the surface rows - disjoint from the volume rows - run right after
        the ghost update on a side stream followed by the callable,
        concurrently with the volume kernel; the side stream joins before
        returning.
        ``volume_events``: optional (start, end) CUDA events recorded around
        the volume kernel on the launching stream (bench.py)."""
        D = self._device()
        torch = D["torch"]
        if out is None:
            out = torch.empty_like(du)
        main = torch.cuda.current_stream()
        st = main.cuda_stream
        dg, ds = D["grid"], D["surf"]
        flags = self._vol_flags(residual=f is not None)
        res = flags & _lib.FLAG_RESIDUAL
        fp = f.data_ptr() if f is not None else None
        # surface rows on a side stream, concurrently with the volume kernel,
        # when an exchange hook follows them (N > 1).  On one GPU the overlap
        # gains 0.6-1.3% per config-5 apply (tools/overlap_probe.py) but
        # slows the volume kernel itself by sharing the SMs (1.63 -> 1.82
        # ms), so the sequential order is kept there.
        concurrent = self.surface_mode != "matrix-free" and after_surface is not None
        # the surface rows read shell values from the ghost layer: refresh first
        check(lib.hhg_ghost_update(dg.ref, du.data_ptr(), st), "ghost_update")
        if concurrent:
            ds.csr(dg)                          # one-time setup, on this stream
            side = D.get("side")
            if side is None:
                side = D["side"] = torch.cuda.Stream()
            side.wait_stream(main)
            with torch.cuda.stream(side):
                self._surface(dg, ds, res, du, fp, out, side.cuda_stream, push=push)
                if after_surface is not None:
                    after_surface(out)
        if not concurrent and after_surface is not None:
            self._surface(dg, ds, res, du, fp, out, st, push=push)
            after_surface(out)
        if volume_events is not None:
            volume_events[0].record(main)
        wp = D["w"].data_ptr() if D["w"] is not None else None
        if self.is_tensor and self._stored is None:
            check(lib.hhg_tensor_volume_apply(dg.ref, self._vol_variant(), flags,
                                              self.coeff.M, D["km"].data_ptr(),
                                              D["coef"].data_ptr(), du.data_ptr(), fp,
                                              out.data_ptr(), self._lattice_work().data_ptr(),
                                              st), "tensor_volume_apply")
        else:
            check(lib.hhg_volume_apply(dg.ref, self._vol_variant(), flags,
                                       D["coef"].data_ptr(), wp, du.data_ptr(), fp,
                                       out.data_ptr(), st), "volume_apply")
        if volume_events is not None:
            volume_events[1].record(main)
        if concurrent:
            main.wait_stream(side)
        elif after_surface is None:
            self._surface(dg, ds, res, du, fp, out, st, push=push)
        self._count()
        return out

    def _surface(self, dg, ds, res_flag, du, fp, out, st, push=None):
        """Surface + Dirichlet rows.  ``surface_mode``: "face" (default) -
        face rows by the face-tiled kernel from static face-major layers,
        edge / vertex rows from the precomputed rows; "csr" - every row from
        the precomputed rows (filled on the device on first use); or
        "matrix-free" (two passes over the incidences).  Bitwise equal.
        ``push`` = (slot_ptr, dst0, dst1, split): also store the interface
        rows into the neighbours' receive buffers (shard.PeerExchange)."""
        if self.surface_mode != "matrix-free":
            c = ds.csr(dg)
            if push is not None and not res_flag:
                check(lib.hhg_surface_apply_csr_push(dg.ref, ds.ref, c["ref"], du.data_ptr(),
                                                     out.data_ptr(), *push, st),
                      "surface_apply_csr_push")
                return
            check(lib.hhg_surface_apply_csr(dg.ref, ds.ref, c["ref"], res_flag, du.data_ptr(),
                                            fp, out.data_ptr(), st), "surface_apply_csr")
        else:
            check(lib.hhg_surface_apply(dg.ref, ds.ref, 0, res_flag, du.data_ptr(), fp,
                                        out.data_ptr(), st), "surface_apply")

    # -- host-buffer pipeline ---------------------------------------------------
    def _pipeline(self, groups=32):
        """Streams, events and per-group tile descriptors of apply_host."""
        if getattr(self, "_pipe", None) is None:
            import ctypes
            D = self._device()
            torch = D["torch"]
            grid, dg = self.grid, D["grid"]
            ne = grid.macro.n_elements
            ng = max(1, min(groups, ne))
            # the first group is a single element: the D2H leg can start as
            # soon as the surface block and one volume block have landed
            bounds = np.unique(np.concatenate(
                [[0], np.linspace(min(1, ne), ne, ng).astype(int)])) if ne > 1 else \
                np.array([0, ne])
            tiles, mtiles = dg.gt.tiles, dg.gt.mtiles
            descs, keep = [], []
            for g in range(ng):
                d = type(dg.desc).from_buffer_copy(dg.desc)
                sel = (tiles[:, 0] >= bounds[g]) & (tiles[:, 0] < bounds[g + 1])
                tg = torch.as_tensor(np.ascontiguousarray(tiles[sel]), device="cuda")
                d.tiles = tg.data_ptr() if len(tg) else None
                d.ntiles = int(sel.sum())
                msel = (mtiles[:, 0] >= bounds[g]) & (mtiles[:, 0] < bounds[g + 1])
                mg = torch.as_tensor(np.ascontiguousarray(mtiles[msel]), device="cuda")
                d.mtiles = mg.data_ptr() if len(mg) else None
                d.nmtiles = int(msel.sum())
                descs.append(d)
                keep += [tg, mg]
            n = grid.n_nodes
            self._pipe = {
                "bounds": bounds, "descs": descs, "keep": keep,
                "streams": [torch.cuda.Stream() for _ in range(3)],
                "du": torch.empty(n, dtype=torch.float64, device="cuda"),
                "out": torch.empty(n, dtype=torch.float64, device="cuda"),
                "byref": ctypes.byref,
            }
        return self._pipe

    def _chunks(self):
        """Host<->device copy ranges of the pipeline: the surface block, then
        one contiguous volume block per group of macro elements."""
        P = self._pipeline()
        grid = self.grid
        ns, vs, nv = grid.n_surface_nodes, grid.vol_start, grid.nodes_per_volume
        out = [(0, ns)]
        for g in range(len(P["descs"])):
            if nv:
                out.append((int(vs[P["bounds"][g]]), int(vs[P["bounds"][g + 1] - 1] + nv)))
            else:
                out.append((ns, ns))
        return out

    def _staging(self, key):
        """Persistent pinned staging vector (numpy inputs of apply_host)."""
        P = self._pipeline()
        if key not in P:
            torch = self._device()["torch"]
            P[key] = torch.empty(self.grid.n_nodes, dtype=torch.float64, pin_memory=True)
        return P[key]

    def apply_host(self, u_host, f_host=None):
        """A u (or f - A u) for host inputs, H2D / kernels / D2H overlapped
        per group of macro elements: the surface block goes first (the ghost
        update needs only surface values), each group's volume block is
        applied as soon as it has landed and copied back while the next
        group is in flight; the surface rows (which read interior values of
        every element) run last.

        Inputs are pinned CPU float64 tensors, or numpy arrays: those are
        copied chunk by chunk into persistent pinned staging buffers by a
        pool of host threads, each chunk's H2D enqueued as soon as its copy
        is done.  Returns a fresh pinned CPU tensor (a numpy view of one for
        numpy inputs)."""
        D = self._device()
        torch = D["torch"]
        P = self._pipeline()
        grid, dg, ds = self.grid, D["grid"], D["surf"]
        h2d, comp, d2h = P["streams"]
        du, out = P["du"], P["out"]
        res = f_host is not None
        df = None
        if res:
            if "df" not in P:
                P["df"] = torch.empty_like(du)
            df = P["df"]
        numpy_in = isinstance(u_host, np.ndarray)
        srcs = [(u_host, du, "stage_u")] + ([(f_host, df, "stage_f")] if res else [])
        # a fresh pinned result per call (the reference returns a new array;
        # torch's caching host allocator recycles freed blocks)
        hout = torch.empty(grid.n_nodes, dtype=torch.float64, pin_memory=True)
        chunks = self._chunks()
        flags = self._vol_flags(residual=res)
        wp = D["w"].data_ptr() if D["w"] is not None else None
        if self.surface_mode != "matrix-free":
            ds.csr(dg)          # one-time fill on this stream, before the others join it
        cur = torch.cuda.current_stream()
        for st in P["streams"]:
            st.wait_stream(cur)
        pending = {}
        if numpy_in:
            pool = P.get("pool")
            if pool is None:
                import os
                from concurrent.futures import ThreadPoolExecutor
                pool = P["pool"] = ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 1))
            views = [(src, self._staging(key).numpy()) for src, _, key in srcs]
            for ci, (a, b) in enumerate(chunks):
                if b > a:
                    pending[ci] = [pool.submit(np.copyto, stg[a:b], src[a:b])
                                   for src, stg in views]
        ev_in = []
        with torch.cuda.stream(h2d):
            for ci, (a, b) in enumerate(chunks):
                if b > a:
                    for fut in pending.get(ci, ()):
                        fut.result()
                    for src, dst, key in srcs:
                        host = self._staging(key) if numpy_in else src
                        dst[a:b].copy_(host[a:b], non_blocking=True)
                e = torch.cuda.Event()
                e.record(h2d)
                ev_in.append(e)
        comp.wait_event(ev_in[0])
        cs = comp.cuda_stream
        fp = df.data_ptr() if res else None
        check(lib.hhg_ghost_update(dg.ref, du.data_ptr(), cs), "ghost_update")
        for g, desc in enumerate(P["descs"]):
            comp.wait_event(ev_in[g + 1])
            check(lib.hhg_volume_apply(P["byref"](desc), self._vol_variant(), flags,
                                       D["coef"].data_ptr(), wp, du.data_ptr(), fp,
                                       out.data_ptr(), cs), "volume_apply")
            e = torch.cuda.Event()
            e.record(comp)
            d2h.wait_event(e)
            a, b = chunks[g + 1]
            if b > a:
                with torch.cuda.stream(d2h):
                    hout[a:b].copy_(out[a:b], non_blocking=True)
        self._surface(dg, ds, flags & _lib.FLAG_RESIDUAL, du, fp, out, cs)
        e = torch.cuda.Event()
        e.record(comp)
        d2h.wait_event(e)
        a, b = chunks[0]
        with torch.cuda.stream(d2h):
            hout[a:b].copy_(out[a:b], non_blocking=True)
        d2h.synchronize()
        self._count()
        return hout.numpy() if numpy_in else hout

    @property
    def _S(self):
        """The surface rows as the reference's scipy CSR matrix
        (``Operator._S``, operators.py:329-365: n_nodes x n_nodes, rows of the
        free surface nodes only, duplicates summed).  Built once, lazily, from
        the rows the device filled for apply / smooth (neighbour ids and
        weights per incidence and direction, diagonal = minus their sum); the
        values are the reference's up to summation order (<= 1e-13)."""
        if getattr(self, "_S_cache", None) is None:
            import scipy.sparse as sp
            D = self._device()
            torch = D["torch"]
            dg, ds = D["grid"], D["surf"]
            c = ds.csr(dg)
            torch.cuda.synchronize()
            rows = np.asarray(ds.st.rows, dtype=np.int64)
            nr = len(rows)
            ptr = c["keep"][0].cpu().numpy()
            nent = int(ptr[-1]) if nr else 0
            col = c["keep"][1].cpu().numpy()[:nent].astype(np.int64)
            val = c["keep"][2].cpu().numpy()[:nent]
            diag = c["keep"][3].cpu().numpy()[:nr]
            r = np.repeat(rows, np.diff(ptr))
            n = self.grid.n_nodes
            S = sp.coo_matrix((np.concatenate([val, diag]),
                               (np.concatenate([r, rows]), np.concatenate([col, rows]))),
                              shape=(n, n)).tocsr()
            S.sum_duplicates()
            self._S_cache = S
        return self._S_cache

    # -- public operations (reference signatures) ------------------------------
    def _host_input(self, x, name):
        """x as an input of the host pipeline (float64 numpy array or pinned-
        friendly contiguous CPU float64 tensor), or None if it is not one."""
        if self.is_tensor:
            return None
        torch = self._device()["torch"]
        if isinstance(x, torch.Tensor):
            if x.is_cuda or x.dtype != torch.float64 or not x.is_contiguous():
                return None
            if x.shape != (self.grid.n_nodes,):
                raise ValueError(f"{name} has wrong length")
            return x
        a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
        if a.shape != (self.grid.n_nodes,):
            raise ValueError(f"{name} has wrong length")
        return a

    def apply(self, u):
        """Matrix action A u with identity on Dirichlet rows."""
        h = self._host_input(u, "grid function")
        if h is not None:
            return self.apply_host(h)
        du, kind = self._to_dev(u)
        return self._from_dev(self.apply_device(du), kind)

    def residual(self, u, f):
        """r = f - A u, forced to zero on Dirichlet rows."""
        hu = self._host_input(u, "grid function")
        hf = self._host_input(f, "right-hand side") if hu is not None else None
        if hu is not None and hf is not None and isinstance(hu, np.ndarray) == \
                isinstance(hf, np.ndarray):
            return self.apply_host(hu, hf)
        du, kind = self._to_dev(u)
        df, _ = self._to_dev(f, "right-hand side")
        return self._from_dev(self.apply_device(du, f=df), kind)

    def _volume_sweeper(self, du, df, omega):
        """Callable running one volume Gauss-Seidel sweep of every element
        (hyperplane wavefronts; reads the ghost layer, which must be current)
        on device tensors du, df.  Between two calls of one sweeper only the
        surface rows of du (and the ghost layer) may change - the smoothers'
        surface sweep - and no other sweeper of this operator may run: the
        hyperplane-major path keeps its copies of f and of du's interior."""
        D = self._device()
        dg = D["grid"]
        st = self._stream()
        src = getattr(self, "source_variant", self.variant)
        if self.is_tensor:
            var = _lib.VAR["nodal"] if src == "nodal" else _lib.VAR["scaling"]
            coef = D.get("tcoef")
            if coef is None:
                stack = self._fac if src == "nodal" else self._sh
                coef = D["tcoef"] = D["torch"].as_tensor(
                    np.ascontiguousarray(np.stack(stack)), device="cuda").reshape(-1)

            def volume():
                check(lib.hhg_tensor_smooth_volume(dg.ref, var, self.coeff.M,
                                                   D["km"].data_ptr(), coef.data_ptr(),
                                                   float(omega), du.data_ptr(),
                                                   df.data_ptr(),
                                                   self._lattice_work().data_ptr(), st),
                      "tensor_smooth_volume")
            return volume
        if src == "nodal":
            var, coef = _lib.VAR["nodal"], D["coef"] if self._stored is None else D["fac"]
        else:
            var, coef = _lib.VAR["scaling"], D["sh"]
        ws = self._skew_workspace()
        # later sweeps of one sweeper: f's skewed copy and the skewed
        # interior of u are current (HHG_SKEW_F_CURRENT | HHG_SKEW_U_CURRENT;
        # between sweeps only surface rows and the ghost shell change)
        flags = [0]

        def volume():
            if ws is None:
                check(lib.hhg_smooth_volume(dg.ref, var, coef.data_ptr(), float(omega),
                                            du.data_ptr(), df.data_ptr(), st), "smooth_volume")
                return
            us, fs, ks = ws
            check(lib.hhg_smooth_volume_skew(dg.ref, var, coef.data_ptr(), float(omega),
                                             du.data_ptr(), df.data_ptr(), us.data_ptr(),
                                             fs.data_ptr(), ks.data_ptr(), flags[0], st),
                  "smooth_volume_skew")
            flags[0] = 3
        return volume

    def smooth_device(self, du, df, sweeps=1, omega=1.0, check_diag=True):
        """Forward GS on device tensors.  Surface rows level by level, ghost
        refresh, then volume wavefronts.  const / stored smooth with the
        scaling (or, for a nodal source, nodal) sweep: their stencil weights
        are bitwise those rows ((c+c)*sh == (c*2)*sh; dumped weights are the
        scaling/nodal row terms).

        ``check_diag``: synchronise and raise the reference's "zero central
        stencil entry" ValueError here (the public ``smooth``).  The
        multigrid cycle passes False and checks the shared status word once
        per solve, so a V-cycle enqueues its sweeps without host round
        trips."""
        D = self._device()
        dg, ds = D["grid"], D["surf"]
        st = self._stream()
        gs = ds.gs_tables(dg)
        volume = self._volume_sweeper(du, df, omega)
        if check_diag:
            lib.hhg_status_reset()
        for _ in range(sweeps):
            check(lib.hhg_smooth_surface_all(dg.ref, ds.ref, gs["ref"], float(omega),
                                             du.data_ptr(), df.data_ptr(), st),
                  "smooth_surface")
            check(lib.hhg_ghost_update(dg.ref, du.data_ptr(), st), "ghost_update")
            volume()
        if check_diag:
            D["torch"].cuda.current_stream().synchronize()
            check(lib.hhg_status(), "smooth")
        return du

    def _skew_workspace(self):
        """(us, fs, ks) of the hyperplane-major volume sweep
        (hhg_smooth_volume_skew): u and f copies, the skewed coefficient once
        per operator; None below level 5 (n < 32, HHG_SKEW_MIN_N), where
        the plain cluster sweep is faster than the moves in and out
        (measured: L5 0.28 -> 0.22 ms, L6 0.69 -> 0.57 ms with the skewed
        whole-lattice sweep)."""
        D = self._device()
        if "skew" not in D:
            gt = D["grid"].gt
            nv = gt.ntets * gt.nvol
            import os
            if gt.n < int(os.environ.get("HHG_SKEW_MIN_N", "32")) or nv == 0:
                D["skew"] = None
            else:
                torch = D["torch"]
                nl = gt.ntets * gt.L      # whole lattices (interior + boundary)
                buf = torch.empty(2 * nl + nv, dtype=torch.float64, device="cuda")
                us, ks, fs = buf[:nl], buf[nl:2 * nl], buf[2 * nl:]
                check(lib.hhg_skew_coefficient(D["grid"].ref, ks.data_ptr(), self._stream()),
                      "skew_coefficient")
                D["skew"] = (us, fs, ks)
        return D["skew"]

    def smooth(self, u, f, sweeps=1, omega=1.0):
        """Forward Gauss-Seidel in global node order, in place; returns u."""
        du, kind = self._to_dev(u)
        df, _ = self._to_dev(f, "right-hand side")
        self.smooth_device(du, df, sweeps, omega)
        if kind == "numpy":
            u[...] = du.cpu().numpy()
        elif du.data_ptr() != u.data_ptr():
            u.copy_(du)
        return u

    def _count(self, napplies=1):
        v = self.variant
        if self.is_tensor:
            return
        if v in ("scaling", "scaling_ma2", "hybrid"):
            cnt = analytic_count("scaling", 3)
        elif v in ("nodal", "const", "stored"):
            cnt = analytic_count(v, 3)
        else:
            return
        total = self._nvol * self.grid.macro.n_elements * napplies
        self.flops_add += cnt.add * total
        self.flops_mul += cnt.mul * total

    def stencil_weights(self, t):
        """Volume stencil table of macro element t: rows (centre, s_0..s_13),
        restated from the dump kernels (kernels.py:293-468)."""
        w = np.zeros((self._nvol, 15))
        if not self._nvol:
            return w
        if self._stored is not None:
            return self._stored[t].copy()
        from .mesh import SimplexLattice
        n = self.grid.n
        lat = self.grid.lat
        ijk = SimplexLattice(3, n - 4).coords + 1
        p = lat.index(ijk)
        nb = [lat.index(ijk + d) for d in self._env.dirs]
        if self.variant == "const":
            s = self.const_value * 2.0 * self._sh[t]
            w[:, 0] = -s.sum()
            w[:, 1:] = s
            return w
        if self.is_tensor:
            return self._tensor_weights(t, p, nb, w)
        kv = self.coeff.values[t]
        k0 = kv[p]
        if self.variant == "nodal":
            env = self._env
            buf = np.empty((len(p), 55))
            buf[:, 0] = k0
            for d in range(14):
                buf[:, 1 + d] = kv[nb[d]]
            for dst, a, b in env.cse_schedule:
                buf[:, dst] = buf[:, a] + buf[:, b]
            fac = self._fac[t]
            tot = np.zeros(len(p))
            for d in range(14):
                lo, hi = env.term_ptr[d], env.term_ptr[d + 1]
                s = buf[:, env.cse_sums[env.term_elem[lo]]] * fac[lo]
                for tt in range(lo + 1, hi):
                    s = s + buf[:, env.cse_sums[env.term_elem[tt]]] * fac[tt]
                w[:, 1 + d] = s
                tot = tot + s
            w[:, 0] = -tot
            return w
        sh = self._sh[t]
        tot = np.zeros(len(p))
        for d in range(14):
            sd = (k0 + kv[nb[d]]) * sh[d]
            w[:, 1 + d] = sd
            tot = tot + sd
        w[:, 0] = -tot
        return w

    def _tensor_weights(self, t, p, nb, w):
        """Tensor stencil table (dump_scaling_tensor_3d / dump_nodal_tensor_3d,
        kernels.py:377-468), same association order."""
        km = [f.values[t] for f in self.coeff.fields]
        M = len(km)
        tot = np.zeros(len(p))
        if self.variant == "nodal":
            env = self._env
            fac = self._fac[t]
            es = []
            for m in range(M):
                buf = np.empty((len(p), 55))
                buf[:, 0] = km[m][p]
                for d in range(14):
                    buf[:, 1 + d] = km[m][nb[d]]
                for dst, a, b in env.cse_schedule:
                    buf[:, dst] = buf[:, a] + buf[:, b]
                es.append(buf[:, env.cse_sums])
            for d in range(14):
                s = np.zeros(len(p))
                for tt in range(env.term_ptr[d], env.term_ptr[d + 1]):
                    e = env.term_elem[tt]
                    for m in range(M):
                        s = s + es[m][:, e] * fac[m, tt]
                w[:, 1 + d] = s
                tot = tot + s
        else:
            shm = self._sh[t]
            for d in range(14):
                s = np.zeros(len(p))
                for m in range(M):
                    s = s + (km[m][p] + km[m][nb[d]]) * shm[m, d]
                w[:, 1 + d] = s
                tot = tot + s
        w[:, 0] = -tot
        return w

    def store_stencils(self):
        """Precompute all volume stencils; returns the stored-variant twin
        (operators.py:549-561).  Scaling and nodal stencils are dumped on the
        device by one kernel over all elements (hhg_dump_stencils, the
        reference's dump kernels) and stay there; `_stored[t]` copies
        element t's table to the host on demand."""
        op = object.__new__(Operator)
        op.__dict__.update(self.__dict__)
        op.variant = "stored"
        op.source_variant = self.variant
        op.flops_add = 0
        op.flops_mul = 0
        ne, nv = self.grid.macro.n_elements, self._nvol
        if self.is_tensor or self.variant == "const" or nv == 0:
            w = np.stack([self.stencil_weights(t) for t in range(ne)]) if ne else \
                np.zeros((0, nv, 15))
            torch = require_cuda()
            dev = torch.as_tensor(np.ascontiguousarray(w), device="cuda").reshape(-1)
        else:
            D = self._device()
            torch = D["torch"]
            dev = torch.empty(ne * nv * 15, dtype=torch.float64, device="cuda")
            var = _lib.VAR["nodal"] if self.variant == "nodal" else _lib.VAR["scaling"]
            coef = D["coef"] if self.variant == "nodal" else D["sh"]
            check(lib.hhg_dump_stencils(D["grid"].ref, var, coef.data_ptr(), dev.data_ptr(),
                                        self._stream()), "dump_stencils")
        op._stored = _StoredWeights(dev, ne, nv)
        op.bytes_required = ne * nv * 15 * 8
        # the twin shares this operator's device grid / surface tables
        op._dev = dict(self._device())
        op._dev["w"] = dev
        return op
