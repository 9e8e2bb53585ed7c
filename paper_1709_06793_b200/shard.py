"""Macro-element sharding across GPUs (one process per GPU) with the
interface exchange of the surface rows.

Partition: contiguous slabs of Kuhn cubes stacked in z, one
slab per rank (config 5: 4 x 4 x 1 cubes = 96 macro tetrahedra per GPU).
Every rank refines its own sub-mesh with a local HHG numbering; faces cut by
the partition are *not* Dirichlet (the sub-mesh gets the global boundary
faces explicitly).

Volume rows need no communication: a macro element's rows depend only on
its own lattice plus ghost shell, and the shell values of interface
primitives are duplicated consistently on both ranks.  Surface rows of the
interface primitives are sums over macro elements on both sides: each rank
computes the one-sided partial rows from its own elements (exactly what the
local surface kernel does for a face whose other side is absent), the two
ranks swap the partial values of the interface nodes (one NCCL send/recv per
neighbour per apply) and both add them in rank order, so the duplicated rows
stay bitwise identical on both sides.  Dot products count each interface
node once (owner = lower rank) and all-reduce one double.
"""
from __future__ import annotations

import numpy as np

from .mesh import MacroMesh, kuhn_blocks

__all__ = ["slab_mesh", "InterfaceMap", "exchange_partials", "owned_mask",
           "ShardedOperator", "sharded_cg", "PeerExchange"]


def slab_mesh(rank: int, world: int, nx: int = 4, ny: int = 4) -> MacroMesh:
    """Rank's slab [0,1]x[0,1]x[rank h, (rank+1) h] of nx*ny Kuhn cubes
    (h = 1/max(nx, ny)); boundary faces are those of the global box."""
    h = 1.0 / max(nx, ny)
    xs = np.linspace(0.0, nx * h, nx + 1)
    ys = np.linspace(0.0, ny * h, ny + 1)
    z0, z1 = rank * h, (rank + 1) * h
    tmp = kuhn_blocks(xs, ys, np.array([z0, z1]))
    V = tmp.vertices
    keep = []
    for f, bnd in zip(tmp.faces, tmp.boundary_face):
        if not bnd:
            continue
        z = V[f, 2]
        if np.all(z == z0) and rank > 0:
            continue                        # interface with rank - 1
        if np.all(z == z1) and rank < world - 1:
            continue                        # interface with rank + 1
        keep.append(tuple(f))
    return MacroMesh(tmp.vertices, tmp.elements, boundary_faces=keep)


class InterfaceMap:
    """Local node ids shared with the neighbour ranks, in a rank-independent
    order (lexicographic in (y, x) of the interface plane)."""

    def __init__(self, grid, rank: int, world: int, h: float):
        self.rank, self.world = rank, world
        X = grid.node_coords
        free = ~grid.dirichlet_mask
        self.neighbours = {}
        self._lower_plane = None
        for nbr, z in ((rank - 1, rank * h), (rank + 1, (rank + 1) * h)):
            if nbr < 0 or nbr >= world:
                continue
            plane = X[:, 2] == z
            if nbr < rank:
                self._lower_plane = np.nonzero(plane)[0]
            ids = np.nonzero(plane & free)[0]
            order = np.lexsort((X[ids, 0], X[ids, 1]))
            self.neighbours[nbr] = np.ascontiguousarray(ids[order])

    def owned_mask(self, n_nodes):
        """True where this rank owns the node (lower rank owns interfaces)."""
        m = np.ones(n_nodes, dtype=bool)
        if self._lower_plane is not None:
            m[self._lower_plane] = False      # incl. Dirichlet copies
        return m


def owned_mask(imap: InterfaceMap, n_nodes: int):
    return imap.owned_mask(n_nodes)


def exchange_partials(out, imap: InterfaceMap, dist, index_tensors=None):
    """Sum the one-sided interface rows of ``out`` (a torch tensor on the
    rank's device, or CPU for gloo) with the neighbours' partials; the sum
    is formed in rank order so both copies are bitwise equal."""
    import torch
    if not imap.neighbours:
        return out
    # gloo moves host tensors only: stage device vectors through host memory
    stage = out.is_cuda and dist.get_backend() == "gloo"
    native = out.is_cuda and not stage and out.dtype == torch.float64
    if native:
        from ._lib import check, lib
        st = torch.cuda.current_stream().cuda_stream
    ops, recv, ids_t = [], {}, {}
    for nbr, ids in imap.neighbours.items():
        idx = index_tensors[nbr] if index_tensors is not None else \
            torch.as_tensor(ids, device=out.device)
        if native:
            idx = idx.to(torch.int64).contiguous()
        ids_t[nbr] = idx
        if native:      # pack with the library's gather kernel
            send = torch.empty(len(idx), dtype=out.dtype, device=out.device)
            check(lib.hhg_gather(len(idx), idx.data_ptr(), out.data_ptr(), send.data_ptr(), st),
                  "gather")
        else:
            send = out.index_select(0, idx).contiguous()
        if stage:
            send = send.cpu()
        buf = torch.empty_like(send)
        recv[nbr] = (send, buf)
        ops.append(dist.P2POp(dist.isend, send, nbr))
        ops.append(dist.P2POp(dist.irecv, buf, nbr))
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    for nbr, (mine, theirs) in recv.items():
        if native:      # out[ids] = theirs + mine (lower rank first), in place
            check(lib.hhg_interface_add(len(ids_t[nbr]), ids_t[nbr].data_ptr(), mine.data_ptr(),
                                        theirs.data_ptr(), int(nbr < imap.rank), out.data_ptr(),
                                        st), "interface_add")
            continue
        total = (theirs + mine) if nbr < imap.rank else (mine + theirs)
        out.index_copy_(0, ids_t[nbr], total.to(out.device))
    return out


class PeerUnavailable(RuntimeError):
    """CUDA IPC peer mapping failed on some rank (raised on all ranks)."""


class PeerExchange:
    """Interface exchange over peer memory (NVLink / NVSwitch, CUDA IPC):
    the compute step and the transfer in one kernel.

    The surface-row kernel stores every interface row it computes straight
    into the neighbour's receive buffer (``hhg_surface_apply_csr_push``),
    a one-thread kernel fences and bumps the neighbour's arrival counter
    (``hhg_p2p_signal``), and ``hhg_p2p_pull`` waits for the neighbour's
    counter and adds the received values in rank order - the same sum as
    :func:`exchange_partials`, so both copies of an interface row stay
    bitwise equal.  Receive buffers are double-buffered by apply parity: a
    rank can only push apply e+2 after it has seen the neighbour's signal
    e+1, which the neighbour sends after finishing its pull of apply e.

    Peers are connected through CUDA IPC handles exchanged with
    ``torch.distributed`` (:meth:`connect`), or, to emulate several ranks in
    one process on one device, directly (:meth:`connect_local`); the
    emulation must run every rank's :meth:`start` before any :meth:`finish`
    so no kernel ever waits on another launch of the same GPU."""

    def __init__(self, op, imap: InterfaceMap):
        import torch
        if getattr(op, "surface_mode", "csr") == "matrix-free":
            # the pushes are stored by the precomputed-row / face-tiled
            # surface kernels only
            raise ValueError("peer exchange needs surface_mode 'csr' or 'face'")
        self.torch, self.op, self.imap = torch, op, imap
        self.rank = imap.rank
        D = op._device()
        rows = np.asarray(D["surf"].st.rows)          # ascending global ids
        self.nbrs = sorted(imap.neighbours)
        slot = np.full(max(len(rows), 1), -1, dtype=np.int32)
        base = 0
        self.base = {}
        for nb in self.nbrs:
            ids = np.asarray(imap.neighbours[nb])
            r = np.searchsorted(rows, ids)
            if len(ids) and (r.max() >= len(rows) or np.any(rows[r] != ids)):
                raise ValueError("interface node is not a free surface row")
            self.base[nb] = base
            slot[r] = base + np.arange(len(ids), dtype=np.int32)
            base += len(ids)
        dev = "cuda"
        self.slot = torch.as_tensor(slot, device=dev)
        self.ids = {nb: torch.as_tensor(imap.neighbours[nb], device=dev) for nb in self.nbrs}
        self.count = {nb: len(imap.neighbours[nb]) for nb in self.nbrs}
        # what each neighbour writes into: recv[nb] (2 parities) and its
        # arrival counter flag[nb]; own allocations so an IPC handle maps
        # exactly them
        self.recv, self.flag = {}, {}
        for nb in self.nbrs:
            self.recv[nb] = self._alloc(16 * max(self.count[nb], 1))
            self.flag[nb] = self._alloc(8)
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)
        self.peer_recv, self.peer_flag = {}, {}
        self._opened = []
        self.epoch = 0

    _owned = None

    def _alloc(self, nbytes):
        import ctypes
        from ._lib import check, lib
        p = ctypes.c_void_p()
        check(lib.hhg_device_alloc(nbytes, ctypes.byref(p)), "device_alloc")
        if self._owned is None:
            self._owned = []
        self._owned.append(p.value)
        return p.value

    def close(self):
        from ._lib import lib
        for p in self._opened:
            lib.hhg_ipc_close_handle(p)
        for p in self._owned or []:
            lib.hhg_device_free(p)
        self._opened, self._owned = [], []

    # -- connection --------------------------------------------------------
    def connect(self, dist):
        """Exchange CUDA IPC handles of the receive buffers and counters with
        the neighbours (all ranks call this collectively).  A failure on any
        rank - getting or opening a handle - raises PeerUnavailable on EVERY
        rank (the outcome is agreed through the same collectives), so callers
        can fall back to another transport without a hang."""
        import ctypes
        from ._lib import check, lib
        mine, err = {}, None
        try:
            for nb in self.nbrs:
                hr, hf = ctypes.create_string_buffer(64), ctypes.create_string_buffer(64)
                check(lib.hhg_ipc_get_handle(self.recv[nb], hr), "ipc_get_handle")
                check(lib.hhg_ipc_get_handle(self.flag[nb], hf), "ipc_get_handle")
                mine[nb] = (hr.raw, hf.raw)
        except Exception as exc:                  # noqa: BLE001 - reported to every rank
            err = f"rank {self.rank}: {exc}"
        allh = [None] * dist.get_world_size()
        dist.all_gather_object(allh, (mine, err))
        errs = [e for _, e in allh if e]
        if not errs:
            try:
                for nb in self.nbrs:
                    hr, hf = allh[nb][0][self.rank]     # nb's buffers that receive from me
                    pr, pf = ctypes.c_void_p(), ctypes.c_void_p()
                    check(lib.hhg_ipc_open_handle(hr, ctypes.byref(pr)), "ipc_open_handle")
                    self._opened.append(pr.value)
                    check(lib.hhg_ipc_open_handle(hf, ctypes.byref(pf)), "ipc_open_handle")
                    self._opened.append(pf.value)
                    self.peer_recv[nb], self.peer_flag[nb] = pr.value, pf.value
            except Exception as exc:              # noqa: BLE001
                err = f"rank {self.rank}: {exc}"
            oks = [None] * dist.get_world_size()
            dist.all_gather_object(oks, err)
            errs = [e for e in oks if e]
        if errs:
            self.close()
            raise PeerUnavailable("; ".join(errs))

    def connect_local(self, peers):
        """Single-process emulation: ``peers[nb]`` is the neighbour's
        PeerExchange on the same device."""
        for nb in self.nbrs:
            other = peers[nb]
            self.peer_recv[nb] = other.recv[self.rank]
            self.peer_flag[nb] = other.flag[self.rank]

    # -- one exchange --------------------------------------------------------
    def _push(self):
        par = self.epoch % 2
        dst = [None, None]
        for q, nb in enumerate(self.nbrs):
            dst[q] = self.peer_recv[nb] + 8 * par * max(self.count[nb], 1)
        split = self.base[self.nbrs[1]] if len(self.nbrs) > 1 else (1 << 62)
        return (self.slot.data_ptr(), dst[0], dst[1], split)

    def apply(self, u, out=None, volume_events=None):
        """A u with the interface rows completed: surface rows (with the
        pushes), the signal and the pull on a side stream while the volume
        kernel runs (Operator.apply_device's after_surface hook)."""
        from ._lib import check, lib
        self.epoch += 1
        if not self.nbrs:
            return self.op.apply_device(u, out=out, volume_events=volume_events)

        def exchange(o):
            st = self.torch.cuda.current_stream().cuda_stream
            for nb in self.nbrs:
                check(lib.hhg_p2p_signal(self.peer_flag[nb], st), "p2p_signal")
            self._pull(o, st)

        return self.op.apply_device(u, out=out, push=self._push(), after_surface=exchange,
                                    volume_events=volume_events)

    def start(self, u, out=None):
        """Apply with the interface rows pushed to the neighbours and signal
        them; returns the output (interface rows still one-sided)."""
        from ._lib import check, lib
        self.epoch += 1
        out = self.op.apply_device(u, out=out, push=self._push() if self.nbrs else None)
        st = self.torch.cuda.current_stream().cuda_stream
        for nb in self.nbrs:
            check(lib.hhg_p2p_signal(self.peer_flag[nb], st), "p2p_signal")
        return out

    def finish(self, out):
        """Wait for the neighbours' values of this apply and complete the
        interface rows in rank order."""
        self._pull(out, self.torch.cuda.current_stream().cuda_stream)
        return out

    def _pull(self, out, st):
        from ._lib import check, lib
        par = self.epoch % 2
        for nb in self.nbrs:
            check(lib.hhg_p2p_pull(out.data_ptr(), self.ids[nb].data_ptr(), self.count[nb],
                                   self.recv[nb] + 8 * par * max(self.count[nb], 1),
                                   self.flag[nb], self.epoch, int(nb < self.rank),
                                   self.err.data_ptr(), st), "p2p_pull")

    def check(self):
        """Raise if a pull timed out (call after synchronising)."""
        if int(self.err.item()):
            raise RuntimeError("peer exchange: neighbour values did not arrive")


class ShardedOperator:
    """One rank's share of a partitioned operator: the local slab operator
    plus the interface exchange.

    ``op`` is the rank's :class:`~.operators.Operator` (device path) or, for
    the CPU multi-process tests, any object with ``apply(u) -> ndarray`` on
    the rank's local numbering.  Vectors are torch tensors (CUDA for the
    device path, CPU for gloo).  On the device the surface rows are launched
    first and the exchange runs on a side stream while the volume kernel
    computes the (communication-free) volume rows."""

    def __init__(self, op, imap: InterfaceMap, dist, dirichlet_mask, transport="nccl"):
        import torch
        self.op, self.imap, self.dist = op, imap, dist
        self.torch = torch
        self._idx, self._masks = {}, {}
        if transport not in ("nccl", "p2p"):
            raise ValueError("transport must be 'nccl' or 'p2p'")
        self.peer = None
        if transport == "p2p":
            self.peer = PeerExchange(op, imap)
            self.peer.connect(dist)
        self._dirichlet = np.asarray(dirichlet_mask, dtype=bool)
        self._owned = imap.owned_mask(len(self._dirichlet)) & ~self._dirichlet

    def _index(self, device):
        key = str(device)
        if key not in self._idx:
            self._idx[key] = {k: self.torch.as_tensor(v, device=device)
                              for k, v in self.imap.neighbours.items()}
        return self._idx[key]

    def _mask(self, name, device):
        key = (name, str(device))
        if key not in self._masks:
            m = self._owned if name == "owned" else ~self._dirichlet
            self._masks[key] = self.torch.as_tensor(m.astype(np.float64), device=device)
        return self._masks[key]

    def apply(self, u):
        """A u with the interface rows completed (identity Dirichlet rows)."""
        torch = self.torch
        if u.is_cuda and self.peer is not None:
            return self.peer.apply(u)
        if u.is_cuda and hasattr(self.op, "apply_device"):
            idx = self._index(u.device)
            # runs on the operator's side stream right after the surface
            # rows, concurrently with the volume kernel
            return self.op.apply_device(
                u, after_surface=lambda out: exchange_partials(out, self.imap, self.dist, idx))
        out = torch.from_numpy(np.asarray(self.op.apply(u.numpy()), dtype=np.float64))
        return exchange_partials(out, self.imap, self.dist, self._index(out.device))

    def check(self):
        """Raise if a peer-memory exchange timed out (call after a host sync)."""
        if self.peer is not None:
            self.peer.check()

    def residual(self, u, f):
        """f - A u, zero on Dirichlet rows."""
        return (f - self.apply(u)) * self._mask("free", u.device)

    def dot(self, a, b, out=None):
        """Global dot: every shared node counted once (owner = lower rank),
        Dirichlet entries excluded, one all-reduce of one double.  On the
        device: the owner-masked dot kernel into a device scalar (``out``,
        kept on the device: no host round trip)."""
        if a.is_cuda:
            from .multigrid import DeviceVec
            if getattr(self, "_vec", None) is None:
                self._vec = DeviceVec(self.torch)
            m = self._mask_u8(a.device)
            if out is None:
                out = self.torch.zeros(1, dtype=self.torch.float64, device=a.device)
            self._vec.dot_masked(a, b, m, out)
            self.dist.all_reduce(out)
            return out
        local = (a * b * self._mask("owned", a.device)).sum().reshape(1)
        self.dist.all_reduce(local)
        return local

    def _mask_u8(self, device):
        key = ("owned_u8", str(device))
        if key not in self._masks:
            self._masks[key] = self.torch.as_tensor(self._owned.astype(np.uint8), device=device)
        return self._masks[key]


def sharded_cg(sop: ShardedOperator, f, tol=1e-10, max_iter=10000):
    """Plain CG on the partitioned system (the reference's _cg,
    multigrid.py:169-194, with global dots): stop when ||r|| <= tol ||b||.
    Returns (x, iterations, final residual norm).

    Device vectors: every update is a fused kernel with its scalars in
    device memory (hhg_cg_update: x += a p, r -= a Ap and the owned partial
    of r.r; hhg_xpay_ratio), dots are owner-masked with one all-reduce of a
    device scalar, and the only host read per iteration is the stopping
    test.  CPU vectors (gloo tests): the same sequence in torch."""
    torch = sop.torch
    free = sop._mask("free", f.device)
    x = torch.zeros_like(f)
    r = f * free
    p = r.clone()
    if f.is_cuda:
        return _sharded_cg_device(sop, x, r, p, tol, max_iter)
    rs = sop.dot(r, r)
    b0 = float(torch.sqrt(rs).item())
    sop.check()
    if b0 == 0.0:
        return x, 0, 0.0
    it, res = 0, b0
    for it in range(1, max_iter + 1):
        Ap = sop.apply(p) * free
        alpha = rs / sop.dot(p, Ap)
        x = x + alpha * p
        r = r - alpha * Ap
        rs_new = sop.dot(r, r)
        res = float(torch.sqrt(rs_new).item())
        sop.check()                       # host sync point: lost peer signals raise
        if res <= tol * b0:
            break
        p = r + (rs_new / rs) * p
        rs = rs_new
    return x, it, res


def _sharded_cg_device(sop, x, r, p, tol, max_iter):
    torch = sop.torch
    from .multigrid import DeviceVec
    V = DeviceVec(torch)
    sc = torch.zeros(4, dtype=torch.float64, device=x.device)
    rs, pAp, rs_new = sc[0:1], sc[1:2], sc[2:3]
    host = torch.zeros(1, dtype=torch.float64, pin_memory=True)
    sop.dot(r, r, out=rs)
    b0 = float(np.sqrt(rs.item()))
    sop.check()
    if b0 == 0.0:
        return x, 0, 0.0
    owned = sop._mask_u8(x.device)
    it, res = 0, b0
    for it in range(1, max_iter + 1):
        # p's Dirichlet entries stay 0 (r starts 0 there and every update
        # keeps it), so the identity Dirichlet rows of A p are 0 as well
        Ap = sop.apply(p)
        sop.dot(p, Ap, out=pAp)
        V.cg_update(rs, pAp, p, Ap, x, r, rs_new, owned)   # owned partial of r.r
        sop.dist.all_reduce(rs_new)
        host.copy_(rs_new, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        res = float(np.sqrt(host.item()))
        sop.check()                       # host sync point: lost peer signals raise
        if res <= tol * b0:
            break
        V.xpay(rs_new, rs, r, p)
        rs.copy_(rs_new)
    return x, it, res
