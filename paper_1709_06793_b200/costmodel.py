"""Per-DoF operation counts and the memory-traffic model.

Restates `pkg/src/hhgscale/costmodel.py:36-79` (the paper's Table 4/5,
PAPER.md:1407-1551) and adds the B200 roofline bookkeeping used by bench.py:
algorithmic HBM bytes of one batched volume apply.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["OpCount", "Traffic", "analytic_count", "traffic",
           "volume_apply_bytes", "operations_table", "traffic_table",
           "replay_node", "measured_count"]


@dataclass(frozen=True)
class OpCount:
    add: int
    mul: int

    @property
    def total(self):
        return self.add + self.mul


_ANALYTIC = {
    ("scaling", 3): (41, 28),
    ("nodal", 3): (125, 86),
    ("const", 3): (14, 15),
    ("stored", 3): (14, 15),
    ("scaling", 2): (17, 12),
    ("nodal", 2): (26, 18),
    ("const", 2): (6, 7),
    ("stored", 2): (6, 7),
}


def analytic_count(variant: str, dim: int) -> OpCount:
    try:
        a, m = _ANALYTIC[(variant, dim)]
    except KeyError:
        raise KeyError(f"no operation count for variant {variant!r} in {dim}D") from None
    return OpCount(a, m)


@dataclass(frozen=True)
class Traffic:
    optimistic: int
    pessimistic: int


def traffic(variant: str, n_nodes: int) -> Traffic:
    """Stencil-weight bytes per apply over N volume nodes (3-D, Table 5)."""
    N = int(n_nodes)
    if variant == "stored":
        return Traffic(120 * N, 120 * N)
    if variant == "nodal":
        return Traffic(768 + 8 * N, 768 + 120 * N)
    if variant == "scaling":
        return Traffic(112 + 8 * N, 112 + 120 * N)
    raise KeyError(f"no traffic model for variant {variant!r}")


def volume_apply_bytes(level: int, n_tets: int, residual: bool = False) -> int:
    """Algorithmic HBM bytes of one batched volume apply (each value moved
    once): read v and k over the whole lattice of every
    macro element (interior from the global vector, shell from the ghost
    layer) and write one fp64 per volume row; a residual also reads f."""
    n = 1 << level
    lat = (n + 1) * (n + 2) * (n + 3) // 6
    nvol = (n - 1) * (n - 2) * (n - 3) // 6 if n >= 4 else 0
    per = 16 * lat + 8 * nvol + (8 * nvol if residual else 0)
    return per * n_tets


def operations_table():
    return [{"dim": d, "variant": v, "adds": a, "mults": m, "total": a + m}
            for (v, d), (a, m) in sorted(_ANALYTIC.items(), key=lambda kv: (-kv[0][1], kv[0][0]))]


def traffic_table(n_nodes: int):
    """Rows of the Table-5 traffic model for the 3-D variants at N nodes
    (costmodel.py:250-258 of the reference)."""
    out = []
    for v in ("stored", "nodal", "scaling"):
        tr = traffic(v, n_nodes)
        out.append({"variant": v, "n_nodes": int(n_nodes),
                    "bytes_optimistic": tr.optimistic, "bytes_pessimistic": tr.pessimistic})
    return out


# -- measured counts: replay one volume row on the host ------------------------

class _Tape:
    """Counts the floating-point adds (subtractions included) and multiplies
    of a host replay; the arithmetic itself is plain IEEE float64."""

    def __init__(self):
        self.adds = 0
        self.muls = 0

    def add(self, a, b):
        self.adds += 1
        return a + b

    def sub(self, a, b):
        self.adds += 1
        return a - b

    def mul(self, a, b):
        self.muls += 1
        return a * b

    def count(self):
        return OpCount(self.adds, self.muls)


def _row_points(grid, c):
    """Lattice position of volume row c and of its 14 neighbours (DIRS_3D
    order) in an element's lattice."""
    from .mesh import DIRS_3D, SimplexLattice
    n = grid.n
    inner = SimplexLattice(3, n - 4).coords[c] + 1
    lat = grid.lat
    return int(lat.index(inner)), [int(x) for x in lat.index(inner + DIRS_3D)]


def replay_node(op, u, t, c):
    """Volume row c (volume rank, HHG order) of macro element t of
    ``op.apply(u)`` recomputed on the host in the kernels' operation order
    (costmodel.py:116-212 of the reference).  Returns ``(value, OpCount)``;
    the value is bitwise what the bitwise-mode kernels write for that row."""
    grid = op.grid
    if grid.dim != 3:
        raise ValueError("replay is implemented for 3-D grids")
    if op.is_tensor and op.variant in ("scaling", "nodal"):
        raise ValueError("tensor variants have no analytic count")
    p, nb = _row_points(grid, int(c))
    v = np.asarray(u, dtype=np.float64)[grid.elem_gidx[t]]
    T = _Tape()
    variant = {"hybrid": "scaling", "scaling_ma2": "scaling"}.get(op.variant, op.variant)
    if variant in ("const", "stored"):
        # (kernels.py:22-87) c0 * v0 + sum_d s_d v_d
        if variant == "const":
            w = op.const_value * 2.0 * np.asarray(op._sh[t])
            centre = -w.sum()
        else:
            rec = np.asarray(op._stored[t][c])
            centre, w = rec[0], rec[1:]
        acc = T.mul(float(centre), float(v[p]))
        for d, q in enumerate(nb):
            acc = T.add(acc, T.mul(float(w[d]), float(v[q])))
        return acc, T.count()
    kc = op.coeff.values[t]
    v0 = float(v[p])
    if variant == "scaling":
        # (kernels.py:90-136) ((k0 + kq) sh_d) (vq - v0), summed in d order
        sh, k0 = op._sh[t], float(kc[p])
        acc = None
        for d, q in enumerate(nb):
            term = T.mul(T.mul(T.add(k0, float(kc[q])), float(sh[d])), T.sub(float(v[q]), v0))
            acc = term if acc is None else T.add(acc, term)
        return acc, T.count()
    if variant == "nodal":
        # (kernels.py:139-189) 40-add element sums, then per direction the
        # factor-weighted sums s_d and s_d (vq - v0)
        env, fac = op._env, op._fac[t]
        slots = [0.0] * env.n_slots
        slots[0] = float(kc[p])
        for d, q in enumerate(nb):
            slots[1 + d] = float(kc[q])
        for dst, a, b in env.cse_schedule:
            slots[dst] = T.add(slots[a], slots[b])
        acc = None
        for d, q in enumerate(nb):
            lo, hi = int(env.term_ptr[d]), int(env.term_ptr[d + 1])
            sd = T.mul(slots[env.cse_sums[env.term_elem[lo]]], float(fac[lo]))
            for x in range(lo + 1, hi):
                sd = T.add(sd, T.mul(slots[env.cse_sums[env.term_elem[x]]], float(fac[x])))
            term = T.mul(sd, T.sub(float(v[q]), v0))
            acc = term if acc is None else T.add(acc, term)
        return acc, T.count()
    raise ValueError(f"cannot replay variant {op.variant!r}")


def measured_count(op, max_nodes: int = 32, seed: int = 0) -> OpCount:
    """Per-row operation count measured by replaying sampled volume rows of
    every macro element (costmodel.py:215-237 of the reference); every
    sampled row must cost the same."""
    grid = op.grid
    if op._nvol == 0:
        raise ValueError("grid has no volume-interior nodes; refine further")
    rng = np.random.default_rng(seed)
    u = rng.normal(size=grid.n_nodes)
    per = max(1, max_nodes // grid.macro.n_elements)
    seen = set()
    for t in range(grid.macro.n_elements):
        for c in rng.choice(op._nvol, size=min(per, op._nvol), replace=False):
            seen.add(replay_node(op, u, t, int(c))[1])
    if len(seen) != 1:
        raise AssertionError(f"non-uniform per-node cost: {sorted((x.add, x.mul) for x in seen)}")
    return seen.pop()


def apply_step_bytes(grid, op) -> int:
    """Bytes one full device-resident Operator.apply moves with this
    implementation's data structures (bench.py's step-level roofline): the
    volume kernel (volume_apply_bytes), the ghost-layer update (gather list
    8 B + u 8 B + ghost write 8 B per shell point), the surface rows and
    the Dirichlet identity rows (8-B id, read, write).  Surface rows:
    face-tiled mode - per face point and layer (the face, and each incident
    element's layer next to it) the static coefficient 8 B + id 4 B + u 8 B,
    and the 8-B result; rows left to the precomputed rows (macro edges and
    vertices, or all rows in "csr" mode) - per entry a 4-B column, an 8-B
    weight and the 8-B neighbour value, per row its offset, id, centre
    value and result (32 B)."""
    D = op._device()
    gt = D["grid"].gt
    ds = D["surf"]
    st = ds.st
    ptr = st.entry_ptr()
    vol = volume_apply_bytes(grid.level, gt.ntets)
    ghost = 24 * gt.ntets * gt.S
    faces = getattr(ds, "faces", None)
    if faces is not None and len(faces.faces) and ds.desc.nfaces:
        npf = grid.nodes_per_face
        surf = 0
        for rec in faces.faces:
            layers = 3 if rec[0][1] >= 0 else 2
            surf += npf * (layers * 20 + 8)
        sub = np.asarray(faces.sub_rows, dtype=np.int64)
        surf += int(20 * (ptr[sub + 1] - ptr[sub]).sum() + 32 * len(sub))
    else:
        surf = 20 * int(ptr[-1]) + 32 * len(st.rows)
    dirich = 24 * len(st.dir_ids)
    return int(vol + ghost + surf + dirich)
