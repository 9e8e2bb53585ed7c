"""Per-DoF operation counts and the memory-traffic model.

Restates `pkg/src/hhgscale/costmodel.py:36-79` (the paper's Table 4/5,
PAPER.md:1407-1551) and adds the B200 roofline bookkeeping used by bench.py:
algorithmic HBM bytes of one batched volume apply.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["OpCount", "Traffic", "analytic_count", "traffic",
           "volume_apply_bytes", "operations_table"]


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
