"""TEST INFRASTRUCTURE: assembled-matrix oracle and CPU operator restatement.

``assemble_global`` restates /root/reference/pkg/src/hhgscale/oracle.py:57-159:
an element loop over every fine tetrahedron of every macro element, the
Hadamard factor form of Lemma 3.2 — edge means
0.5 (k_i + k_j) off the diagonal, zero row sums (scaling), or the element
mean of k times the constant-coefficient matrix (nodal) — and identity rows
on Dirichlet nodes.  Element stiffness matrices use a face-normal formula of
their own (not the product's inverse-Jacobian code), so the check is
independent of the setup code it verifies.

``CpuOperator`` restates Operator.apply / residual / smooth
(operators.py:485-536): surface rows from an element-assembled shell CSR,
volume rows through the C kernels of liboracle.so, Dirichlet identity.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import kernels as ok

_LOCAL_EDGES = ((0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3))
_OPP_FACE = ((1, 2, 3), (0, 2, 3), (0, 1, 3), (0, 1, 2))


def stiffness(verts, cc=None):
    """P1 stiffness of a batch of tetrahedra (m, 4, 3) from face normals:
    grad(lambda_i) = N_i / (N_i . (x_i - x_f)) with N_i the normal of the
    face opposite vertex i and x_f any vertex of that face.  With a constant
    3x3 tensor ``cc`` the entries are vol * grad_i . cc grad_j."""
    verts = np.asarray(verts, dtype=np.float64)
    m = verts.shape[0]
    grads = np.empty((m, 4, 3))
    for i, (a, b, c) in enumerate(_OPP_FACE):
        N = np.cross(verts[:, b] - verts[:, a], verts[:, c] - verts[:, a])
        h = np.einsum("md,md->m", N, verts[:, i] - verts[:, a])
        grads[:, i] = N / h[:, None]
    e1, e2, e3 = (verts[:, q] - verts[:, 0] for q in (1, 2, 3))
    vol = np.abs(np.einsum("md,md->m", e1, np.cross(e2, e3))) / 6.0
    if cc is None:
        return np.einsum("mid,mjd->mij", grads, grads) * vol[:, None, None]
    return np.einsum("mid,de,mje->mij", grads, np.asarray(cc), grads) * vol[:, None, None]


def _tensor_element_matrices(coeff, t, lidx, verts, form):
    """Sum over the M components of the factored component matrices
    (oracle.py:90-110): k_m rides on grad (m = 0) or on c_m . grad."""
    A = None
    for m, fld in enumerate(coeff.fields):
        kel = fld.values[t][lidx]
        A_m = stiffness(verts) if m == 0 else stiffness(
            verts, np.outer(coeff.dirs[m], coeff.dirs[m]))
        if form == "nodal":
            part = kel.mean(axis=1)[:, None, None] * A_m
        else:
            part = 0.5 * (kel[:, :, None] + kel[:, None, :]) * A_m
        A = part if A is None else A + part
    if form != "nodal":
        idx = np.arange(4)
        A[:, idx, idx] = 0.0
        A[:, idx, idx] = -A.sum(axis=2)
    return A


def _factor(kel, A_hat, form):
    if form == "nodal":
        return kel.mean(axis=1)[:, None, None] * A_hat
    A = 0.5 * (kel[:, :, None] + kel[:, None, :]) * A_hat
    idx = np.arange(4)
    A[:, idx, idx] = 0.0
    A[:, idx, idx] = -A.sum(axis=2)
    return A


def assemble_global(grid, variant, coeff=None, hybrid_nodal=frozenset(), reduced=False,
                    shell_only=False, rows_mask=None):
    """Sparse matrix whose action is the matrix-free apply.

    variant: const | nodal | scaling | scaling_ma2 (3-D: = scaling) | hybrid.
    shell_only restricts the element loop to shell elements (enough for
    surface rows); rows_mask keeps only the selected rows (no identity rows
    added then).
    """
    from paper_1709_06793_b200.mesh import lattice_elements
    le = lattice_elements(3, grid.level, shell_only)
    lidx = grid.lat.index(le)
    rows_l, cols_l, data_l = [], [], []
    keep_rows = ~grid.dirichlet_mask if rows_mask is None else rows_mask
    for t in range(grid.macro.n_elements):
        ids = grid.elem_gidx[t][lidx]
        A_hat = stiffness(grid.node_coords[ids])
        if hasattr(coeff, "fields"):                     # tensor coefficient
            verts = grid.node_coords[ids]
            if variant == "hybrid":
                An = _tensor_element_matrices(coeff, t, lidx, verts, "nodal")
                As = _tensor_element_matrices(coeff, t, lidx, verts, "scaling")
                use = np.isin(grid.node_kind[ids], [int(k) for k in hybrid_nodal])
                A = np.where(use[:, :, None], An, As)
            else:
                A = _tensor_element_matrices(coeff, t, lidx, verts,
                                             "nodal" if variant == "nodal" else "scaling")
        elif variant == "const":
            A = (1.0 if coeff is None else float(coeff)) * A_hat
        else:
            kel = coeff.values[t][lidx]
            if variant == "nodal":
                A = _factor(kel, A_hat, "nodal")
            elif variant == "hybrid":
                An, As = _factor(kel, A_hat, "nodal"), _factor(kel, A_hat, "scaling")
                use = np.isin(grid.node_kind[ids], [int(k) for k in hybrid_nodal])
                A = np.where(use[:, :, None], An, As)
            else:
                A = _factor(kel, A_hat, "scaling")
        r = np.repeat(ids, 4, axis=1).ravel()
        c = np.tile(ids, (1, 4)).ravel()
        keep = keep_rows[r]
        rows_l.append(r[keep])
        cols_l.append(c[keep])
        data_l.append(A.ravel()[keep])
    rows = np.concatenate(rows_l) if rows_l else np.zeros(0, np.int64)
    cols = np.concatenate(cols_l) if cols_l else np.zeros(0, np.int64)
    data = np.concatenate(data_l) if data_l else np.zeros(0)
    N = grid.n_nodes
    if reduced:
        new = np.full(N, -1, dtype=np.int64)
        new[grid.interior_ids] = np.arange(grid.n_interior)
        k = new[cols] >= 0
        A = sp.coo_matrix((data[k], (new[rows[k]], new[cols[k]])),
                          shape=(grid.n_interior, grid.n_interior)).tocsr()
    else:
        if rows_mask is None:
            d = np.nonzero(grid.dirichlet_mask)[0]
            rows = np.concatenate([rows, d])
            cols = np.concatenate([cols, d])
            data = np.concatenate([data, np.ones(len(d))])
        A = sp.coo_matrix((data, (rows, cols)), shape=(N, N)).tocsr()
    A.sum_duplicates()
    return A


def rel_apply_err(out, A, u, dirichlet):
    """max |out - A u| / max |A u| with identity rows on Dirichlet nodes
    (tests/test_operators.py:47-52 convention)."""
    ref = A.dot(u)
    ref[dirichlet] = u[dirichlet]
    return float(np.abs(out - ref).max() / np.abs(ref).max())


class CpuOperator:
    """CPU restatement of Operator (volume: C kernels; surface: shell CSR)."""

    def __init__(self, grid, variant, coeff=None, hybrid_nodal=frozenset(),
                 sh=None, fac=None):
        from paper_1709_06793_b200.reference_stencils import (environment,
                                                             nodal_factors,
                                                             reference_stencil)
        self.grid, self.variant, self.coeff = grid, variant, coeff
        ne = grid.macro.n_elements
        self.env = environment(3)
        self.tensor = hasattr(coeff, "fields")
        if self.tensor:
            from paper_1709_06793_b200.reference_stencils import tensor_tables
            tabs = [tensor_tables(grid, t, coeff.dirs) for t in range(ne)]
            self.sh = [a for a, _ in tabs]
            self.fac = [b for _, b in tabs]
            self.km = [np.ascontiguousarray([f.values[t] for f in coeff.fields])
                       for t in range(ne)]
        else:
            self.sh = sh if sh is not None else [reference_stencil(grid, t)[1] / 2.0
                                                 for t in range(ne)]
            self.fac = fac if fac is not None else (
                [nodal_factors(grid, t) for t in range(ne)] if variant == "nodal" else None)
        surf = np.zeros(grid.n_nodes, dtype=bool)
        surf[:grid.n_surface_nodes] = True
        surf &= ~grid.dirichlet_mask
        self.surf_rows = np.nonzero(surf)[0]
        self.S = assemble_global(grid, variant, coeff, hybrid_nodal, shell_only=True,
                                 rows_mask=surf)
        self.nvol = grid.nodes_per_volume
        from paper_1709_06793_b200.mesh import SimplexLattice
        n = grid.n
        self.vol_pos = grid.lat.index(SimplexLattice(3, n - 4).coords + 1) if n >= 4 \
            else np.zeros(0, np.int64)

    def _volume(self, t, uloc):
        g, n = self.grid, self.grid.n
        base = g.lat.base
        if self.tensor:
            e = self.env
            if self.variant == "nodal":
                return ok.apply_nodal_tensor_3d(n, base, uloc, self.km[t], e.cse_schedule,
                                                e.cse_sums, self.fac[t], e.term_ptr,
                                                e.term_elem)
            return ok.apply_scaling_tensor_3d(n, base, uloc, self.km[t], self.sh[t])
        if self.variant == "nodal":
            e = self.env
            return ok.apply_nodal_3d(n, base, uloc, self.coeff.values[t], e.cse_schedule,
                                     e.cse_sums, self.fac[t], e.term_ptr, e.term_elem)
        if self.variant == "const":
            c = 1.0 if self.coeff is None else float(self.coeff)
            s = c * 2.0 * self.sh[t]
            return ok.apply_const_3d(n, base, uloc, s, -s.sum())
        return ok.apply_scaling_3d(n, base, uloc, self.coeff.values[t], self.sh[t])

    def apply(self, u):
        g = self.grid
        out = self.S.dot(u)
        if self.nvol:
            for t in range(g.macro.n_elements):
                s0 = g.vol_start[t]
                out[s0:s0 + self.nvol] = self._volume(t, u[g.elem_gidx[t]])
        out[g.dirichlet_mask] = u[g.dirichlet_mask]
        return out

    def residual(self, u, f):
        r = f - self.apply(u)
        r[self.grid.dirichlet_mask] = 0.0
        return r

    def smooth(self, u, f, sweeps=1, omega=1.0):
        g, n = self.grid, self.grid.n
        S = self.S
        diag = S.diagonal()
        for _ in range(sweeps):
            ok.csr_gs(self.surf_rows, S.indptr, S.indices, S.data, diag, u, f, omega)
            if not self.nvol:
                continue
            for t in range(g.macro.n_elements):
                uloc = np.ascontiguousarray(u[g.elem_gidx[t]])
                s0 = g.vol_start[t]
                fv = f[s0:s0 + self.nvol]
                if self.tensor:
                    e = self.env
                    if self.variant == "nodal":
                        ok.gs_nodal_tensor_3d(n, g.lat.base, uloc, fv, self.km[t],
                                              e.cse_schedule, e.cse_sums, self.fac[t],
                                              e.term_ptr, e.term_elem, omega)
                    else:
                        ok.gs_scaling_tensor_3d(n, g.lat.base, uloc, fv, self.km[t],
                                                self.sh[t], omega)
                elif self.variant == "nodal":
                    e = self.env
                    ok.gs_nodal_3d(n, g.lat.base, uloc, fv, self.coeff.values[t],
                                   e.cse_schedule, e.cse_sums, self.fac[t], e.term_ptr,
                                   e.term_elem, omega)
                else:
                    ok.gs_scaling_3d(n, g.lat.base, uloc, fv, self.coeff.values[t],
                                     self.sh[t], omega)
                u[s0:s0 + self.nvol] = uloc[self.vol_pos]
        return u
