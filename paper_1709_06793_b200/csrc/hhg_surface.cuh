// Surface rows (macro vertex / edge / face primitives), matrix free.
//
// The reference assembles these rows element-wise from the shell fine
// elements into a scipy CSR (operators.py:329-365).  Grouped by neighbour
// direction, the contribution of one incident macro element to the row of a
// boundary lattice point is the scaled stencil with a one-sided partial
// reference stencil (only patch elements inside that macro element), so a
// surface row is  sum_{incident elements} sum_d (k0+kq) psh_c[d] (vq - v0)
// (scaling) or the nodal analogue with zeroed factors for outside elements.
// Two passes (one thread per incidence, then one per row); incidences are
// summed in a fixed order, so results are deterministic run to run.  The
// default apply path precomputes these rows instead (hhg_smooth.cuh).
#pragma once
#include "hhg_common.cuh"

namespace hhg {

struct SurfDesc {
  int n;
  long long L, S, nrows;
  const long long *vol_start;
  const int *srow;
  const double *ghost, *kc, *u, *f;
  double *out;
  const long long *rows;
  const unsigned char *row_nodal;
  const int *inc_ptr, *inc_tet, *inc_code;
  const unsigned char *inc_cls;
  const double *psh, *pfac;
  // element-major incidences
  long long ninc;
  const int *p_tet, *p_code;
  const unsigned char *p_cls, *p_nodal;
  const int *row_inc;
  double *partial;
};

// Lattice addressing of one incidence (point (i, j, k) of element t) and
// its in-element neighbours, all in 32-bit closed forms.  Plane index
// a = dk + 1 selects the precomputed constants of planes k-1, k, k+1.
struct IncPlanes {
  int kb[3], rk[3];   // lattice:  base(q, j) = kb + j*rk - j(j-1)/2
  int ib[3], ri[3];   // inner lattice of the volume block (plane q-1)
  int gb[3];          // shell offset of plane q (q >= 1)
};

__device__ __forceinline__ IncPlanes inc_planes(int n, int k) {
  IncPlanes P;
  const int m4 = n - 4;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const int q = k - 1 + a;
    P.kb[a] = tetra32(n) - tetra32(n - q);
    P.rk[a] = n + 1 - q;
    P.ib[a] = (q >= 1) ? tetra32(m4) - tetra32(m4 - (q - 1)) : 0;
    P.ri[a] = n - 2 - q;
    P.gb[a] = (q >= 1) ? (n + 1) * (n + 2) / 2 + 3 * ((q - 1) * n - (q - 1) * q / 2) : 0;
  }
  return P;
}

__device__ __forceinline__ int inc_koff(const IncPlanes &P, int a, int qi, int qj) {
  return P.kb[a] + qj * P.rk[a] - qj * (qj - 1) / 2 + qi;
}

// offset of a lattice point's value: interior -> volume block (returns
// true), shell -> compact ghost shell (returns false)
__device__ __forceinline__ bool inc_voff(const IncPlanes &P, int a, int n, int qi, int qj,
                                         int qk, int &off) {
  const bool interior = qk >= 1 && qj >= 1 && qi >= 1 && qi + qj + qk <= n - 1;
  if (interior) {
    const int jj = qj - 1;
    off = P.ib[a] + jj * P.ri[a] - jj * (jj - 1) / 2 + qi - 1;
  } else if (qk == 0) {
    off = qj * (n + 1) - qj * (qj - 1) / 2 + qi;
  } else {
    off = P.gb[a] + (qj == 0 ? qi : (n + 1 - qk) + 2 * (qj - 1) + (qi > 0 ? 1 : 0));
  }
  return interior;
}

// neighbour (v, k) pairs of one incidence for the apply; directions that
// leave the macro element get (v0, 0) so they contribute exactly zero
__device__ __forceinline__ void inc_gather(const SurfDesc &D, int t, int i, int j, int k,
                                           unsigned mask, double v0, double2 (&q)[14],
                                           double &k0) {
  const int n = D.n;
  const IncPlanes P = inc_planes(n, k);
  const double *kt = D.kc + (long long)t * D.L;
  const double *ut = D.u + D.vol_start[t];
  const double *gt = D.ghost + (long long)t * D.S;
  k0 = kt[inc_koff(P, 1, i, j)];
#pragma unroll
  for (int d = 0; d < 14; ++d) {
    const int di = c_dirs_h(d, 0), dj = c_dirs_h(d, 1), dk = c_dirs_h(d, 2);
    const int qi = i + di, qj = j + dj, qk = k + dk;
    if (mask >> d & 1) {
      int off;
      const bool in = inc_voff(P, dk + 1, n, qi, qj, qk, off);
      q[d].x = in ? ut[off] : gt[off];
      q[d].y = kt[inc_koff(P, dk + 1, qi, qj)];
    } else {
      q[d].x = v0;
      q[d].y = 0.0;
    }
  }
}

// pass 1: one thread per incidence in element-major (lattice) order — the
// one-sided partial row of that boundary point; its own value comes from
// the ghost shell, so neighbouring threads read neighbouring lattice points
template <bool MIXED>
__global__ void __launch_bounds__(128)
surface_partial_kernel(SurfDesc D) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= D.ninc) return;
  const int t = D.p_tet[e];
  const int code = D.p_code[e];
  const int i = code & 1023, j = (code >> 10) & 1023, k = (code >> 20) & 1023;
  const int cls = D.p_cls[e];
  const unsigned mask = c_cls_dirmask[cls];
  const int n = D.n;
  const IncPlanes P = inc_planes(n, k);
  int off;
  inc_voff(P, 1, n, i, j, k, off);            // a boundary point: shell offset
  const double v0 = D.ghost[(long long)t * D.S + off];
  double2 q[14];
  double k0;
  inc_gather(D, t, i, j, k, mask, v0, q, k0);
  double part;
  if (!MIXED || !D.p_nodal[e]) {
    const double *sh = D.psh + ((long long)t * 14 + cls) * 14;
    part = 0.0;
#pragma unroll
    for (int d = 0; d < 14; ++d)
      if (mask >> d & 1)
        part = dadd(part, dmul(dmul(dadd(k0, q[d].y), __ldg(sh + d)), dsub(q[d].x, v0)));
  } else {
    const double *fac = D.pfac + ((long long)t * 14 + cls) * 72;
    part = nodal_row_exact(v0, k0, q, fac);
  }
  D.partial[e] = part;
}

// pass 2: one thread per free surface row, partials summed in element
// order (the association of surface_csr_kernel, hhg_smooth.cuh)
template <bool RES>
__global__ void surface_reduce_kernel(SurfDesc D) {
  const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r >= D.nrows) return;
  double row = 0.0;
  for (int x = D.inc_ptr[r]; x < D.inc_ptr[r + 1]; ++x)
    row = dadd(row, D.partial[D.row_inc[x]]);
  const long long gid = D.rows[r];
  if (RES) row = dsub(D.f[gid], row);
  D.out[gid] = row;
}

// Dirichlet rows act as the identity (operators.py:497); residual rows are 0
template <bool RES>
__global__ void dirichlet_kernel(long long nd, const long long *ids,
                                 const double *u, double *out) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= nd) return;
  const long long g = ids[e];
  out[g] = RES ? 0.0 : u[g];
}

__global__ void ghost_kernel(long long total, const long long *gid,
                             const double *u, double *ghost) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x)
  {
    HHG_BOUND(gid[e], 0, 1LL << 40, "ghost update: global id");
    ghost[e] = __ldg(u + gid[e]);
  }
}

}  // namespace hhg
