// Surface rows (macro vertex / edge / face primitives), matrix free.
//
// The reference assembles these rows element-wise from the shell fine
// elements into a scipy CSR (operators.py:329-365).  Grouped by neighbour
// direction, the contribution of one incident macro element to the row of a
// boundary lattice point is the scaled stencil with a one-sided partial
// reference stencil (only patch elements inside that macro element), so a
// surface row is  sum_{incident elements} sum_d (k0+kq) psh_c[d] (vq - v0)
// (scaling) or the nodal analogue with zeroed factors for outside elements.
// One thread per row; incidences are visited in a fixed order, so results
// are deterministic run to run.
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
};

// value of lattice point (i, j, k) of element t from the global vector or the
// element's ghost shell (same addressing as the volume staging)
__device__ __forceinline__ double load_point(const SurfDesc &D, int t, int i,
                                             int j, int k) {
  const int n = D.n;
  const int rowlen = n + 1 - k - j;
  const bool inner = (k >= 1) && (j >= 1) && (k + j <= n - 2);
  if (inner && i >= 1 && i <= rowlen - 2)
    return D.u[D.vol_start[t] + lbase(n - 4, k - 1, j - 1) + i - 1];
  const double *g = D.ghost + (long long)t * D.S + D.srow[k * (n + 1) + j];
  return inner ? g[i == 0 ? 0 : 1] : g[i];
}

template <bool RES>
__global__ void surface_kernel(SurfDesc D) {
  const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r >= D.nrows) return;
  const long long gid = D.rows[r];
  const double v0 = D.u[gid];
  const bool nodal = D.row_nodal[r] != 0;
  double row = 0.0;
  for (int e = D.inc_ptr[r]; e < D.inc_ptr[r + 1]; ++e) {
    const int t = D.inc_tet[e];
    const int code = D.inc_code[e];
    const int i = code & 1023, j = (code >> 10) & 1023, k = (code >> 20) & 1023;
    const int cls = D.inc_cls[e];
    const unsigned mask = c_cls_dirmask[cls];
    const double *kt = D.kc + (long long)t * D.L;
    const double k0 = kt[lbase(D.n, k, j) + i];
    double2 q[14];
#pragma unroll
    for (int d = 0; d < 14; ++d) {
      if (mask >> d & 1) {
        const int qi = i + c_dirs[d][0], qj = j + c_dirs[d][1], qk = k + c_dirs[d][2];
        q[d].x = load_point(D, t, qi, qj, qk);
        q[d].y = kt[lbase(D.n, qk, qj) + qi];
      } else {  // outside the macro element: contributes exactly zero
        q[d].x = v0;
        q[d].y = 0.0;
      }
    }
    double part;
    if (!nodal) {
      const double *sh = D.psh + ((long long)t * 14 + cls) * 14;
      part = 0.0;
#pragma unroll
      for (int d = 0; d < 14; ++d)
        if (mask >> d & 1)
          part = dadd(part, dmul(dmul(dadd(k0, q[d].y), sh[d]), dsub(q[d].x, v0)));
    } else {
      const double *fac = D.pfac + ((long long)t * 14 + cls) * 72;
      part = nodal_row_exact(v0, k0, q, fac);
    }
    row = dadd(row, part);
  }
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
    ghost[e] = __ldg(u + gid[e]);
}

}  // namespace hhg
