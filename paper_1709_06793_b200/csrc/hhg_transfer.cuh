// Lattice-native grid transfers (multigrid.py:23-77, 130-138): linear
// interpolation from level l-1 to level l and its transpose.
//
// In every macro element the fine lattice is the coarse one refined once: a
// fine point F with even coordinates is the coarse point F/2 (weight 1); any
// other fine point is the midpoint of the one coarse edge whose direction d
// has F's coordinate parity (7 parities <-> the 7 positive stencil
// directions), parents (F - d)/2 and (F + d)/2 (weights 1/2).
//
//  * prolongation, fine volume rows: one thread per fine interior point,
//    parents addressed in closed form (coarse volume block, or the coarse
//    element's ghost-shell id table for parents on its boundary);
//  * restriction, coarse volume rows: a coarse interior point's children
//    are 2C and 2C +- d, all interior fine points of the same element, read
//    in ascending fine id - the order of the reference's P^T product
//    (scipy csc matvec: y[i] += P[j, i] x[j] over j ascending), so the sum is
//    bitwise the reference's;
//  * rows of surface nodes (vertices / edges / faces, a few percent) from a
//    small host-built CSR (hhg_transfer.{p,r}_*), through hhg_csr_spmv.
#pragma once
#include "../../include/hhg_b200.h"
#include "hhg_common.cuh"

namespace hhg {

// coarse global id of coarse lattice point (i, j, k) of element t
__device__ __forceinline__ long long coarse_gid(const hhg_transfer &T, int t, int i, int j,
                                                int k) {
  const int n = T.nc;
  if (i >= 1 && j >= 1 && k >= 1 && i + j + k <= n - 1)
    return T.c_vol_start[t] + lbase32(n - 4, k - 1, j - 1) + i - 1;
  const bool two = k >= 1 && j >= 1 && k + j <= n - 2;   // rows stored as end points
  return T.c_shell_gid[(long long)t * T.c_shell_size + srow32(n, k, j) +
                       (two ? (i == 0 ? 0 : 1) : i)];
}

// parity code (i & 1) | (j & 1) << 1 | (k & 1) << 2 -> positive direction
__constant__ int8_t c_par_dir[8][3] = {{0, 0, 0}, {1, 0, 0},  {0, 1, 0},  {1, -1, 0},
                                      {0, 0, 1}, {1, 0, -1}, {0, 1, -1}, {1, -1, 1}};

// fine volume rows: y = P x (accumulate: y += P x); grid (planes, elements)
__global__ void prolong_volume_kernel(hhg_transfer T, const double *__restrict__ xc,
                                      double *__restrict__ yf, int accumulate) {
  const int t = blockIdx.y, k = 1 + blockIdx.x;
  const int nf = T.nf;
  if (k > nf - 3) return;
  const long long plane = T.f_vol_start[t] + lbase32(nf - 4, k - 1, 0);
  // interior rows j = 1 .. nf-2-k of plane k, row j has nf-1-j-k points
  int off = 0;
  for (int j = 1; j <= nf - 2 - k; ++j) {
    const int len = nf - 1 - j - k;
    for (int i0 = threadIdx.x; i0 < len; i0 += blockDim.x) {
      const int i = 1 + i0;
      const int code = (i & 1) | (j & 1) << 1 | (k & 1) << 2;
      double s;
      if (code == 0) {
        s = xc[coarse_gid(T, t, i >> 1, j >> 1, k >> 1)];
      } else {
        const int di = c_par_dir[code][0], dj = c_par_dir[code][1], dk = c_par_dir[code][2];
        const double lo = xc[coarse_gid(T, t, (i - di) >> 1, (j - dj) >> 1, (k - dk) >> 1)];
        const double hi = xc[coarse_gid(T, t, (i + di) >> 1, (j + dj) >> 1, (k + dk) >> 1)];
        s = dadd(dmul(0.5, lo), dmul(0.5, hi));
      }
      const long long g = plane + off + i0;
      yf[g] = accumulate ? dadd(yf[g], s) : s;
    }
    off += len;
  }
}

// the 15 children of a coarse interior point C: 2C + o, sorted by the fine
// (k, j, i) numbering (ascending fine id); weight 1 for o = 0, else 1/2
__constant__ int8_t c_child[15][3] = {
    {0, 0, -1}, {1, 0, -1}, {-1, 1, -1}, {0, 1, -1}, {0, -1, 0}, {1, -1, 0}, {-1, 0, 0},
    {0, 0, 0},  {1, 0, 0},  {-1, 1, 0},  {0, 1, 0},  {0, -1, 1}, {1, -1, 1}, {-1, 0, 1},
    {0, 0, 1}};

// coarse volume rows: y = P^T x; grid (coarse planes, elements)
__global__ void restrict_volume_kernel(hhg_transfer T, const double *__restrict__ xf,
                                       double *__restrict__ yc) {
  const int t = blockIdx.y, k = 1 + blockIdx.x;
  const int nc = T.nc, nf = T.nf;
  if (k > nc - 3) return;
  const long long cplane = T.c_vol_start[t] + lbase32(nc - 4, k - 1, 0);
  const long long fbase = T.f_vol_start[t];
  int off = 0;
  for (int j = 1; j <= nc - 2 - k; ++j) {
    const int len = nc - 1 - j - k;
    for (int i0 = threadIdx.x; i0 < len; i0 += blockDim.x) {
      const int i = 1 + i0;
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < 15; ++c) {
        const int fi = 2 * i + c_child[c][0], fj = 2 * j + c_child[c][1],
                  fk = 2 * k + c_child[c][2];
        const double x = xf[fbase + lbase32(nf - 4, fk - 1, fj - 1) + fi - 1];
        acc = dadd(acc, dmul(c == 7 ? 1.0 : 0.5, x));
      }
      yc[cplane + off + i0] = acc;
    }
    off += len;
  }
}

}  // namespace hhg
