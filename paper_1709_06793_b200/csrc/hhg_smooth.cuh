// Gauss-Seidel smoother kernels in the reference update order.
//
// Volume rows: the reference sweeps a macro element's interior in (k, j, i)
// lexicographic order in place (kernels.py:510-600).  Every stencil
// direction changes h = i + 2j + 3k by a nonzero amount whose sign agrees
// with lexicographic order ((1,-1,0) -> -1, (1,0,-1) -> -2, (0,1,-1) -> -1,
// (1,-1,1) -> +2, ...), so the points of one hyperplane h are mutually
// independent and see exactly the values the sequential sweep sees: a
// hyperplane wavefront is bitwise the same computation.  One CTA per macro
// element walks the hyperplanes with a block barrier between them.
//
// Surface rows: level-scheduled.  Row r depends on the rows q < r among its
// neighbours; level(r) = 1 + max level(q).  All rows of one level update in
// parallel, reading neighbour values through global ids (never the ghost
// copy, which would be stale inside a sweep).
#pragma once
#include "hhg_common.cuh"
#include "hhg_surface.cuh"

namespace hhg {

__device__ int g_status;  // HHG_OK or HHG_ERR_ZERO_DIAG

struct GSDesc {
  int n, ntets;
  long long L, S, nvol;
  const long long *vol_start;  // SPLIT: global ids; LATTICE: unused
  const int *srow;
  const double *ghost;         // SPLIT: refreshed after the surface sweep
  const double *kc;
  double *u;                   // SPLIT: global vector; LATTICE: [ntets*L]
  const double *f;             // SPLIT: global; LATTICE: [ntets*nvol]
  const double *coef;          // sh[14] or fac[72] per tet
  int coef_stride;
  double omega;
  int lattice;                 // 1: per-element lattice arrays
};

__device__ __forceinline__ double *gs_addr(const GSDesc &D, int t, int i, int j,
                                           int k, bool &ghost_pt) {
  const int n = D.n;
  if (D.lattice) {
    ghost_pt = false;
    return D.u + (long long)t * D.L + lbase(n, k, j) + i;
  }
  const int rowlen = n + 1 - k - j;
  const bool inner = (k >= 1) && (j >= 1) && (k + j <= n - 2);
  if (inner && i >= 1 && i <= rowlen - 2) {
    ghost_pt = false;
    return D.u + D.vol_start[t] + lbase(n - 4, k - 1, j - 1) + i - 1;
  }
  ghost_pt = true;
  const double *g = D.ghost + (long long)t * D.S + D.srow[k * (n + 1) + j];
  return const_cast<double *>(inner ? g + (i == 0 ? 0 : 1) : g + i);
}

template <int VAR>
__global__ void __launch_bounds__(1024)
gs_volume_kernel(GSDesc D) {
  const int t = blockIdx.x;
  const int n = D.n;
  if (n < 4) return;
  __shared__ double sfac[72];
  double coef[14];
  if (VAR == 0) {
#pragma unroll
    for (int d = 0; d < 14; ++d) coef[d] = D.coef[(long long)t * D.coef_stride + d];
  } else {
    for (int e = threadIdx.x; e < 72; e += blockDim.x)
      sfac[e] = D.coef[(long long)t * D.coef_stride + e];
    __syncthreads();
  }
  const double omega = D.omega;
  const int J = (n + 1) / 2 + 1;          // bound on points per (h, k)
  const int hmin = 6, hmax = 3 * n - 6;
  const double *kt = D.kc + (long long)t * D.L;
  for (int h = hmin; h <= hmax; ++h) {
    const int npairs = (n - 3) * J;
    for (int e = threadIdx.x; e < npairs; e += blockDim.x) {
      const int k = 1 + e / J;
      const int jlo0 = h - 2 * k - n + 1;
      const int jlo = jlo0 > 1 ? jlo0 : 1;
      const int j = jlo + e % J;
      const int i = h - 2 * j - 3 * k;
      if (i < 1 || j > n - 2 - k || i + j + k > n - 1) continue;
      bool gp;
      double *up = gs_addr(D, t, i, j, k, gp);
      const double k0 = kt[lbase(n, k, j) + i];
      double2 q[14];
#pragma unroll
      for (int d = 0; d < 14; ++d) {
        const int qi = i + c_dirs[d][0], qj = j + c_dirs[d][1], qk = k + c_dirs[d][2];
        q[d].x = *gs_addr(D, t, qi, qj, qk, gp);
        q[d].y = kt[lbase(n, qk, qj) + qi];
      }
      double acc = 0.0, diag = 0.0;
      if (VAR == 0) {
#pragma unroll
        for (int d = 0; d < 14; ++d) {
          const double sd = dmul(dadd(k0, q[d].y), coef[d]);
          acc = dadd(acc, dmul(sd, q[d].x));
          diag = dsub(diag, sd);
        }
      } else {
        double b[55];
        b[0] = k0;
#pragma unroll
        for (int d = 0; d < 14; ++d) b[1 + d] = q[d].y;
#pragma unroll
        for (int r = 0; r < 40; ++r)
          b[pt_cse(r, 0)] = dadd(b[pt_cse(r, 1)], b[pt_cse(r, 2)]);
#pragma unroll
        for (int d = 0; d < 14; ++d) {
          const int t0 = pt_tptr(d);
          double s = dmul(b[31 + pt_telem(t0)], sfac[t0]);
#pragma unroll
          for (int tt = t0 + 1; tt < pt_tptr(d + 1); ++tt)
            s = dadd(s, dmul(b[31 + pt_telem(tt)], sfac[tt]));
          acc = dadd(acc, dmul(s, q[d].x));
          diag = dsub(diag, s);
        }
      }
      if (diag == 0.0) atomicOr(&g_status, 1);
      const long long c = lbase(n - 4, k - 1, j - 1) + i - 1;
      const double fv = D.lattice ? D.f[(long long)t * D.nvol + c]
                                  : D.f[D.vol_start[t] + c];
      *up = dadd(dmul(dsub(1.0, omega), *up), ddiv(dmul(omega, dsub(fv, acc)), diag));
    }
    __syncthreads();
  }
}

// --- surface rows, one level per launch -----------------------------------
struct SurfGSDesc {
  SurfDesc s;
  const long long *shell_gid;
  const long long *level_rows;  // row indices (into s.rows) of this level
  long long count;
  double omega;
};

__device__ __forceinline__ long long point_gid(const SurfDesc &D,
                                               const long long *shell_gid,
                                               int t, int i, int j, int k) {
  const int n = D.n;
  const int rowlen = n + 1 - k - j;
  const bool inner = (k >= 1) && (j >= 1) && (k + j <= n - 2);
  if (inner && i >= 1 && i <= rowlen - 2)
    return D.vol_start[t] + lbase(n - 4, k - 1, j - 1) + i - 1;
  const long long off = (long long)t * D.S + D.srow[k * (n + 1) + j];
  return shell_gid[inner ? off + (i == 0 ? 0 : 1) : off + i];
}

__global__ void gs_surface_kernel(SurfGSDesc G) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= G.count) return;
  const SurfDesc &D = G.s;
  const long long r = G.level_rows[e];
  const long long gid = D.rows[r];
  double *u = const_cast<double *>(D.u);
  const bool nodal = D.row_nodal[r] != 0;
  double acc = 0.0, diag = 0.0;
  for (int x = D.inc_ptr[r]; x < D.inc_ptr[r + 1]; ++x) {
    const int t = D.inc_tet[x];
    const int code = D.inc_code[x];
    const int i = code & 1023, j = (code >> 10) & 1023, k = (code >> 20) & 1023;
    const int cls = D.inc_cls[x];
    const unsigned mask = c_cls_dirmask[cls];
    const double *kt = D.kc + (long long)t * D.L;
    const double k0 = kt[lbase(D.n, k, j) + i];
    double2 q[14];
#pragma unroll
    for (int d = 0; d < 14; ++d) {
      if (mask >> d & 1) {
        const int qi = i + c_dirs[d][0], qj = j + c_dirs[d][1], qk = k + c_dirs[d][2];
        q[d].x = u[point_gid(D, G.shell_gid, t, qi, qj, qk)];
        q[d].y = kt[lbase(D.n, qk, qj) + qi];
      } else {
        q[d].x = 0.0;
        q[d].y = 0.0;
      }
    }
    if (!nodal) {
      const double *sh = D.psh + ((long long)t * 14 + cls) * 14;
#pragma unroll
      for (int d = 0; d < 14; ++d)
        if (mask >> d & 1) {
          const double sd = dmul(dadd(k0, q[d].y), sh[d]);
          acc = dadd(acc, dmul(sd, q[d].x));
          diag = dsub(diag, sd);
        }
    } else {
      const double *fac = D.pfac + ((long long)t * 14 + cls) * 72;
      double b[55];
      b[0] = k0;
#pragma unroll
      for (int d = 0; d < 14; ++d) b[1 + d] = q[d].y;
#pragma unroll
      for (int rr = 0; rr < 40; ++rr)
        b[pt_cse(rr, 0)] = dadd(b[pt_cse(rr, 1)], b[pt_cse(rr, 2)]);
#pragma unroll
      for (int d = 0; d < 14; ++d) {
        if (!(mask >> d & 1)) continue;
        const int t0 = pt_tptr(d);
        double s = dmul(b[31 + pt_telem(t0)], fac[t0]);
#pragma unroll
        for (int tt = t0 + 1; tt < pt_tptr(d + 1); ++tt)
          s = dadd(s, dmul(b[31 + pt_telem(tt)], fac[tt]));
        acc = dadd(acc, dmul(s, q[d].x));
        diag = dsub(diag, s);
      }
    }
  }
  if (diag == 0.0) atomicOr(&g_status, 1);
  const double om = G.omega;
  u[gid] = dadd(dmul(dsub(1.0, om), u[gid]), ddiv(dmul(om, dsub(D.f[gid], acc)), diag));
}

}  // namespace hhg
