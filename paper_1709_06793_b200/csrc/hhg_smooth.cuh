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
#include <cooperative_groups.h>

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
  const int *hp_ptr;           // [3n-4] hyperplane h = 6 + idx -> point range
  const int *hp_code;          // [nvol] i | j << 10 | k << 20, by hyperplane
  int cpt;                     // CTAs per element (> 1: cooperative launch)
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

// block size: the nodal row's 55-slot buffer needs > 64 registers
template <int VAR, bool COOP>
constexpr int gs_volume_threads() { return COOP ? 128 : 256; }

// One macro element per CTA group: D.cpt co-resident CTAs share an
// element (blockIdx.x = t * cpt + c) and split every hyperplane's points;
// a barrier separates the hyperplanes - the CTA barrier when cpt == 1,
// else a grid-wide barrier of the cooperative launch (the sweep stays
// bitwise the lexicographic one: points of one hyperplane are independent,
// and all elements' volume rows are independent given the ghost shells).
// Values another CTA wrote in the previous hyperplane are read with
// ld.global.cg (no stale L1 copy); own-element k is read-only.
template <int VAR, bool COOP>
__global__ void __launch_bounds__(gs_volume_threads<VAR, COOP>(), COOP ? 2 : 1)
gs_volume_kernel(GSDesc D) {
  const int cpt = COOP ? D.cpt : 1;
  const int t = blockIdx.x / cpt;
  const int part = blockIdx.x - t * cpt;
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
  const int hmin = 6, hmax = 3 * n - 6;
  const double *kt = D.kc + (long long)t * D.L;
  const int stride = cpt * blockDim.x;
  const int first = part * blockDim.x + threadIdx.x;
  double *ut = D.lattice ? D.u + (long long)t * D.L : D.u + D.vol_start[t];
  const double *gt = D.ghost + (long long)t * D.S;
  const double *ft = D.lattice ? D.f + (long long)t * D.nvol : D.f + D.vol_start[t];

  // static part of a point (code, k at the point and its neighbours, f):
  // for the thread's first point of the next hyperplane it is loaded
  // before the barrier, so only the neighbour values remain behind it
  struct Static {
    int code;
    double k0, fv;
    double kq[14];
  };
  auto load_static = [&](int e, Static &S) {
    S.code = __ldg(D.hp_code + e);
    const int i = S.code & 1023, j = (S.code >> 10) & 1023, k = (S.code >> 20) & 1023;
    const IncPlanes P = inc_planes(n, k);
    S.k0 = __ldg(kt + inc_koff(P, 1, i, j));
#pragma unroll
    for (int d = 0; d < 14; ++d)
      S.kq[d] = __ldg(kt + inc_koff(P, c_dirs_h(d, 2) + 1, i + c_dirs_h(d, 0),
                                    j + c_dirs_h(d, 1)));
    S.fv = __ldg(ft + lbase32(n - 4, k - 1, j - 1) + i - 1);
  };
  auto update = [&](const Static &S) {
    const int i = S.code & 1023, j = (S.code >> 10) & 1023, k = (S.code >> 20) & 1023;
    const IncPlanes P = inc_planes(n, k);
    double *up;
    if (D.lattice) {
      up = ut + inc_koff(P, 1, i, j);
    } else {
      int off;
      inc_voff(P, 1, n, i, j, k, off);              // interior point
      up = ut + off;
    }
    double2 q[14];
#pragma unroll
    for (int d = 0; d < 14; ++d) {
      const int dk = c_dirs_h(d, 2);
      const int qi = i + c_dirs_h(d, 0), qj = j + c_dirs_h(d, 1), qk = k + dk;
      if (D.lattice) {
        const int ko = inc_koff(P, dk + 1, qi, qj);
        q[d].x = COOP ? __ldcg(ut + ko) : ut[ko];
      } else {
        int off;
        const bool in = inc_voff(P, dk + 1, n, qi, qj, qk, off);
        q[d].x = in ? (COOP ? __ldcg(ut + off) : ut[off]) : __ldg(gt + off);
      }
      q[d].y = S.kq[d];
    }
    double acc = 0.0, diag = 0.0;
    if (VAR == 0) {
#pragma unroll
      for (int d = 0; d < 14; ++d) {
        const double sd = dmul(dadd(S.k0, q[d].y), coef[d]);
        acc = dadd(acc, dmul(sd, q[d].x));
        diag = dsub(diag, sd);
      }
    } else {
      double b[55];
      nodal_buffer(S.k0, q, b);
      nodal_gs_terms<0>(acc, diag, q, b, sfac);
    }
    if (diag == 0.0) atomicOr(&g_status, 1);
    const double old = COOP ? __ldcg(up) : *up;
    *up = dadd(dmul(dsub(1.0, omega), old), ddiv(dmul(omega, dsub(S.fv, acc)), diag));
  };

  Static pre;
  bool have = hmin <= hmax && D.hp_ptr[0] + first < D.hp_ptr[1];
  if (have) load_static(D.hp_ptr[0] + first, pre);
  for (int h = hmin; h <= hmax; ++h) {
    const int ha = D.hp_ptr[h - hmin], hb = D.hp_ptr[h - hmin + 1];
    if (have) update(pre);
    for (int e = ha + first + stride; e < hb; e += stride) {
      Static S;
      load_static(e, S);
      update(S);
    }
    if (h < hmax) {
      const int na = D.hp_ptr[h + 1 - hmin], nb = D.hp_ptr[h + 2 - hmin];
      have = na + first < nb;
      if (have) load_static(na + first, pre);
    }
    if constexpr (COOP) cooperative_groups::this_grid().sync();
    else __syncthreads();
  }
}

// Cluster form of the volume sweep: one thread-block cluster of CL CTAs per
// macro element (elements are independent given their ghost shells, so no
// grid-wide barrier is needed - clusters of different elements run and
// finish independently), a hardware cluster barrier (release / acquire,
// cluster scope) between hyperplanes, values written by other CTAs of the
// cluster read through L2 (ld.global.cg).  Each thread takes its points of
// a hyperplane two at a time and issues both points' neighbour loads before
// either update, so twice the loads are in flight; the static part of the
// next hyperplane's first pair (k values, f, point code) is loaded before
// the barrier.  Same point set per hyperplane, same arithmetic: bitwise the
// lexicographic sweep.
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_nctas() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;\n" : "=r"(r));
  return r;
}

#ifndef HHG_GS_CT
#define HHG_GS_CT 128            // threads per CTA of the cluster sweep (scaling)
#endif
#ifndef HHG_GS_PRELOAD
#define HHG_GS_PRELOAD 1         // static part of the next pair loaded before the barrier
#endif
template <int VAR>
constexpr int gs_cluster_threads() { return VAR == 0 ? HHG_GS_CT : 128; }

template <int VAR>
__global__ void __launch_bounds__(gs_cluster_threads<VAR>())
gs_volume_cluster_kernel(GSDesc D) {
  const int cpt = (int)cluster_nctas();
  const int t = blockIdx.x / cpt;
  const int part = (int)cluster_ctarank();
  const int n = D.n;
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
  const int hmin = 6, hmax = 3 * n - 6;
  const double *kt = D.kc + (long long)t * D.L;
  const int stride = cpt * blockDim.x;
  const int first = part * blockDim.x + threadIdx.x;
  double *ut = D.u + D.vol_start[t];
  const double *gt = D.ghost + (long long)t * D.S;
  const double *ft = D.f + D.vol_start[t];

  struct Static {
    int code;
    double k0, fv;
    double kq[14];
  };
  auto load_static = [&](int e, Static &S) {
    S.code = __ldg(D.hp_code + e);
    const int i = S.code & 1023, j = (S.code >> 10) & 1023, k = (S.code >> 20) & 1023;
    const IncPlanes P = inc_planes(n, k);
    S.k0 = __ldg(kt + inc_koff(P, 1, i, j));
#pragma unroll
    for (int d = 0; d < 14; ++d)
      S.kq[d] = __ldg(kt + inc_koff(P, c_dirs_h(d, 2) + 1, i + c_dirs_h(d, 0),
                                    j + c_dirs_h(d, 1)));
    S.fv = __ldg(ft + lbase32(n - 4, k - 1, j - 1) + i - 1);
  };
  // neighbour values (through L2: other CTAs of the cluster write them)
  auto gather = [&](const Static &S, double (&qv)[14], int &uoff) {
    const int i = S.code & 1023, j = (S.code >> 10) & 1023, k = (S.code >> 20) & 1023;
    const IncPlanes P = inc_planes(n, k);
    inc_voff(P, 1, n, i, j, k, uoff);                     // interior point
#pragma unroll
    for (int d = 0; d < 14; ++d) {
      const int dk = c_dirs_h(d, 2);
      int off;
      const bool in = inc_voff(P, dk + 1, n, i + c_dirs_h(d, 0), j + c_dirs_h(d, 1), k + dk, off);
      qv[d] = in ? __ldcg(ut + off) : __ldg(gt + off);
    }
  };
  auto finish = [&](const Static &S, const double (&qv)[14], int uoff) {
    double2 q[14];
#pragma unroll
    for (int d = 0; d < 14; ++d) q[d] = make_double2(qv[d], S.kq[d]);
    double acc = 0.0, diag = 0.0;
    if (VAR == 0) {
#pragma unroll
      for (int d = 0; d < 14; ++d) {
        const double sd = dmul(dadd(S.k0, q[d].y), coef[d]);
        acc = dadd(acc, dmul(sd, q[d].x));
        diag = dsub(diag, sd);
      }
    } else {
      double b[55];
      nodal_buffer(S.k0, q, b);
      nodal_gs_terms<0>(acc, diag, q, b, sfac);
    }
    if (diag == 0.0) atomicOr(&g_status, 1);
    const double old = __ldcg(ut + uoff);
    __stcg(ut + uoff, dadd(dmul(dsub(1.0, omega), old), ddiv(dmul(omega, dsub(S.fv, acc)), diag)));
  };

  Static pa, pb;
  int na = 0;              // static points preloaded for the current hyperplane (0..2)
  auto preload = [&](int h) {
    const int a = D.hp_ptr[h - hmin], b = D.hp_ptr[h + 1 - hmin];
    na = 0;
    if (a + first < b) { load_static(a + first, pa); na = 1; }
    if (a + first + stride < b) { load_static(a + first + stride, pb); na = 2; }
  };
  if (HHG_GS_PRELOAD && hmin <= hmax) preload(hmin);
  for (int h = hmin; h <= hmax; ++h) {
    const int hb = D.hp_ptr[h + 1 - hmin];
    int e = D.hp_ptr[h - hmin] + first;
    if (!HHG_GS_PRELOAD) {
      e -= 2 * stride;                  // no preloaded pair: the loop takes them all
    } else if (na == 2) {
      double qa[14], qb[14];
      int oa, ob;
      gather(pa, qa, oa);
      gather(pb, qb, ob);
      finish(pa, qa, oa);
      finish(pb, qb, ob);
    } else if (na == 1) {
      double qa[14];
      int oa;
      gather(pa, qa, oa);
      finish(pa, qa, oa);
    }
    for (e += 2 * stride; e < hb; e += 2 * stride) {
      Static sa, sb;
      load_static(e, sa);
      const bool two = e + stride < hb;
      if (two) load_static(e + stride, sb);
      double qa[14], qb[14];
      int oa, ob = 0;
      gather(sa, qa, oa);
      if (two) gather(sb, qb, ob);
      finish(sa, qa, oa);
      if (two) finish(sb, qb, ob);
    }
    if (HHG_GS_PRELOAD && h < hmax) preload(h + 1);
    cluster_sync_all();
  }
}

// Skewed (hyperplane-major) form of the volume sweep.  Each element's whole
// (n+1)-lattice - interior points and the boundary points the ghost shell
// holds - is stored in hyperplane order (h = i + 2j + 3k, then k, then j;
// position xstart[h (n+1) + k] + j), u and the coefficient k as separate
// copies (us, ks: ntets * L).  One hyperplane is a contiguous run, the
// neighbours of consecutive points of a run are consecutive points of the
// neighbouring runs (direction d moves h by di + 2dj + 3dk), and - with the
// boundary layer in the same array - every neighbour of every interior
// point is addressed the same way: no bounds tests, no ghost branch, no
// divergence.  u (with the ghost values) is moved in before the sweep and
// the interior back after it (a separate pass: storing each new value into
// the global vector from the sweep - scattered 8-byte stores - measured
// 1.5x slower at level 8), f (interior order of the hyperplane lists) once
// per smoothing call, k once per operator.  Same points per
// hyperplane, same arithmetic as gs_volume_kernel: bitwise the
// lexicographic sweep.
//   MODE 0: dst[t L + p] = u or ghost value of lattice point p (gather)
//   MODE 1: u[interior p] = src[t L + p]                      (scatter)
//   MODE 2: dst[t L + p] = kc[t L + lattice(p)]               (coefficient)
// (skewed order on the write side of the gathers: the scattered 8-byte
// reads are L2 hits - one element's block is ~23 MB at level 8 - while
// scattered partial-sector writes would cost DRAM fills)
template <int MODE>
__global__ void skew_move_kernel(GSDesc D, const int *__restrict__ xcode,
                                 const double *__restrict__ src, double *__restrict__ dst) {
  const int t = blockIdx.y;
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= D.L) return;
  const int n = D.n;
  const int code = __ldg(xcode + p);
  const int i = code & 1023, j = (code >> 10) & 1023, k = (code >> 20) & 1023;
  const long long sk = (long long)t * D.L + p;
  if (MODE == 2) {
    dst[sk] = __ldg(D.kc + (long long)t * D.L + lbase32(n, k, j) + i);
    return;
  }
  if (MODE == 0) {
    bool ghost;
    GSDesc E = D;
    E.u = const_cast<double *>(src);
    dst[sk] = __ldg(gs_addr(E, t, i, j, k, ghost));
  } else if (i >= 1 && j >= 1 && k >= 1 && i + j + k <= n - 1) {
    dst[D.vol_start[t] + lbase32(n - 4, k - 1, j - 1) + i - 1] = src[sk];
  }
}

// The scatter back to u walked in u's own (volume-block) order: the
// writes fill whole sectors and the 8-byte reads of the skewed copy are
// the scattered side (L2 hits: an element's copy is ~23 MB), where
// skew_move_kernel<1> wrote u one scattered 8-byte word per thread
// (partial-sector writes: L2 at 73% of its peak, DRAM at 31%).
#ifndef HHG_SKEW_SCATTER_LAT
#define HHG_SKEW_SCATTER_LAT 1
#endif
__global__ void skew_scatter_kernel(GSDesc D, const int *__restrict__ icode,
                                    const int *__restrict__ xstart, const double *__restrict__ us,
                                    double *__restrict__ u) {
  const int t = blockIdx.y;
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= D.nvol) return;
  const int n = D.n;
  const int code = __ldg(icode + c);
  const int i = code & 1023, j = (code >> 10) & 1023, k = (code >> 20) & 1023;
  const int pos = __ldg(xstart + (i + 2 * j + 3 * k) * (n + 1) + k) + j;
  u[D.vol_start[t] + c] = __ldg(us + (long long)t * D.L + pos);
}

// refresh the boundary (ghost) points of us only: the interior is current
// (the previous sweep of the same smoothing left it equal to u)
__global__ void skew_boundary_kernel(GSDesc D, const int *__restrict__ bcode,
                                     const int *__restrict__ bpos, int nb, double *us) {
  const int t = blockIdx.y;
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const int code = __ldg(bcode + b);
  const int i = code & 1023, j = (code >> 10) & 1023, k = (code >> 20) & 1023;
  bool ghost;
  us[(long long)t * D.L + __ldg(bpos + b)] = __ldg(gs_addr(D, t, i, j, k, ghost));
}

// f in the order of the hyperplane lists (interior points only)
__global__ void skew_f_kernel(GSDesc D, const double *__restrict__ f, double *__restrict__ fs) {
  const int t = blockIdx.y;
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= D.nvol) return;
  const int n = D.n;
  const int code = __ldg(D.hp_code + e);
  const int i = code & 1023, j = (code >> 10) & 1023, k = (code >> 20) & 1023;
  fs[(long long)t * D.nvol + e] = __ldg(f + D.vol_start[t] + lbase32(n - 4, k - 1, j - 1) + i - 1);
}

template <int VAR>
__global__ void __launch_bounds__(gs_cluster_threads<VAR>())
gs_volume_skew_kernel(GSDesc D, double *us, const double *__restrict__ fs,
                      const double *__restrict__ ks, const int *__restrict__ xstart) {
  const int cpt = (int)cluster_nctas();
  const int t = blockIdx.x / cpt;
  const int part = (int)cluster_ctarank();
  const int n = D.n;
  // the element's stencil constants in shared memory (sh[14] or fac[72]):
  // broadcast reads, 28 registers fewer than a per-thread copy of sh
  __shared__ double sfac[72];
  for (int e = threadIdx.x; e < (VAR == 0 ? 14 : 72); e += blockDim.x)
    sfac[e] = D.coef[(long long)t * D.coef_stride + e];
  const double omega = D.omega;
  const int hmin = 6, hmax = 3 * n - 6;
  double *ue = us + (long long)t * D.L;
  const double *ke = ks + (long long)t * D.L;
  const double *fe = fs + (long long)t * D.nvol;
  const int stride = cpt * blockDim.x;
  const int first = part * blockDim.x + threadIdx.x;
  // ring of the xstart rows of hyperplanes h-3 .. h+3 (row hq in slot
  // hq & 7): positions come from shared memory; row h+4 is staged during
  // hyperplane h
  extern __shared__ int st_ring[];
  const int srl = n + 1;
  auto stage_row = [&](int hq) {
    if (hq > 3 * n) return;
    const int *src = xstart + hq * srl;
    int *dst = st_ring + (hq & 7) * srl;
    for (int x = threadIdx.x; x < srl; x += blockDim.x) dst[x] = __ldg(src + x);
  };
  for (int hq = hmin - 3; hq <= hmin + 3; ++hq) stage_row(hq);
  __syncthreads();
  auto point = [&](int h, int e, int code) {
    const int j = (code >> 10) & 1023, k = (code >> 20) & 1023;
    double2 q[14];
#pragma unroll
    for (int d = 0; d < 14; ++d) {
      const int di = c_dirs_h(d, 0), dj = c_dirs_h(d, 1), dk = c_dirs_h(d, 2);
      const int hq = h + di + 2 * dj + 3 * dk;
      const int pos = st_ring[(hq & 7) * srl + k + dk] + j + dj;
      HHG_BOUND(pos, 0, D.L, "skewed sweep: neighbour position");
      q[d] = make_double2(__ldcg(ue + pos), __ldg(ke + pos));
    }
    const int self = st_ring[(h & 7) * srl + k] + j;
    HHG_BOUND(self, 0, D.L, "skewed sweep: point position");
    HHG_BOUND(e, 0, D.nvol, "skewed sweep: list index");
    const double old = __ldcg(ue + self), k0 = __ldg(ke + self), fv = __ldg(fe + e);
    double acc = 0.0, diag = 0.0;
    if (VAR == 0) {
#pragma unroll
      for (int d = 0; d < 14; ++d) {
        const double sd = dmul(dadd(k0, q[d].y), sfac[d]);
        acc = dadd(acc, dmul(sd, q[d].x));
        diag = dsub(diag, sd);
      }
    } else {
      double b[55];
      nodal_buffer(k0, q, b);
      nodal_gs_terms<0>(acc, diag, q, b, sfac);
    }
    if (diag == 0.0) atomicOr(&g_status, 1);
    const double v = dadd(dmul(dsub(1.0, omega), old), ddiv(dmul(omega, dsub(fv, acc)), diag));
    __stcg(ue + self, v);
  };
  // the point code of the thread's next point is loaded one point ahead
  // (for the first point of the next hyperplane: before the barrier)
  int ha = __ldg(D.hp_ptr), hb = __ldg(D.hp_ptr + 1);
  int code = ha + first < hb ? __ldg(D.hp_code + ha + first) : 0;
  for (int h = hmin; h <= hmax; ++h) {
    for (int e = ha + first; e < hb; e += stride) {
      const int code_next = e + stride < hb ? __ldg(D.hp_code + e + stride) : 0;
      point(h, e, code);
      code = code_next;
    }
    stage_row(h + 4);
    if (h < hmax) {
      ha = hb;
      hb = __ldg(D.hp_ptr + h + 2 - hmin);
      code = ha + first < hb ? __ldg(D.hp_code + ha + first) : 0;
    }
    cluster_sync_all();
  }
}

// --- surface rows, one level per launch -----------------------------------
struct SurfGSDesc {
  SurfDesc s;
  const long long *shell_gid;
  const long long *level_rows;  // row indices (into s.rows) of this level
  long long count;
  double omega;
  // precomputed rows (hhg_smooth_surface_prepare): neighbour ids and
  // weights in the exact accumulation order, and the diagonals
  const long long *ent_ptr;
  int *ent_col;
  double *ent_val, *row_diag;
  // level-ordered slots (gs_surface_slots_kernel)
  long long nslots;
  const long long *slot_gid;
  const int *slot_cnt, *slot_col, *slot_dyn;
  const double *slot_diag, *slot_val;
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

__device__ __forceinline__ void gs_surface_row(const SurfGSDesc &G, long long r) {
  const SurfDesc &D = G.s;
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
        q[d].x = __ldcg(u + point_gid(D, G.shell_gid, t, qi, qj, qk));
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
      nodal_buffer(k0, q, b);
      nodal_gs_terms<0>(acc, diag, q, b, fac, mask);
    }
  }
  if (diag == 0.0) atomicOr(&g_status, 1);
  const double om = G.omega;
  u[gid] = dadd(dmul(dsub(1.0, om), __ldcg(u + gid)), ddiv(dmul(om, dsub(D.f[gid], acc)), diag));
}


// setup: the weights of every surface row in the order gs_surface_row
// accumulates them (incidence, then direction), and -sum of them as the
// diagonal — computed once on the device (k is fixed), bitwise the values
// gs_surface_row would recompute in every sweep
template <int D, class FAC>
__device__ __forceinline__ void nodal_row_weights(double &diag, double *&val,
                                                  const double (&b)[55], const FAC &fac,
                                                  unsigned mask) {
  if constexpr (D < 14) {
    if (mask >> D & 1) {
      const double sd = dir_sum<D>(b, fac);
      *val++ = sd;
      diag = dsub(diag, sd);
    }
    nodal_row_weights<D + 1>(diag, val, b, fac, mask);
  }
}

__global__ void gs_surface_fill_kernel(SurfGSDesc G) {
  const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const SurfDesc &D = G.s;
  if (r >= D.nrows) return;
  const bool nodal = D.row_nodal[r] != 0;
  double diag = 0.0;
  double *val = G.ent_val + G.ent_ptr[r];
  int *col = G.ent_col + G.ent_ptr[r];
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
      q[d].x = 0.0;
      q[d].y = 0.0;
      if (mask >> d & 1) {
        const int qi = i + c_dirs[d][0], qj = j + c_dirs[d][1], qk = k + c_dirs[d][2];
        q[d].y = kt[lbase(D.n, qk, qj) + qi];
        *col++ = (int)point_gid(D, G.shell_gid, t, qi, qj, qk);
      }
    }
    if (!nodal) {
      const double *sh = D.psh + ((long long)t * 14 + cls) * 14;
#pragma unroll
      for (int d = 0; d < 14; ++d)
        if (mask >> d & 1) {
          const double sd = dmul(dadd(k0, q[d].y), sh[d]);
          *val++ = sd;
          diag = dsub(diag, sd);
        }
    } else {
      const double *fac = D.pfac + ((long long)t * 14 + cls) * 72;
      double b[55];
      nodal_buffer(k0, q, b);
      nodal_row_weights<0>(diag, val, b, fac, mask);
    }
  }
  G.row_diag[r] = diag;
}

// one GS row from the precomputed list: acc = sum w u (stored order)
__device__ __forceinline__ void gs_surface_row_csr(const SurfGSDesc &G, long long r) {
  const SurfDesc &D = G.s;
  const long long gid = D.rows[r];
  double *u = const_cast<double *>(D.u);
  double acc = 0.0;
  const long long e1 = G.ent_ptr[r + 1];
  long long e = G.ent_ptr[r];
  // loads batched 8 at a time (independent), accumulation still in order
  for (; e + 8 <= e1; e += 8) {
    int cl[8];
    double w[8], x[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) cl[m] = __ldg(G.ent_col + e + m);
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      w[m] = __ldg(G.ent_val + e + m);
      x[m] = __ldcg(u + (unsigned)cl[m]);
    }
#pragma unroll
    for (int m = 0; m < 8; ++m) acc = dadd(acc, dmul(w[m], x[m]));
  }
  for (; e < e1; ++e)
    acc = dadd(acc, dmul(__ldg(G.ent_val + e), __ldcg(u + (unsigned)__ldg(G.ent_col + e))));
  const double diag = G.row_diag[r];
  if (diag == 0.0) atomicOr(&g_status, 1);
  const double om = G.omega;
  u[gid] = dadd(dmul(dsub(1.0, om), __ldcg(u + gid)), ddiv(dmul(om, dsub(D.f[gid], acc)), diag));
}

// Sharded surface sweep (shard_mg.py): the rows of one level of the global
// schedule, as explicit lists.  Rows owned by this rank alone update
// directly; a row on an interface plane is shared with the neighbour rank,
// whose macro elements contribute the other part of its sum: each rank forms
// its partial (acc over its own incidences, its part of the diagonal), the
// partials are exchanged and added in rank order, and both ranks finish
// the row with the same numbers.
__global__ void gs_surface_rows_kernel(SurfGSDesc G, const long long *rows, long long count) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e < count) gs_surface_row_csr(G, rows[e]);
}

__global__ void gs_surface_partial_kernel(SurfGSDesc G, const long long *rows, long long count,
                                          double *acc, double *diag) {
  const long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (x >= count) return;
  const long long r = rows[x];
  const double *u = G.s.u;
  double a = 0.0;
  for (long long e = G.ent_ptr[r]; e < G.ent_ptr[r + 1]; ++e)
    a = dadd(a, dmul(__ldg(G.ent_val + e), __ldcg(u + (unsigned)__ldg(G.ent_col + e))));
  acc[x] = a;
  diag[x] = G.row_diag[r];
}

__global__ void gs_surface_finish_kernel(SurfGSDesc G, const long long *rows, long long count,
                                         const double *acc, const double *diag) {
  const long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (x >= count) return;
  const long long gid = G.s.rows[rows[x]];
  double *u = const_cast<double *>(G.s.u);
  const double d = diag[x];
  if (d == 0.0) atomicOr(&g_status, 1);
  const double om = G.omega;
  u[gid] = dadd(dmul(dsub(1.0, om), __ldcg(u + gid)), ddiv(dmul(om, dsub(G.s.f[gid], acc[x])), d));
}

// apply / residual of the surface rows from the precomputed weights:
// part = sum_d w_d (v_d - v0) per incidence (direction order), row = sum of
// parts (incidence order) — the association of surface_partial_kernel +
// surface_reduce_kernel, with w_d = (k0 + k_d) * psh_d (or the nodal s_d)
// read instead of recomputed
// Interface push (multi-GPU, peer memory): rows with push_slot[r] >= 0 are
// interface rows shared with a neighbour rank; their one-sided value is
// also stored straight into that neighbour's receive buffer over NVLink
// (dst0 for slots < split, dst1 otherwise), in the same kernel that
// computes it.
struct SurfPush {
  const int *slot;      // [nrows] or nullptr
  double *dst0, *dst1;  // peer receive buffers (this apply's parity)
  long long split;
};

template <bool RES>
__global__ void surface_csr_kernel(SurfGSDesc G, double *out, long long ndir,
                                   const long long *dir_ids, SurfPush push = SurfPush{},
                                   const int *sub = nullptr, long long nsub = 0) {
  const long long x0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const SurfDesc &D = G.s;
  // rows: all of them, or the sub-list (edge / vertex rows next to the
  // face-tiled kernel); Dirichlet rows ride along after them
  const long long nr = sub ? nsub : D.nrows;
  if (x0 >= nr) {
    // Dirichlet rows: identity (0 for f - Au)
    const long long e = x0 - nr;
    if (e < ndir) {
      const long long g = dir_ids[e];
      out[g] = RES ? 0.0 : D.u[g];
    }
    return;
  }
  const long long r = sub ? (long long)sub[x0] : x0;
  const long long gid = D.rows[r];
  const double v0 = D.u[gid];
  long long e = G.ent_ptr[r];
  double row = 0.0;
  for (int x = D.inc_ptr[r]; x < D.inc_ptr[r + 1]; ++x) {
    const int cnt = __popc(c_cls_dirmask[D.inc_cls[x]]);   // 1..12 entries
    int cl[12];
    double w[12], vq[12];
#pragma unroll
    for (int m = 0; m < 12; ++m)
      if (m < cnt) cl[m] = __ldg(G.ent_col + e + m);
#pragma unroll
    for (int m = 0; m < 12; ++m)
      if (m < cnt) {
        w[m] = __ldg(G.ent_val + e + m);
        vq[m] = __ldg(D.u + (unsigned)cl[m]);
      }
    double part = dmul(w[0], dsub(vq[0], v0));
#pragma unroll
    for (int m = 1; m < 12; ++m)
      if (m < cnt) part = dadd(part, dmul(w[m], dsub(vq[m], v0)));
    e += cnt;
    row = dadd(row, part);
  }
  if (RES) row = dsub(D.f[gid], row);
  out[gid] = row;
  if (!RES && push.slot) {
    const int sl = __ldg(push.slot + r);
    if (sl >= 0) {
      if (sl < push.split) push.dst0[sl] = row;
      else push.dst1[sl - push.split] = row;
    }
  }
}

// after the pushes of this apply: make them visible system-wide, then bump
// the neighbour's arrival counter (one signal per apply and neighbour)
__global__ void p2p_signal_kernel(unsigned long long *remote_flag) {
  __threadfence_system();
  atomicAdd_system(remote_flag, 1ULL);
}

// wait until the neighbour's push of this apply has arrived: one thread of
// one CTA spins (bounded, *err set on timeout) so no spinning CTA takes SM
// slots from the volume kernel running concurrently; the adds follow as a
// separate, non-spinning launch on the same stream (p2p_add_kernel)
__global__ void p2p_wait_kernel(const unsigned long long *flag, unsigned long long target,
                                int *err) {
  if (threadIdx.x != 0) return;
  unsigned long long v = 0;
  long long spins = 0;
  for (;;) {
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
    if (v >= target) break;
    if (++spins > (1LL << 30)) break;          // ~a minute: never hang the GPU
    __nanosleep(64);
  }
  if (v < target) atomicExch(err, 1);
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}

// complete the interface rows in rank order: out = recv + mine if
// recv_first else mine + recv (bitwise the NCCL path's sum on both ranks);
// skipped after a timeout
__global__ void p2p_add_kernel(double *out, const long long *ids, long long count,
                               const double *recv, int recv_first, const int *err) {
  if (*((volatile const int *)err)) return;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    const long long g = ids[i];
    const double theirs = __ldcv(recv + i);
    const double mine = out[g];
    out[g] = recv_first ? dadd(theirs, mine) : dadd(mine, theirs);
  }
}

// kernels.csr_gs (kernels.py:979-992): forward Gauss-Seidel over the given
// rows of a CSR matrix, strictly in list order, bitwise the sequential loop
// (acc += data * u[col] in stored order, diagonal skipped).  One warp: the
// lanes load and multiply a row's entries 32 at a time, lane 0 adds the
// products in order; a zero diagonal stops the sweep at that row and sets
// the status word (the reference raises there).
__global__ void csr_gs_kernel(long long nr, const long long *rows, const long long *indptr,
                              const long long *indices, const double *data, const double *diag,
                              double *u, const double *f, double omega) {
  const int lane = threadIdx.x;
  for (long long ri = 0; ri < nr; ++ri) {
    const long long r = rows[ri];
    const long long e0 = indptr[r], e1 = indptr[r + 1];
    double acc = 0.0;
    for (long long b = e0; b < e1; b += 32) {
      const long long e = b + lane;
      double prod = 0.0;
      bool use = false;
      if (e < e1) {
        const long long c = indices[e];
        use = c != r;
        if (use) prod = dmul(data[e], __ldcv(u + c));
      }
      const unsigned m = __ballot_sync(0xffffffffu, use);
      const int cnt = (int)min(32LL, e1 - b);
      for (int x = 0; x < cnt; ++x) {
        const double px = __shfl_sync(0xffffffffu, prod, x);
        if (lane == 0 && (m >> x & 1)) acc = dadd(acc, px);
      }
    }
    const double d0 = diag[r];
    if (d0 == 0.0) {
      if (lane == 0) atomicOr(&g_status, 1);
      return;
    }
    if (lane == 0)
      __stcg(u + r, dadd(dmul(dsub(1.0, omega), __ldcv(u + r)),
                         ddiv(dmul(omega, dsub(f[r], acc)), d0)));
    __syncwarp();
    __threadfence_block();
  }
}

__global__ void gs_surface_kernel(SurfGSDesc G) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e < G.count) gs_surface_row(G, G.level_rows[e]);   // recomputing form
}

// Row of the surface sweep split in two: everything that does not depend
// on u (row id, entry range, diagonal, f, the first PF column ids and
// weights) is fetched before the grid barrier that precedes the row's
// level, so after the barrier only the neighbour values remain to be read.
constexpr int kSurfPF = 24;   // face rows have ~24 entries
struct SurfRowPF {
  long long gid, e0, e1;
  double diag, fv;
  int col[kSurfPF];
  double val[kSurfPF];
};

__device__ __forceinline__ void surf_row_prefetch(const SurfGSDesc &G, long long r,
                                                  SurfRowPF &p) {
  const SurfDesc &D = G.s;
  p.gid = __ldg(D.rows + r);
  p.e0 = __ldg(G.ent_ptr + r);
  p.e1 = __ldg(G.ent_ptr + r + 1);
  p.diag = __ldg(G.row_diag + r);
  p.fv = __ldg(D.f + p.gid);
#pragma unroll
  for (int m = 0; m < kSurfPF; ++m)
    if (p.e0 + m < p.e1) {
      p.col[m] = __ldg(G.ent_col + p.e0 + m);
      p.val[m] = __ldg(G.ent_val + p.e0 + m);
    }
}

__device__ __forceinline__ void surf_row_finish(const SurfGSDesc &G, const SurfRowPF &p) {
  double *u = const_cast<double *>(G.s.u);
  double x[kSurfPF];
#pragma unroll
  for (int m = 0; m < kSurfPF; ++m)
    if (p.e0 + m < p.e1) x[m] = __ldcg(u + (unsigned)p.col[m]);
  const double old = __ldcg(u + p.gid);
  double acc = 0.0;
#pragma unroll
  for (int m = 0; m < kSurfPF; ++m)
    if (p.e0 + m < p.e1) acc = dadd(acc, dmul(p.val[m], x[m]));
  for (long long e = p.e0 + kSurfPF; e < p.e1; ++e)
    acc = dadd(acc, dmul(__ldg(G.ent_val + e), __ldcg(u + (unsigned)__ldg(G.ent_col + e))));
  if (p.diag == 0.0) atomicOr(&g_status, 1);
  const double om = G.omega;
  u[p.gid] = dadd(dmul(dsub(1.0, om), old), ddiv(dmul(om, dsub(p.fv, acc)), p.diag));
}

// all levels in one cooperative launch: rows of a level are spread over the
// grid, a grid-wide barrier (with its memory fence) separates the levels;
// neighbour values are read with ld.global.cg so no stale L1 copy survives
// a level boundary.  Each thread's first row of the next level is
// prefetched (surf_row_prefetch) before the barrier.
__global__ void __launch_bounds__(64)
gs_surface_all_kernel(SurfGSDesc G, const long long *level_ptr, int nlev) {
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  // row m of a level goes to block m % gridDim: a narrow level still
  // spreads over all participating SMs
  const long long tid = threadIdx.x * (long long)gridDim.x + blockIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  SurfRowPF pf;
  bool have = false;
  if (nlev > 0 && level_ptr[0] + tid < level_ptr[1]) {
    surf_row_prefetch(G, G.level_rows[level_ptr[0] + tid], pf);
    have = true;
  }
  for (int lv = 0; lv < nlev; ++lv) {
    const long long a = level_ptr[lv], b = level_ptr[lv + 1];
    if (have) surf_row_finish(G, pf);
    for (long long e = a + tid + nth; e < b; e += nth) {
      surf_row_prefetch(G, G.level_rows[e], pf);
      surf_row_finish(G, pf);
    }
    have = false;
    if (lv + 1 < nlev) {
      const long long e = level_ptr[lv + 1] + tid;
      if (e < level_ptr[lv + 2]) {
        surf_row_prefetch(G, G.level_rows[e], pf);
        have = true;
      }
    }
    grid.sync();
  }
}

// The same sweep on ONE thread-block cluster, from the level-ordered slots
// (hhg_surface_gs.slot_*): a level's rows are spread over the cluster's
// CTAs; between levels a split hardware cluster barrier (arrive.release,
// then wait.acquire; cluster scope) replaces the grid barrier.  Between the
// arrive and the wait each thread fetches its next row - id, count,
// diagonal, f, column ids, weights (one coalesced load per field) - AND the
// neighbour values that cannot change before that row runs: volume and
// Dirichlet ids, rows of earlier levels (final since the last wait) and of
// later levels (still old).  Only neighbours in the level just written
// (slot_dyn bits, ~2 per row) are read after the wait.  Entries, order and
// arithmetic are gs_surface_row_csr's: bitwise the same.
constexpr int kSlotPF = HHG_SURF_SLOT_PF;
struct SlotRow {
  long long gid;
  int cnt;
  unsigned dyn;
  double diag, fv;
  int col[kSlotPF];
  double w[kSlotPF], x[kSlotPF];
};

__device__ __forceinline__ void slot_prefetch(const SurfGSDesc &G, long long e, SlotRow &p) {
  const long long ns = G.nslots;
  const double *u = G.s.u;
  p.gid = __ldg(G.slot_gid + e);
  p.cnt = __ldg(G.slot_cnt + e);
  p.dyn = (unsigned)__ldg(G.slot_dyn + e);
  p.diag = __ldg(G.slot_diag + e);
#pragma unroll
  for (int m = 0; m < kSlotPF; ++m) {   // padded slots hold (0, 0.0)
    p.col[m] = __ldg(G.slot_col + m * ns + e);
    p.w[m] = __ldg(G.slot_val + m * ns + e);
  }
  p.fv = __ldg(G.s.f + p.gid);
#pragma unroll
  for (int m = 0; m < kSlotPF; ++m)
    if (m < p.cnt && !(p.dyn >> m & 1)) p.x[m] = __ldcg(u + (unsigned)p.col[m]);
}

__device__ __forceinline__ void slot_finish(const SurfGSDesc &G, long long e, SlotRow &p) {
  double *u = const_cast<double *>(G.s.u);
#pragma unroll
  for (int m = 0; m < kSlotPF; ++m)
    if (m < p.cnt && (p.dyn >> m & 1)) p.x[m] = __ldcg(u + (unsigned)p.col[m]);
  const double old = __ldcg(u + p.gid);
  double acc = 0.0;
#pragma unroll
  for (int m = 0; m < kSlotPF; ++m)
    if (m < p.cnt) acc = dadd(acc, dmul(p.w[m], p.x[m]));
  if (p.cnt > kSlotPF) {               // long (edge / vertex) rows: the rest
    const long long r = __ldg(G.level_rows + e);
    const long long e1 = __ldg(G.ent_ptr + r + 1);
#pragma unroll 1
    for (long long q = __ldg(G.ent_ptr + r) + kSlotPF; q < e1; q += 8) {
      int cl[8];
      double w[8], xv[8];
#pragma unroll
      for (int m = 0; m < 8; ++m)
        if (q + m < e1) {
          cl[m] = __ldg(G.ent_col + q + m);
          w[m] = __ldg(G.ent_val + q + m);
        }
#pragma unroll
      for (int m = 0; m < 8; ++m)
        if (q + m < e1) xv[m] = __ldcg(u + (unsigned)cl[m]);
#pragma unroll
      for (int m = 0; m < 8; ++m)
        if (q + m < e1) acc = dadd(acc, dmul(w[m], xv[m]));
    }
  }
  if (p.diag == 0.0) atomicOr(&g_status, 1);
  const double om = G.omega;
  u[p.gid] = dadd(dmul(dsub(1.0, om), old), ddiv(dmul(om, dsub(p.fv, acc)), p.diag));
}

__global__ void surface_slots_kernel(SurfGSDesc G, long long *gid, int *cnt, double *diag,
                                     int *col, double *val, int *dyn, const int *gid_level,
                                     long long nlv) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long ns = G.nslots;
  if (e >= ns) return;
  const long long r = G.level_rows[e];
  const long long e0 = G.ent_ptr[r], c = G.ent_ptr[r + 1] - e0;
  const long long g = G.s.rows[r];
  const int lv = g < nlv ? gid_level[g] : -1;
  gid[e] = g;
  cnt[e] = (int)c;
  diag[e] = G.row_diag[r];
  unsigned bits = 0;
  for (int m = 0; m < kSlotPF; ++m) {
    const int cl = m < c ? G.ent_col[e0 + m] : 0;
    col[m * ns + e] = cl;
    val[m * ns + e] = m < c ? G.ent_val[e0 + m] : 0.0;
    if (m < c && cl < nlv && gid_level[cl] == lv - 1 && lv > 0) bits |= 1u << m;
  }
  dyn[e] = (int)bits;
}

#ifndef HHG_SURF_BAR
#define HHG_SURF_BAR 1           // grid barrier arrive: 0 fence + atomicAdd, 1 red.release
#endif
#ifndef HHG_SURF_GRID_RPB
#define HHG_SURF_GRID_RPB 8      // grid surface sweep: mean level rows per CTA
#endif
#ifndef HHG_SURF_CT
#define HHG_SURF_CT 256          // threads per CTA of the cluster surface sweep
#endif
#ifndef HHG_SURF_GRID_CT
#define HHG_SURF_GRID_CT 64      // threads per CTA of the grid surface sweep
#endif

// GRID = false: one thread-block cluster, hardware split barrier.
// GRID = true: a cooperative grid (wide schedules need more SMs' memory
// parallelism) with a split software barrier: arrive = block barrier, then
// one thread's fence + atomic add on *bar; wait = that thread's acquire
// spin until all blocks of this level arrived, then a block barrier.
// Either way the next row's static part is fetched between arrive and wait.
template <bool GRID>
__global__ void __launch_bounds__(GRID ? HHG_SURF_GRID_CT : HHG_SURF_CT)
gs_surface_slots_kernel(SurfGSDesc G, const long long *level_ptr, int nlev, unsigned *bar) {
  const long long nb = GRID ? (long long)gridDim.x : (long long)cluster_nctas();
  const long long rank = GRID ? (long long)blockIdx.x : (long long)cluster_ctarank();
  const long long tid = threadIdx.x * nb + rank;
  const long long nth = nb * blockDim.x;
  SlotRow pf;
  bool have = nlev > 0 && level_ptr[0] + tid < level_ptr[1];
  if (have) slot_prefetch(G, level_ptr[0] + tid, pf);
  for (int lv = 0; lv < nlev; ++lv) {
    const long long b = level_ptr[lv + 1];
    // one inlined copy of each step (register pressure)
    for (long long e = level_ptr[lv] + tid; e < b; e += nth) {
      if (!have) slot_prefetch(G, e, pf);
      have = false;
      slot_finish(G, e, pf);
    }
    if constexpr (GRID) {
      __syncthreads();
      if (threadIdx.x == 0) {
#if HHG_SURF_BAR == 1
        // release reduction (fence.acq_rel + red) instead of a full fence
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
#else
        __threadfence();
        atomicAdd(bar, 1u);
#endif
      }
    } else {
      asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    }
    have = false;
    if (lv + 1 < nlev) {
      const long long e = b + tid;
      have = e < level_ptr[lv + 2];
      if (have) slot_prefetch(G, e, pf);
    }
    if constexpr (GRID) {
      if (threadIdx.x == 0) {
        const unsigned target = (unsigned)((lv + 1) * nb);
        unsigned v;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
        } while (v < target);
      }
      __syncthreads();
    } else {
      asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    }
  }
}

}  // namespace hhg
