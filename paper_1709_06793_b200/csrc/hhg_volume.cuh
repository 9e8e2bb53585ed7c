// Volume (macro-element interior) stencil kernels.
//
// One CTA owns a tile of (i, j) lattice columns of one macro element —
// 32 consecutive i (one warp, coalesced rows) x W*B rows j — and marches
// the k planes upward.  Plane tiles (+1 halo) of the pair (v, k) are staged
// into a shared-memory ring with cp.async, NS-1 planes ahead; each thread
// keeps a three-plane register window of the values its B outputs need, so
// every staged value is read from shared memory once per plane.
//
// Source of v: global vector (interior rows are contiguous volume-block
// runs, HHG numbering) + compact ghost shell per element, or a full lattice
// array per element (per-element ABI).  k always comes from the lattice.
// All lattice-local offsets are 32-bit closed forms (no table lookups on the
// staging path); element bases are formed once per tile.
#pragma once
#include "hhg_common.cuh"

namespace hhg {

constexpr int VOL_COLS = 34;  // 32 lanes + halo

// ablation switch for tools/tune_volume.py (0 in every product build):
// 1 = no arithmetic (store v0), 2 = no staging after the prologue,
// 3 = no stores, 4 = staging ring only (no window loads, arithmetic, stores),
// 5 = k not staged (v only; timing of a k path off the LSU)
#ifndef HHG_VOL_EXPT
#define HHG_VOL_EXPT 0
#endif
// experiments (tools/tune_volume.py): L2 prefetch distance of the tile rows
// in planes (0 = off) and an L2 sector-promotion hint on the staging copies
#ifndef HHG_VOL_PF
#define HHG_VOL_PF 0
#endif
// ring layout of volume_kernel_mirror: 0 = interleaved (v, k) pairs (16-B
// slots, one LDS.128 per window point; the 8-byte staging writes of a warp
// are 16 B apart = 2x the shared wavefronts), 1 = separate v and k planes
// with a padded row stride of HHG_VOL_CS doubles (contiguous staging writes;
// two LDS.64 per window point)
#ifndef HHG_VOL_SOA
#define HHG_VOL_SOA 0
#endif
// FMA mode: split each row's accumulation into two chains
#ifndef HHG_SH_SMEM
#define HHG_SH_SMEM 0
#endif
#ifndef HHG_FMA_SPLIT
#define HHG_FMA_SPLIT 0
#endif
#ifndef HHG_VOL_CS
#define HHG_VOL_CS 40
#endif
#ifndef HHG_VOL_L2H
#define HHG_VOL_L2H ""
#endif

struct VolDesc {
  int n, ntets;
  long long L, nvol, S;
  long long n_nodes;           // length of the global vectors (SPLIT)
  const long long *vol_start;  // global layout: first volume id per tet
  const int *srow;             // shell row offsets (host checks; kernels use srow32)
  const double *ghost;         // [ntets*S]
  const double *kc;            // [ntets*L]
  const double *u;             // global vector (SPLIT) or [ntets*L] lattice
  const double *f;             // residual rhs, same layout as out
  double *out;                 // global vector or [ntets*nvol]
  const double *coef;          // per-tet coefficients (sh, fac, const)
  int coef_stride;
  double c0;                   // const variant, coef_stride 14: diagonal weight
  const double *w;             // stored stencils [ntets*nvol*15]
  const int4 *tiles;
  int ntiles;
  const int4 *mtiles;          // tiles of volume_kernel_mirror (8*NW columns)
  int nmtiles;
};

enum VolSrc { SRC_SPLIT = 0, SRC_LATTICE = 1 };

__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::);
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// mbarrier helpers (shared::cta)
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(bar)
               : "memory");
}
// arrive once all cp.async issued so far by this thread have landed
__device__ __forceinline__ void mbar_arrive_cp_async(unsigned bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// opaque copy: stops nvcc from re-folding the 64-bit element base
// (t * L) into every per-slot address computation
template <class P>
__device__ __forceinline__ P *opaque(P *p) {
  unsigned long long x = reinterpret_cast<unsigned long long>(p);
  asm volatile("mov.b64 %0, %0;" : "+l"(x));
  return reinterpret_cast<P *>(x);
}

// element-local offsets are < 2^31: index with zero-extended 32-bit ints
template <class P>
__device__ __forceinline__ P *at(P *base, int off) {
  return base + static_cast<unsigned>(off);
}

// per-tile element bases
struct TileBase {
  const double *k;   // kc of this element
  const double *v;   // SPLIT: u + vol_start (interior origin); LATTICE: u + t*L
  const double *g;   // ghost shell of this element
  double *o;         // output origin (volume rank 0 of this element)
  const double *f;   // residual rhs origin
};

// plane-constant parts of the lattice / inner-lattice / shell closed forms
struct PlaneConst {
  int kplane, rowk;   // lattice:  base(p, j) = kplane + j*rowk - j(j-1)/2
  int iplane, rowi;   // inner:    base'(p-1, j-1) = iplane + (j-1)*rowi - ...
  int gplane;         // shell:    offset of plane p's first shell point
};

__device__ __forceinline__ PlaneConst plane_const(int n, int p) {
  PlaneConst P;
  P.kplane = tetra32(n) - tetra32(n - p);
  P.rowk = n + 1 - p;
  P.iplane = (p >= 1) ? tetra32(n - 4) - tetra32(n - 3 - p) : 0;
  P.rowi = n - 2 - p;
  P.gplane = (p == 0) ? 0 : (n + 1) * (n + 2) / 2 + 3 * ((p - 1) * n - (p - 1) * p / 2);
  return P;
}

// One staging slot = a fixed (row r, column c) of the plane tile, owned by
// one thread for the whole k-march; per plane it issues at most two 8-byte
// cp.async (v, k).  Everything that does not depend on the plane is formed
// once per tile.
struct Slot {
  int i, j;           // lattice coordinates of the slot
  int jk;             // -j(j-1)/2 + i
  int ji;             // -(j-1)(j-2)/2 + i - 1
  int g0;             // plane-0 shell offset j(n+1) - j(j-1)/2 + i
  int gin;            // in-plane shell offset for p >= 1
  unsigned dst;       // shared address of the (v, k) pair
  bool live;
};

template <int SRC>
__device__ __forceinline__ void stage_slot(const TileBase &T, const Slot &S,
                                           const PlaneConst &P, int n, int p,
                                           unsigned slot_off) {
  if (!S.live || S.i + S.j + p > n) return;
  const int ko = P.kplane + S.j * P.rowk + S.jk;
  const double *ks = at(T.k, ko);
  const double *vs;
  if (SRC == SRC_LATTICE) {
    vs = at(T.v, ko);
  } else {
    const bool interior = p >= 1 && S.j >= 1 && S.i >= 1 && S.i + S.j + p <= n - 1;
    if (interior)
      vs = at(T.v, P.iplane + (S.j - 1) * P.rowi + S.ji);
    else
      vs = at(T.g, p == 0 ? S.g0 : P.gplane + S.gin - (S.j == 0 ? 0 : p));
  }
  const unsigned d = S.dst + slot_off;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(vs));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d + 8), "l"(ks));
}

// per-thread register window of one plane: column i (C), i+1 (R), i-1 (L)
template <int B>
struct Win {
  double2 C[B + 2];  // rows j0w-1 .. j0w+B
  double2 R[B + 1];  // rows j0w-1 .. j0w+B-1
  double2 L[B + 1];  // rows j0w   .. j0w+B
};

template <int B, int COLS = VOL_COLS>
__device__ __forceinline__ void load_win(Win<B> &w, const double2 *slot, int r0, int c) {
  const double2 *base = slot + (r0 - 1) * COLS + c;
#pragma unroll
  for (int m = 0; m < B + 2; ++m) w.C[m] = base[m * COLS];
#pragma unroll
  for (int m = 0; m < B + 1; ++m) w.R[m] = base[m * COLS + 1];
#pragma unroll
  for (int m = 0; m < B + 1; ++m) w.L[m] = base[(m + 1) * COLS - 1];
}

// same window from separate v / k planes (row stride CS doubles)
template <int B, int CS>
__device__ __forceinline__ void load_win_soa(Win<B> &w, const double *v, const double *k,
                                             int r0, int c) {
  const int o = (r0 - 1) * CS + c;
#pragma unroll
  for (int m = 0; m < B + 2; ++m) w.C[m] = make_double2(v[o + m * CS], k[o + m * CS]);
#pragma unroll
  for (int m = 0; m < B + 1; ++m) w.R[m] = make_double2(v[o + m * CS + 1], k[o + m * CS + 1]);
#pragma unroll
  for (int m = 0; m < B + 1; ++m)
    w.L[m] = make_double2(v[o + (m + 1) * CS - 1], k[o + (m + 1) * CS - 1]);
}

// gather the 14 neighbours of output row s from below / mid / above windows
// in stencil direction order (DIRS_3D)
template <int B>
__device__ __forceinline__ void neighbours(const Win<B> &lo, const Win<B> &mi,
                                           const Win<B> &hi, int s, double2 (&q)[14]) {
  q[0] = mi.R[s + 1];   // ( 1, 0, 0)
  q[1] = mi.C[s + 2];   // ( 0, 1, 0)
  q[2] = hi.C[s + 1];   // ( 0, 0, 1)
  q[3] = mi.R[s];       // ( 1,-1, 0)
  q[4] = lo.R[s + 1];   // ( 1, 0,-1)
  q[5] = lo.C[s + 2];   // ( 0, 1,-1)
  q[6] = hi.R[s];       // ( 1,-1, 1)
  q[7] = mi.L[s];       // (-1, 0, 0)
  q[8] = mi.C[s];       // ( 0,-1, 0)
  q[9] = lo.C[s + 1];   // ( 0, 0,-1)
  q[10] = mi.L[s + 1];  // (-1, 1, 0)
  q[11] = hi.L[s];      // (-1, 0, 1)
  q[12] = hi.C[s];      // ( 0,-1, 1)
  q[13] = lo.L[s + 1];  // (-1, 1,-1)
}

// neighbour d of output row s (same mapping as neighbours())
template <int B>
__device__ __forceinline__ double2 nbr(const Win<B> &lo, const Win<B> &mi, const Win<B> &hi,
                                       int d, int s) {
  switch (d) {
    case 0: return mi.R[s + 1];
    case 1: return mi.C[s + 2];
    case 2: return hi.C[s + 1];
    case 3: return mi.R[s];
    case 4: return lo.R[s + 1];
    case 5: return lo.C[s + 2];
    case 6: return hi.R[s];
    case 7: return mi.L[s];
    case 8: return mi.C[s];
    case 9: return lo.C[s + 1];
    case 10: return mi.L[s + 1];
    case 11: return hi.L[s];
    case 12: return hi.C[s];
    default: return lo.L[s + 1];
  }
}

// all B scaling rows of a thread, direction-outer / row-inner so the B
// accumulation chains interleave (warps issue in order: independent chains
// placed side by side hide the FP64 latency).  Per row the association is
// exactly the reference's: acc = ((t0 + t1) + t2) + ... with
// t_d = ((k0 + kq) * sh[d]) * (vq - v0).
template <int B, bool FAST>
__device__ __forceinline__ void scaling_rows(const Win<B> &lo, const Win<B> &mi,
                                             const Win<B> &hi, const double (&sh)[14],
                                             double (&out)[B]) {
  double v0[B], k0[B];
#pragma unroll
  for (int s = 0; s < B; ++s) {
    v0[s] = mi.C[s + 1].x;
    k0[s] = mi.C[s + 1].y;
  }
  if (!FAST) {
#pragma unroll
    for (int d = 0; d < 14; ++d)
#pragma unroll
      for (int s = 0; s < B; ++s) {
        const double2 q = nbr<B>(lo, mi, hi, d, s);
        const double term = dmul(dmul(dadd(k0[s], q.y), sh[d]), dsub(q.x, v0[s]));
        out[s] = (d == 0) ? term : dadd(out[s], term);
      }
  } else {
#pragma unroll
    for (int s = 0; s < B; ++s) out[s] = 0.0;
#pragma unroll
    for (int d = 0; d < 7; ++d)
#pragma unroll
      for (int s = 0; s < B; ++s) {
        const double2 a = nbr<B>(lo, mi, hi, d, s), b = nbr<B>(lo, mi, hi, d + 7, s);
        double m = (k0[s] + a.y) * (a.x - v0[s]);
        m = fma(k0[s] + b.y, b.x - v0[s], m);
        out[s] = fma(sh[d], m, out[s]);
      }
  }
}

// Mirror-exact variant.  When sh[d] == sh[d+7] bitwise (checked on the
// host), the reference term of an edge seen from its other end is the exact
// negation:  ((k_q + k_p) * sh) * (v_p - v_q) == -(((k_p + k_q) * sh) *
// (v_q - v_p))  in IEEE arithmetic, and  acc + (-t) == acc - t.  Edges whose
// both ends belong to the same thread are therefore evaluated once:
//   (0,-1, 0) of row s      = -(0,1,0) of row s-1      (same plane)
//   (0, 0,-1) of plane kk   = -(0,0,1) of plane kk-1   (previous step)
//   (0, 1,-1) of row s      = -(0,-1,1) of row s+1, plane kk-1
// 3B-2 of the 14B terms per step are reused; the result is bitwise the
// reference's.  pt2 / pt12 carry the (0,0,1) / (0,-1,1) terms to the next
// step; `first` seeds them from plane kk-1 at the start of a tile.
template <int B>
__device__ __forceinline__ double edge_term(double2 p, double2 q, double sh) {
  return dmul(dmul(dadd(p.y, q.y), sh), dsub(q.x, p.x));
}

template <int B>
__device__ __forceinline__ void scaling_rows_mirror(const Win<B> &lo, const Win<B> &mi,
                                                    const Win<B> &hi, const double (&sh)[14],
                                                    double (&pt2)[B], double (&pt12)[B],
                                                    bool first, double (&out)[B]) {
  if (first) {  // (0,0,1) and (0,-1,1) terms of the points of plane kk-1
#pragma unroll
    for (int s = 0; s < B; ++s) {
      pt2[s] = edge_term<B>(lo.C[s + 1], mi.C[s + 1], sh[2]);
      pt12[s] = edge_term<B>(lo.C[s + 1], mi.C[s], sh[12]);
    }
  }
  double t1[B], t2[B], t12[B];
#pragma unroll
  for (int d = 0; d < 14; ++d)
#pragma unroll
    for (int s = 0; s < B; ++s) {
      const double2 c = mi.C[s + 1];
      double t;
      bool neg = false;
      if (d == 8 && s >= 1) {
        t = t1[s - 1];
        neg = true;
      } else if (d == 9) {
        t = pt2[s];
        neg = true;
      } else if (d == 5 && s + 1 < B) {
        t = pt12[s + 1];
        neg = true;
      } else {
        t = edge_term<B>(c, nbr<B>(lo, mi, hi, d, s), sh[d]);
        if (d == 1) t1[s] = t;
        if (d == 2) t2[s] = t;
        if (d == 12) t12[s] = t;
      }
      if (d == 0) out[s] = t;
      else out[s] = neg ? dsub(out[s], t) : dadd(out[s], t);
    }
#pragma unroll
  for (int s = 0; s < B; ++s) {
    pt2[s] = t2[s];
    pt12[s] = t12[s];
  }
}

// Stencil dumps (kernels.dump_scaling_3d / dump_nodal_3d, kernels.py:293-376):
// per volume row (k, j, i order) the 15 weights (centre, s_0 .. s_13) of all
// macro elements, w[t][c][15] on the device - the stored-stencil baseline's
// input (Operator.store_stencils).  Scaling: s_d = (k0 + k_q) sh_d; nodal:
// the direction sums of the 40-add schedule; centre = -(s_0 + ... + s_13)
// accumulated from 0 in d order, as the reference.  Grid (planes, elements).
template <int VAR>
__global__ void dump_stencils_kernel(int n, long long L, long long nvol, const double *kc,
                                     const double *coef, int coef_stride, double *w) {
  const int t = blockIdx.y, k = 1 + blockIdx.x;
  if (k > n - 3) return;
  __shared__ double sfac[72];
  double sh[14];
  const double *cf = coef + (long long)t * coef_stride;
  if (VAR == 1) {
    for (int e = threadIdx.x; e < 72; e += blockDim.x) sfac[e] = cf[e];
    __syncthreads();
  } else {
#pragma unroll
    for (int d = 0; d < 14; ++d) sh[d] = cf[d];
  }
  const double *kt = kc + (long long)t * L;
  double *wt = w + (long long)t * nvol * 15;
  const int m4 = n - 4;
  const long long plane = tetra32(m4) - tetra32(m4 - (k - 1));   // first row of plane k
  int off = 0;
  for (int j = 1; j <= n - 2 - k; ++j) {
    const int len = n - 1 - j - k;
    for (int i0 = threadIdx.x; i0 < len; i0 += blockDim.x) {
      const int i = 1 + i0;
      double2 q[14];
      const double k0 = kt[lbase32(n, k, j) + i];
#pragma unroll
      for (int d = 0; d < 14; ++d)
        q[d].y = kt[lbase32(n, k + c_dirs_h(d, 2), j + c_dirs_h(d, 1)) + i + c_dirs_h(d, 0)];
      double *row = wt + (plane + off + i0) * 15;
      double tot = 0.0;
      if (VAR == 0) {
#pragma unroll
        for (int d = 0; d < 14; ++d) {
          const double sd = dmul(dadd(k0, q[d].y), sh[d]);
          row[1 + d] = sd;
          tot = dadd(tot, sd);
        }
      } else {
        double b[55];
#pragma unroll
        for (int d = 0; d < 14; ++d) q[d].x = 0.0;
        nodal_buffer(k0, q, b);
        dump_nodal_terms<0>(tot, row, b, sfac);
      }
      row[0] = -tot;
    }
    off += len;
  }
}

template <int VAR, bool FAST>
struct RowOp;

template <bool FAST>
struct RowOp<0, FAST> {  // scaling
  double sh[14];
  __device__ void init(const VolDesc &D, int t, double *) {
#pragma unroll
    for (int d = 0; d < 14; ++d) sh[d] = __ldg(D.coef + (long long)t * D.coef_stride + d);
  }
  __device__ __forceinline__ double operator()(double v0, double k0, const double2 (&q)[14],
                                               int) const {
    return FAST ? scaling_row_fast(v0, k0, q, sh) : scaling_row_exact(v0, k0, q, sh);
  }
};

template <bool FAST>
struct RowOp<1, FAST> {  // nodal integration, factors broadcast from smem
  const double *fac;
  __device__ void init(const VolDesc &D, int t, double *sfac) {
    for (int e = threadIdx.x; e < 72; e += blockDim.x)
      sfac[e] = D.coef[(long long)t * D.coef_stride + e];
    fac = sfac;
  }
  __device__ __forceinline__ double operator()(double v0, double k0, const double2 (&q)[14],
                                               int) const {
    return FAST ? nodal_row_fast(v0, k0, q, fac) : nodal_row_exact(v0, k0, q, fac);
  }
};

template <bool FAST>
struct RowOp<2, FAST> {  // constant coefficient: c0 v0 + sum s_d v_q
  double s[15];
  __device__ void init(const VolDesc &D, int t, double *) {
#pragma unroll
    for (int d = 0; d < 14; ++d) s[d] = __ldg(D.coef + (long long)t * D.coef_stride + d);
    // batched path: 15 weights per element; per-element ABI: 14 + c0 by value
    s[14] = D.coef_stride == 15 ? __ldg(D.coef + (long long)t * 15 + 14) : D.c0;
  }
  __device__ __forceinline__ double operator()(double v0, double, const double2 (&q)[14],
                                               int) const {
    double acc = dmul(s[14], v0);
#pragma unroll
    for (int d = 0; d < 14; ++d) acc = dadd(acc, dmul(s[d], q[d].x));
    return acc;
  }
};

template <bool FAST>
struct RowOp<3, FAST> {  // stored stencils w[c] = (diag, s_0..s_13)
  const double *w;
  __device__ void init(const VolDesc &D, int t, double *) {
    w = D.w + (long long)t * D.nvol * 15;
  }
  __device__ __forceinline__ double operator()(double v0, double, const double2 (&q)[14],
                                               int c) const {
    const double *wc = w + (long long)c * 15;
    double acc = dmul(__ldg(wc), v0);
#pragma unroll
    for (int d = 0; d < 14; ++d) acc = dadd(acc, dmul(__ldg(wc + 1 + d), q[d].x));
    return acc;
  }
};

template <int VAR, int SRC, bool RES, bool FAST, int B, int W, int NS, int MINB,
          bool MIRROR = false>
__global__ void __launch_bounds__(32 * W, MINB)
volume_kernel(VolDesc D) {
  constexpr int ROWS = W * B + 2;          // (W/4 warps) x (4 lane rows) x B
  constexpr int NT = 32 * W;
  constexpr int NSLOT = (ROWS * VOL_COLS + NT - 1) / NT;
  constexpr unsigned PLANE_BYTES = ROWS * VOL_COLS * sizeof(double2);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2 *ring = reinterpret_cast<double2 *>(smem_raw);
  double *sfac = reinterpret_cast<double *>(ring + NS * ROWS * VOL_COLS);
  const unsigned ring_s = static_cast<unsigned>(__cvta_generic_to_shared(ring));

  const int4 tile = D.tiles[blockIdx.x];
  const int t = tile.x, i0 = tile.y, j0 = tile.z, kmax = tile.w;
  const int n = D.n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  TileBase T;
  T.k = opaque(D.kc + (long long)t * D.L);
  if (SRC == SRC_SPLIT) {
    const long long vs = D.vol_start[t];
    T.v = opaque(D.u + vs);
    T.g = opaque(D.ghost + (long long)t * D.S);
    T.o = opaque(D.out + vs);
    T.f = RES ? opaque(D.f + vs) : nullptr;
  } else {
    T.v = opaque(D.u + (long long)t * D.L);
    T.g = nullptr;
    T.o = opaque(D.out + (long long)t * D.nvol);
    T.f = RES ? opaque(D.f + (long long)t * D.nvol) : nullptr;
  }

  RowOp<VAR, FAST> op;
  op.init(D, t, sfac);

  Slot slots[NSLOT];
#pragma unroll
  for (int m = 0; m < NSLOT; ++m) {
    const int e = threadIdx.x + m * NT;
    const int r = e / VOL_COLS, c = e - r * VOL_COLS;
    Slot &S = slots[m];
    S.live = e < ROWS * VOL_COLS;
    S.i = i0 - 1 + c;
    S.j = j0 - 1 + r;
    S.jk = -S.j * (S.j - 1) / 2 + S.i;
    S.ji = -(S.j - 1) * (S.j - 2) / 2 + S.i - 1;
    S.g0 = S.j * (n + 1) - S.j * (S.j - 1) / 2 + S.i;
    // p >= 1: row 0 -> i; row j -> (n - p + 1) + 2 (j - 1) + [i > 0]
    //         (the "- p" is applied per plane for j >= 1)
    S.gin = (S.j == 0) ? S.i : (n + 1) + 2 * (S.j - 1) + (S.i == 0 ? 0 : 1);
    S.dst = ring_s + (unsigned)e * sizeof(double2);
  }

  // ring of NS plane slots with a full / empty mbarrier pair each: a slot
  // is "full" when every thread's cp.async for it has landed (NT async
  // arrivals) and "empty" when every warp has copied its window out of it
  // (W arrivals).  Warps drift freely up to the prefetch distance PD
  // instead of meeting at a CTA barrier every plane.
  constexpr int PD = NS - 2;
  __shared__ __align__(8) unsigned long long bars[2 * NS];
  const unsigned full0 = static_cast<unsigned>(__cvta_generic_to_shared(&bars[0]));
  const unsigned empty0 = full0 + NS * 8;
  if (threadIdx.x == 0) {
    for (int b = 0; b < NS; ++b) {
      mbar_init(full0 + 8 * b, NT);
      mbar_init(empty0 + 8 * b, W);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  auto produce = [&](int p) {
    const int sl = p % NS;
    if (p >= NS) mbar_wait(empty0 + 8 * sl, ((p / NS) - 1) & 1);
    const PlaneConst P = plane_const(n, p);
    const unsigned off = (unsigned)sl * PLANE_BYTES;
    if (HHG_VOL_EXPT != 2 || p < PD) {
#pragma unroll
      for (int m = 0; m < NSLOT; ++m) stage_slot<SRC>(T, slots[m], P, n, p, off);
    }
    mbar_arrive_cp_async(full0 + 8 * sl);
  };

  // prologue: planes 0 .. PD-1 in flight
  for (int p = 0; p < PD && p <= kmax + 1; ++p) produce(p);

  // lane layout: a warp is an 8 (i) x 4 (row groups) patch, warps side by
  // side in i, each thread B consecutive rows of one column.  A warp's
  // lanes then span only 8 + 4B - 1 diagonal levels i + j, so few lanes sit
  // past the element's slanted face, and a warp whose lowest i + j is
  // already invalid skips the arithmetic altogether.
  static_assert(W % 4 == 0, "4 warps of 8 lanes cover the 32 tile columns");
  const int li = lane & 7, lj = lane >> 3;
  const int wi = warp & 3, wj = warp >> 2;   // warps: 4 along i, W/4 along j
  const int r0 = 1 + wj * 4 * B + lj * B;  // first tile row of this thread
  const int c = 1 + wi * 8 + li;
  const int i = i0 + wi * 8 + li;
  const int jw = j0 + wj * 4 * B + lj * B;
  const int warp_min_ij = i0 + wi * 8 + j0 + wj * 4 * B;
  const int m4 = n - 4;
  // per output row s: -(jj)(jj-1)/2 + i - 1 with jj = j - 1
  int oterm[B];
#pragma unroll
  for (int s = 0; s < B; ++s) {
    const int jj = jw + s - 1;
    oterm[s] = -jj * (jj - 1) / 2 + i - 1;
  }

  Win<B> X0, X1, X2;
  double pt2[B], pt12[B];   // mirror-reuse carry (MIRROR only)

  auto step = [&](int q, Win<B> &lo, Win<B> &mi, Win<B> &hi) {
    const int sl = q % NS;
    mbar_wait(full0 + 8 * sl, (q / NS) & 1);
    load_win<B>(hi, ring + sl * ROWS * VOL_COLS, r0, c);
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * sl);
    if (q >= 2 && warp_min_ij <= n - q) {   // some lane of the warp is valid
      const int kk = q - 1;
      const int lim = n - 1 - kk;  // valid outputs: i + j <= lim
      // volume rank of (i, j, kk): inner-lattice row (kk-1, j-1) + i - 1
      const int iplane = tetra32(m4) - tetra32(m4 - (kk - 1));
      const int rowi = m4 + 2 - kk;
      double vals[B];
      if constexpr (VAR == 0 && HHG_VOL_EXPT == 1) {
#pragma unroll
        for (int s = 0; s < B; ++s) vals[s] = mi.C[s + 1].x + lo.R[s + 1].y + hi.L[s].x;
      } else if constexpr (VAR == 0 && MIRROR && !FAST) {
        scaling_rows_mirror<B>(lo, mi, hi, op.sh, pt2, pt12, q == 2, vals);
      } else if constexpr (VAR == 0) {
        scaling_rows<B, FAST>(lo, mi, hi, op.sh, vals);
      } else {
#pragma unroll
        for (int s = 0; s < B; ++s) {
          double2 nb[14];
          neighbours<B>(lo, mi, hi, s, nb);
          const double2 ctr = mi.C[s + 1];
          const int cidx = iplane + (jw + s - 1) * rowi + oterm[s];
          const bool valid = i + jw + s <= lim;
          vals[s] = 0.0;
          if (VAR != 3 || valid) vals[s] = op(ctr.x, ctr.y, nb, cidx);  // stored reads w[cidx]
        }
      }
#pragma unroll
      for (int s = 0; s < B; ++s) {
        // invalid lanes computed on stale shared data; only the store is
        // predicated (no divergent branch around the arithmetic)
        if (i + jw + s <= lim) {
          const int cidx = iplane + (jw + s - 1) * rowi + oterm[s];
          double val = vals[s];
          if (RES) val = dsub(__ldg(at(T.f, cidx)), val);
          __stcs(at(T.o, cidx), val);
        }
      }
    }
    const int pf = q + PD;
    if (pf <= kmax + 1) produce(pf);
  };

  for (int q = 0; q <= kmax + 1; q += 3) {
    step(q, X1, X2, X0);
    if (q + 1 > kmax + 1) break;
    step(q + 1, X2, X0, X1);
    if (q + 2 > kmax + 1) break;
    step(q + 2, X0, X1, X2);
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// Default scaling kernel (bitwise reference order, mirror edge reuse) on a
// register diet: the terms of output plane kk+1 that involve plane kk-... are
// produced one step early, so only two planes of the window are live during
// the arithmetic; only sh[0..6] are held; staging slots keep one packed
// register.  Same tiles, ring, mbarriers and lane layout as volume_kernel.
// ---------------------------------------------------------------------------
template <int B>
struct MirrorCarry {
  double t2[B];    // (0,0,1) term of each row at plane kk   -> (0,0,-1) at kk+1
  double t12[B];   // (0,-1,1) term of each row at plane kk  -> (0,1,-1) at kk+1
  double t4[B];    // (1,0,-1) term of each row at plane kk+1 (neighbour on kk)
  double t13[B];   // (-1,1,-1) term of each row at plane kk+1
  double t5;       // (0,1,-1) term of the last row at plane kk+1
};

template <int B>
__device__ __forceinline__ void mirror_seed(const Win<B> &lo, const Win<B> &mi,
                                           const double (&sh)[7], MirrorCarry<B> &c) {
#pragma unroll
  for (int s = 0; s < B; ++s) {
    c.t2[s] = edge_term<B>(lo.C[s + 1], mi.C[s + 1], sh[2]);
    c.t12[s] = edge_term<B>(lo.C[s + 1], mi.C[s], sh[5]);      // sh[12] == sh[5]
    c.t4[s] = edge_term<B>(mi.C[s + 1], lo.R[s + 1], sh[4]);
    c.t13[s] = edge_term<B>(mi.C[s + 1], lo.L[s + 1], sh[6]);  // sh[13] == sh[6]
  }
  c.t5 = edge_term<B>(mi.C[B], lo.C[B + 1], sh[5]);
}

// rows of plane kk from windows mi (kk) and hi (kk+1) plus the carry;
// leaves the carry for plane kk+1.  Accumulation order d = 0..13 exactly.
template <int B>
__device__ __forceinline__ void mirror_step(const Win<B> &mi, const Win<B> &hi,
                                            const double (&sh)[7], MirrorCarry<B> &c,
                                            double (&out)[B]) {
  double t1[B], n2[B], n12[B];
#pragma unroll
  for (int s = 0; s < B; ++s) {
    const double2 p = mi.C[s + 1];
    double a = edge_term<B>(p, mi.R[s + 1], sh[0]);                 // d 0
    const double t1s = edge_term<B>(p, mi.C[s + 2], sh[1]);         // d 1
    t1[s] = t1s;
    a = dadd(a, t1s);
    n2[s] = edge_term<B>(p, hi.C[s + 1], sh[2]);                    // d 2
    a = dadd(a, n2[s]);
    a = dadd(a, edge_term<B>(p, mi.R[s], sh[3]));                   // d 3
    a = dadd(a, c.t4[s]);                                           // d 4
    a = (s + 1 < B) ? dsub(a, c.t12[s + 1]) : dadd(a, c.t5);        // d 5
    a = dadd(a, edge_term<B>(p, hi.R[s], sh[6]));                   // d 6
    a = dadd(a, edge_term<B>(p, mi.L[s], sh[0]));                   // d 7
    a = (s >= 1) ? dsub(a, t1[s - 1]) : dadd(a, edge_term<B>(p, mi.C[s], sh[1]));  // d 8
    a = dsub(a, c.t2[s]);                                           // d 9
    a = dadd(a, edge_term<B>(p, mi.L[s + 1], sh[3]));               // d 10
    a = dadd(a, edge_term<B>(p, hi.L[s], sh[4]));                   // d 11
    n12[s] = edge_term<B>(p, hi.C[s], sh[5]);                       // d 12
    a = dadd(a, n12[s]);
    a = dadd(a, c.t13[s]);                                          // d 13
    out[s] = a;
  }
#pragma unroll
  for (int s = 0; s < B; ++s) {
    c.t2[s] = n2[s];
    c.t12[s] = n12[s];
    c.t4[s] = edge_term<B>(hi.C[s + 1], mi.R[s + 1], sh[4]);
    c.t13[s] = edge_term<B>(hi.C[s + 1], mi.L[s + 1], sh[6]);
  }
  c.t5 = edge_term<B>(hi.C[B], mi.C[B + 1], sh[5]);
}

// --------------------------------------------------------------------------
// FMA edge-flux step.  P[s] carries the pre-summed down-plane terms
// (0,0,-1), (1,0,-1), (-1,1,-1), (0,1,-1) of row s of plane kk; the step
// finishes the rows of plane kk from windows mi (kk) and hi (kk+1) and
// leaves P for plane kk+1.  sh[d] == sh[d+7] (host-checked): the terms of
// an edge seen from its two ends are negatives of each other.
// --------------------------------------------------------------------------
__device__ __forceinline__ double fterm(double2 p, double2 q, double sh, double acc) {
  return fma((p.y + q.y) * sh, q.x - p.x, acc);
}
__device__ __forceinline__ double fflux(double2 p, double2 q, double sh) {
  return ((p.y + q.y) * sh) * (q.x - p.x);
}
// sh * [(k0+ka)(va-v0) + (k0+kb)(vb-v0)] + acc
__device__ __forceinline__ double fpair(double2 p, double2 a, double2 b, double sh, double acc) {
  double m = (p.y + a.y) * (a.x - p.x);
  m = fma(p.y + b.y, b.x - p.x, m);
  return fma(sh, m, acc);
}

template <int B>
__device__ __forceinline__ void fma_seed(const Win<B> &lo, const Win<B> &mi,
                                        const double (&sh)[7], double (&P)[B]) {
#pragma unroll
  for (int s = 0; s < B; ++s) {
    const double2 c = mi.C[s + 1];
    double a = fflux(c, lo.C[s + 1], sh[2]);                 // (0,0,-1)
    a = fterm(c, lo.R[s + 1], sh[4], a);                     // (1,0,-1)
    a = fterm(c, lo.L[s + 1], sh[6], a);                     // (-1,1,-1)
    a = fterm(c, lo.C[s + 2], sh[5], a);                     // (0,1,-1)
    P[s] = a;
  }
}

template <int B>
__device__ __forceinline__ void fma_step(const Win<B> &mi, const Win<B> &hi,
                                        const double (&sh)[7], double (&P)[B],
                                        double (&out)[B]) {
  double Pn[B], F1[B];
#pragma unroll
  for (int s = 0; s < B; ++s) {
    const double2 p = mi.C[s + 1];
#if HHG_FMA_SPLIT
    // two accumulation chains per row (in-plane / up-plane terms), summed
    // at the end: half the dependent-latency chain per row
    double acc = P[s];
    double up = fflux(p, hi.C[s + 1], sh[2]);                // (0,0,1), shared with kk+1
    Pn[s] = -up;
    acc = fpair(p, mi.R[s + 1], mi.L[s], sh[0], acc);        // (1,0,0) (-1,0,0)
    up = fterm(p, hi.R[s], sh[6], up);                       // (1,-1,1)
    acc = fpair(p, mi.R[s], mi.L[s + 1], sh[3], acc);        // (1,-1,0) (-1,1,0)
    up = fterm(p, hi.L[s], sh[4], up);                       // (-1,0,1)
    if (s + 1 < B) {                                         // (0,1,0), shared with s+1
      F1[s] = fflux(p, mi.C[s + 2], sh[1]);
      acc += F1[s];
    } else {
      acc = fterm(p, mi.C[s + 2], sh[1], acc);
    }
    if (s >= 1) {                                            // (0,-1,1), shared with
      const double F12 = fflux(p, hi.C[s], sh[5]);           // (0,1,-1) of row s-1 at kk+1
      up += F12;
      Pn[s - 1] -= F12;
    } else {
      up = fterm(p, hi.C[s], sh[5], up);
    }
    acc = (s >= 1) ? acc - F1[s - 1] : fterm(p, mi.C[s], sh[1], acc);   // (0,-1,0)
    out[s] = acc + up;
#else
    double acc = P[s];
    acc = fpair(p, mi.R[s + 1], mi.L[s], sh[0], acc);        // (1,0,0) (-1,0,0)
    acc = fpair(p, mi.R[s], mi.L[s + 1], sh[3], acc);        // (1,-1,0) (-1,1,0)
    if (s + 1 < B) {                                         // (0,1,0), shared with s+1
      F1[s] = fflux(p, mi.C[s + 2], sh[1]);
      acc += F1[s];
    } else {
      acc = fterm(p, mi.C[s + 2], sh[1], acc);
    }
    acc = (s >= 1) ? acc - F1[s - 1] : fterm(p, mi.C[s], sh[1], acc);   // (0,-1,0)
    const double F2 = fflux(p, hi.C[s + 1], sh[2]);          // (0,0,1), shared with kk+1
    acc += F2;
    Pn[s] = -F2;
    acc = fterm(p, hi.R[s], sh[6], acc);                     // (1,-1,1)
    acc = fterm(p, hi.L[s], sh[4], acc);                     // (-1,0,1)
    if (s >= 1) {                                            // (0,-1,1), shared with
      const double F12 = fflux(p, hi.C[s], sh[5]);           // (0,1,-1) of row s-1 at kk+1
      acc += F12;
      Pn[s - 1] -= F12;
    } else {
      acc = fterm(p, hi.C[s], sh[5], acc);
    }
    out[s] = acc;
#endif
  }
#pragma unroll
  for (int s = 0; s < B; ++s) {
    const double2 c = hi.C[s + 1];
    double a = fterm(c, mi.R[s + 1], sh[4], Pn[s]);          // (1,0,-1)
    a = fterm(c, mi.L[s + 1], sh[6], a);                     // (-1,1,-1)
    if (s == B - 1) a = fterm(c, mi.C[B + 1], sh[5], a);     // (0,1,-1), last row
    P[s] = a;
  }
}

// NW warps per CTA, each 8 columns x 4B rows (8x4 lanes, B rows per lane):
// a tile is 8*NW columns x 4B rows of one element, marching in k
// MODE 0: bitwise reference order (mirror_step); MODE 1: FMA edge-flux form
template <int SRC, bool RES, int B, int NS, int MINB, int NW, int MODE = 0>
__global__ void __launch_bounds__(32 * NW, MINB)
volume_kernel_mirror(VolDesc D) {
  constexpr int ROWS = 4 * B + 2;
  constexpr int COLS = 8 * NW + 2;
  constexpr int NT = 32 * NW;
  constexpr int NSLOT = (ROWS * COLS + NT - 1) / NT;
  constexpr bool SOA = HHG_VOL_SOA != 0;
  constexpr int CS = SOA ? HHG_VOL_CS : COLS;
  static_assert(CS >= COLS, "padded stride below the tile width");
  constexpr unsigned PLANE_BYTES = ROWS * CS * sizeof(double2);
  constexpr unsigned KOFF = SOA ? ROWS * CS * sizeof(double) : sizeof(double);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2 *ring = reinterpret_cast<double2 *>(smem_raw);
  const unsigned ring_s = static_cast<unsigned>(__cvta_generic_to_shared(ring));

  const int4 tile = D.mtiles[blockIdx.x];
  const int t = tile.x, i0 = tile.y, j0 = tile.z, kmax = tile.w;
  const int n = D.n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  TileBase T;
  T.k = opaque(D.kc + (long long)t * D.L);
  if (SRC == SRC_SPLIT) {
    const long long vs = D.vol_start[t];
    T.v = opaque(D.u + vs);
    T.g = opaque(D.ghost + (long long)t * D.S);
    T.o = opaque(D.out + vs);
    T.f = RES ? opaque(D.f + vs) : nullptr;
  } else {
    T.v = opaque(D.u + (long long)t * D.L);
    T.g = nullptr;
    T.o = opaque(D.out + (long long)t * D.nvol);
    T.f = RES ? opaque(D.f + (long long)t * D.nvol) : nullptr;
  }
#if HHG_SH_SMEM
  // the element's 7 stencil constants in shared memory: under register
  // pressure the compiler re-reads them (broadcast LDS) instead of spilling
  __shared__ double s_sh[7];
  if (threadIdx.x < 7) s_sh[threadIdx.x] = __ldg(D.coef + (long long)t * D.coef_stride + threadIdx.x);
  const double (&sh)[7] = s_sh;
#else
  double sh[7];
#pragma unroll
  for (int d = 0; d < 7; ++d) sh[d] = __ldg(D.coef + (long long)t * D.coef_stride + d);
#endif

  constexpr int PD = NS - 2;
  __shared__ __align__(8) unsigned long long bars[2 * NS];
  const unsigned full0 = static_cast<unsigned>(__cvta_generic_to_shared(&bars[0]));
  const unsigned empty0 = full0 + NS * 8;
  if (threadIdx.x == 0) {
    for (int b = 0; b < NS; ++b) {
      mbar_init(full0 + 8 * b, NT);
      mbar_init(empty0 + 8 * b, NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // Staging slots carry their offsets from plane to plane: with
  // T2(m) = (m+1)(m+2)/2 the lattice offset of (i, j, p+1) is that of
  // (i, j, p) plus T2(n-p) - j, the volume-block offset grows by
  // T2(n-3-p) - (j-1), the ghost offset by 3(n-p) - [j > 0]; only these
  // uniform deltas are formed per plane.
  struct IncSlot {
    int ko, vo, go;   // lattice, volume-block, ghost offsets at the next plane
    int pmax;         // last plane containing the point (i + j + p <= n)
    int ij;           // i | j << 16
    unsigned so;      // byte offset of the slot's v inside a plane of the ring
  };
  IncSlot sl_[NSLOT];
#pragma unroll
  for (int m = 0; m < NSLOT; ++m) {
    const int e = threadIdx.x + m * NT;
    const int r = e / COLS, cc = e - r * COLS;
    const int si = i0 - 1 + cc, sj = j0 - 1 + r;
    sl_[m].ij = si | (sj << 16);
    sl_[m].pmax = (e < ROWS * COLS) ? n - si - sj : -1;
    sl_[m].ko = sj * (n + 1) - sj * (sj - 1) / 2 + si;                   // plane 0
    sl_[m].vo = (sj - 1) * (n - 3) - (sj - 1) * (sj - 2) / 2 + si - 1;    // plane 1
    sl_[m].go = sl_[m].ko;                                               // plane 0
    sl_[m].so = SOA ? (unsigned)(r * CS + cc) * 8u : (unsigned)e * 16u;
  }
  const int t2n = (n + 1) * (n + 2) / 2;
  auto produce = [&](int p) {
    const int sl = p % NS;
    if (p >= NS) mbar_wait(empty0 + 8 * sl, ((p / NS) - 1) & 1);
    const unsigned off = ring_s + (unsigned)sl * PLANE_BYTES;
    const bool copy = HHG_VOL_EXPT != 2 || p < PD;   // EXPT 2: arithmetic only
#pragma unroll
    for (int m = 0; m < NSLOT; ++m) {
      IncSlot &S = sl_[m];
      const int si = S.ij & 0xffff, sj = S.ij >> 16;
      {
        // predicated copies instead of a divergent branch per slot
        const int live = copy && p <= S.pmax;
        const bool interior = p >= 1 && si >= 1 && sj >= 1 && p < S.pmax;
        const double *vs = interior ? at(T.v, S.vo) : at(T.g, S.go);
        const double *ks = at(T.k, S.ko);
        const unsigned d = off + S.so;
        if (live) {
          HHG_BOUND(S.ko, 0, D.L, "volume staging: lattice offset");
          if (interior) HHG_BOUND(S.vo, 0, D.nvol, "volume staging: volume-block offset");
          else if (SRC == SRC_SPLIT) HHG_BOUND(S.go, 0, D.S, "volume staging: ghost offset");
          HHG_BOUND(d + KOFF + 8 - ring_s, 0, NS * PLANE_BYTES + 1, "volume staging: ring byte");
        }
        if constexpr (HHG_VOL_EXPT == 5) {   // ablation: v staged, k not (timing only)
          asm volatile(
              "{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n"
              " @q cp.async.ca.shared.global [%0], [%1], 8;\n}\n" ::"r"(d),
              "l"(vs), "r"(live));
        } else {
          asm volatile(
              "{\n .reg .pred q;\n setp.ne.b32 q, %4, 0;\n"
              " @q cp.async.ca.shared.global" HHG_VOL_L2H " [%0], [%1], 8;\n"
              " @q cp.async.ca.shared.global" HHG_VOL_L2H " [%2], [%3], 8;\n}\n" ::"r"(d),
              "l"(vs), "r"(d + KOFF), "l"(ks), "r"(live));
        }
      }
      // advance to plane p + 1
      if (HHG_VOL_EXPT != 5) S.ko += (n - p + 1) * (n - p) / 2 + (n - p + 1) - sj;   // T2(n - p) - j
      if (p >= 1) S.vo += (n - 2 - p) * (n - 1 - p) / 2 - (sj - 1);  // T2(n-3-p) - (j-1)
      if (p == 0)
        S.go = t2n + (sj == 0 ? si : n + 2 * (sj - 1) + (si > 0 ? 1 : 0));
      else
        S.go += 3 * (n - p) - (sj > 0 ? 1 : 0);
    }
    mbar_arrive_cp_async(full0 + 8 * sl);
#if HHG_VOL_PF > 0
    // experiment: L2 prefetch of the tile's rows HHG_VOL_PF planes ahead
    // (4 lines per 34-point row segment, k and v rows: 112 threads)
    {
      const int q = p + HHG_VOL_PF;
      if (SRC == SRC_SPLIT && q <= kmax + 1 && threadIdx.x < 112) {
        const int seg = threadIdx.x >> 2, part = threadIdx.x & 3;
        const int sj = j0 - 1 + (seg >> 1);
        int si = i0 - 1 + part * 11;
        if (seg & 1) {
          si = min(si, n - 1 - sj - q);
          if (q >= 1 && sj >= 1 && si >= 1 && si >= i0 - 1)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(at(T.v, lbase32(n - 4, q - 1, sj - 1) + si - 1)));
        } else {
          si = min(si, n - sj - q);
          if (si >= i0 - 1 && sj >= 0)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(at(T.k, lbase32(n, q, sj) + si)));
        }
      }
    }
#endif
  };

  for (int p = 0; p < PD && p <= kmax + 1; ++p) produce(p);

  const int li = lane & 7, lj = lane >> 3;
  const int r0 = 1 + lj * B;
  const int c = 1 + warp * 8 + li;
  const int i = i0 + warp * 8 + li;
  const int jw = j0 + lj * B;
  const int warp_min_ij = i0 + warp * 8 + j0;
  const int m4 = n - 4;
  int oterm[B];
#pragma unroll
  for (int s = 0; s < B; ++s) {
    const int jj = jw + s - 1;
    oterm[s] = -jj * (jj - 1) / 2 + i - 1;
  }

  Win<B> X0, X1, X2;
  MirrorCarry<B> carry;   // MODE 0
  double P[B];            // MODE 1

  // fetch plane q into window w, release its slot, refill PD planes ahead
  auto fetch = [&](int q, Win<B> &w) {
    const int sl = q % NS;
    mbar_wait(full0 + 8 * sl, (q / NS) & 1);
    if constexpr (SOA) {
      const double *pv = reinterpret_cast<const double *>(smem_raw + sl * PLANE_BYTES);
      load_win_soa<B, CS>(w, pv, pv + ROWS * CS, r0, c);
    } else {
      load_win<B, COLS>(w, ring + sl * ROWS * COLS, r0, c);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * sl);
    if (q + PD <= kmax + 1) produce(q + PD);
  };
  auto emit = [&](int kk, const double (&vals)[B]) {
    const int lim = n - 1 - kk;
    const int iplane = tetra32(m4) - tetra32(m4 - (kk - 1));
    const int rowi = m4 + 2 - kk;
#pragma unroll
    for (int s = 0; s < B; ++s)
      if (i + jw + s <= lim) {
        const int cidx = iplane + (jw + s - 1) * rowi + oterm[s];
        HHG_BOUND(cidx, 0, D.nvol, "volume emit: output row");
        double val = vals[s];
        if (RES) val = dsub(__ldg(at(T.f, cidx)), val);
        if (HHG_VOL_EXPT == 3) {                 // ablation: no stores
          if (val == 12345.678) __stcs(at(T.o, cidx), val);
        } else {
          __stcs(at(T.o, cidx), val);
        }
      }
  };
  // output plane kk = q - 1 from mi (plane kk) and hi (plane kk + 1)
  auto step = [&](int q, Win<B> &mi, Win<B> &hi) {
    fetch(q, hi);
    if constexpr (HHG_VOL_EXPT == 4) return;       // ablation: staging ring only
    if (warp_min_ij <= n - q) {   // some lane of the warp is valid
      double vals[B];
      if constexpr (HHG_VOL_EXPT == 1) {          // data movement only
#pragma unroll
        for (int s = 0; s < B; ++s) vals[s] = hi.C[s + 1].x + mi.R[s].y + mi.L[s + 1].x;
      } else if constexpr (MODE == 0) {
        mirror_step<B>(mi, hi, sh, carry, vals);
      } else {
        fma_step<B>(mi, hi, sh, P, vals);
      }
      emit(q - 1, vals);
    }
  };

  if (kmax >= 1) {
    fetch(0, X0);
    fetch(1, X1);
    if (warp_min_ij <= n - 2) {
      if constexpr (MODE == 0) mirror_seed<B>(X0, X1, sh, carry);
      else fma_seed<B>(X0, X1, sh, P);
    }
    step(2, X1, X2);
    for (int q = 3; q <= kmax + 1; q += 3) {
      step(q, X2, X0);
      if (q + 1 > kmax + 1) break;
      step(q + 1, X0, X1);
      if (q + 2 > kmax + 1) break;
      step(q + 2, X1, X2);
    }
  }
  cp_async_wait<0>();
}


// ---------------------------------------------------------------------------
// Warp-specialised form of volume_kernel_mirror: one warpgroup of producers
// (128 threads, 4 staging slots each, setmaxnreg 40) fills the plane ring
// with cp.async and runs up to NS planes ahead, bounded only by the empty
// barriers; one warpgroup of consumers (setmaxnreg 216) does window loads,
// the mirror arithmetic and the stores, with no staging instructions in its
// stream.  Same tiles, ring, lane layout and arithmetic as the mirror kernel
// (bitwise equal).  2 CTAs x 8 warps per SM.
// ---------------------------------------------------------------------------
template <int SRC, bool RES, int B, int NS, int MODE = 0>
__global__ void __launch_bounds__(256, 2)
volume_kernel_ws(VolDesc D) {
  constexpr int NW = 4;                     // consumer warps (8 columns each)
  constexpr int ROWS = 4 * B + 2;
  constexpr int COLS = 8 * NW + 2;
  constexpr int NP = 128;                   // producer threads
  constexpr int NSLOT = (ROWS * COLS + NP - 1) / NP;
  constexpr unsigned PLANE_BYTES = ROWS * COLS * sizeof(double2);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2 *ring = reinterpret_cast<double2 *>(smem_raw);
  const unsigned ring_s = static_cast<unsigned>(__cvta_generic_to_shared(ring));

  const int4 tile = D.mtiles[blockIdx.x];
  const int t = tile.x, i0 = tile.y, j0 = tile.z, kmax = tile.w;
  const int n = D.n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  __shared__ __align__(8) unsigned long long bars[2 * NS];
  const unsigned full0 = static_cast<unsigned>(__cvta_generic_to_shared(&bars[0]));
  const unsigned empty0 = full0 + NS * 8;
  if (threadIdx.x == 0) {
    for (int b = 0; b < NS; ++b) {
      mbar_init(full0 + 8 * b, NP);
      mbar_init(empty0 + 8 * b, NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp >= NW) {
    // ---------------- producer warpgroup ----------------
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    const int ptid = threadIdx.x - NW * 32;
    const double *Tk = opaque(D.kc + (long long)t * D.L);
    const double *Tv, *Tg;
    if (SRC == SRC_SPLIT) {
      Tv = opaque(D.u + D.vol_start[t]);
      Tg = opaque(D.ghost + (long long)t * D.S);
    } else {
      Tv = opaque(D.u + (long long)t * D.L);
      Tg = nullptr;
    }
    int ko[NSLOT], vo[NSLOT], go[NSLOT], pmax[NSLOT], ij[NSLOT];
#pragma unroll
    for (int m = 0; m < NSLOT; ++m) {
      const int e = ptid + m * NP;
      const int r = e / COLS, cc = e - r * COLS;
      const int si = i0 - 1 + cc, sj = j0 - 1 + r;
      ij[m] = si | (sj << 16);
      pmax[m] = (e < ROWS * COLS) ? n - si - sj : -1;
      ko[m] = sj * (n + 1) - sj * (sj - 1) / 2 + si;                   // plane 0
      vo[m] = (sj - 1) * (n - 3) - (sj - 1) * (sj - 2) / 2 + si - 1;    // plane 1
      go[m] = ko[m];                                                   // plane 0
    }
    const int t2n = (n + 1) * (n + 2) / 2;
    for (int p = 0; p <= kmax + 1; ++p) {
      const int sl = p % NS;
      if (p >= NS) mbar_wait(empty0 + 8 * sl, ((p / NS) - 1) & 1);
      const unsigned off = ring_s + (unsigned)sl * PLANE_BYTES;
#pragma unroll
      for (int m = 0; m < NSLOT; ++m) {
        const int si = ij[m] & 0xffff, sj = ij[m] >> 16;
        const int live = p <= pmax[m];
        const bool interior = p >= 1 && si >= 1 && sj >= 1 && p < pmax[m];
        const double *vs = interior ? at(Tv, vo[m]) : at(Tg, go[m]);
        const double *ks = at(Tk, ko[m]);
        const unsigned d = off + (unsigned)(ptid + m * NP) * sizeof(double2);
        asm volatile(
            "{\n .reg .pred q;\n setp.ne.b32 q, %4, 0;\n"
            " @q cp.async.ca.shared.global [%0], [%1], 8;\n"
            " @q cp.async.ca.shared.global [%2], [%3], 8;\n}\n" ::"r"(d),
            "l"(vs), "r"(d + 8), "l"(ks), "r"(live));
        ko[m] += (n - p + 1) * (n - p) / 2 + (n - p + 1) - sj;
        if (p >= 1) vo[m] += (n - 2 - p) * (n - 1 - p) / 2 - (sj - 1);
        if (p == 0)
          go[m] = t2n + (sj == 0 ? si : n + 2 * (sj - 1) + (si > 0 ? 1 : 0));
        else
          go[m] += 3 * (n - p) - (sj > 0 ? 1 : 0);
      }
      mbar_arrive_cp_async(full0 + 8 * sl);
    }
    cp_async_wait<0>();
    return;
  }

  // ---------------- consumer warpgroup ----------------
  asm volatile("setmaxnreg.inc.sync.aligned.u32 216;\n" ::: "memory");
  double *To, *Tf;
  if (SRC == SRC_SPLIT) {
    const long long vs = D.vol_start[t];
    To = opaque(D.out + vs);
    Tf = RES ? opaque(const_cast<double *>(D.f) + vs) : nullptr;
  } else {
    To = opaque(D.out + (long long)t * D.nvol);
    Tf = RES ? opaque(const_cast<double *>(D.f) + (long long)t * D.nvol) : nullptr;
  }
  double sh[7];
#pragma unroll
  for (int d = 0; d < 7; ++d) sh[d] = __ldg(D.coef + (long long)t * D.coef_stride + d);

  const int li = lane & 7, lj = lane >> 3;
  const int r0 = 1 + lj * B;
  const int c = 1 + warp * 8 + li;
  const int i = i0 + warp * 8 + li;
  const int jw = j0 + lj * B;
  const int warp_min_ij = i0 + warp * 8 + j0;
  const int m4 = n - 4;
  int oterm[B];
#pragma unroll
  for (int s = 0; s < B; ++s) {
    const int jj = jw + s - 1;
    oterm[s] = -jj * (jj - 1) / 2 + i - 1;
  }

  Win<B> X0, X1, X2;
  MirrorCarry<B> carry;   // MODE 0
  double P[B];            // MODE 1
  auto fetch = [&](int q, Win<B> &w) {
    const int sl = q % NS;
    mbar_wait(full0 + 8 * sl, (q / NS) & 1);
    load_win<B, COLS>(w, ring + sl * ROWS * COLS, r0, c);
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * sl);
  };
  auto emit = [&](int kk, const double (&vals)[B]) {
    const int lim = n - 1 - kk;
    const int iplane = tetra32(m4) - tetra32(m4 - (kk - 1));
    const int rowi = m4 + 2 - kk;
#pragma unroll
    for (int s = 0; s < B; ++s)
      if (i + jw + s <= lim) {
        const int cidx = iplane + (jw + s - 1) * rowi + oterm[s];
        double val = vals[s];
        if (RES) val = dsub(__ldg(at(Tf, cidx)), val);
        __stcs(at(To, cidx), val);
      }
  };
  auto step = [&](int q, Win<B> &mi, Win<B> &hi) {
    fetch(q, hi);
    if (warp_min_ij <= n - q) {
      double vals[B];
      if constexpr (MODE == 0) mirror_step<B>(mi, hi, sh, carry, vals);
      else fma_step<B>(mi, hi, sh, P, vals);
      emit(q - 1, vals);
    }
  };
  if (kmax >= 1) {
    fetch(0, X0);
    fetch(1, X1);
    if (warp_min_ij <= n - 2) {
      if constexpr (MODE == 0) mirror_seed<B>(X0, X1, sh, carry);
      else fma_seed<B>(X0, X1, sh, P);
    }
    step(2, X1, X2);
    for (int q = 3; q <= kmax + 1; q += 3) {
      step(q, X2, X0);
      if (q + 1 > kmax + 1) break;
      step(q + 1, X0, X1);
      if (q + 2 > kmax + 1) break;
      step(q + 2, X1, X2);
    }
  }
}

}  // namespace hhg
