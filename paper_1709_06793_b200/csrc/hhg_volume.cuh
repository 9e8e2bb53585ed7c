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
#pragma once
#include "hhg_common.cuh"

namespace hhg {

constexpr int VOL_COLS = 34;  // 32 lanes + halo

struct VolDesc {
  int n, ntets;
  long long L, nvol, S;
  const long long *vol_start;  // global layout: first volume id per tet
  const int *srow;             // shell row offsets
  const double *ghost;         // [ntets*S]
  const double *kc;            // [ntets*L]
  const double *u;             // global vector (SPLIT) or [ntets*L] lattice
  const double *f;             // residual rhs, same layout as out
  double *out;                 // global vector or [ntets*nvol]
  const double *coef;          // per-tet coefficients (sh, fac, const)
  int coef_stride;
  const double *w;             // stored stencils [ntets*nvol*15]
  const int4 *tiles;
  int ntiles;
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

// issue the copies of lattice plane p of this tile into one ring slot
template <int SRC, int ROWS>
__device__ __forceinline__ void stage_plane(const VolDesc &D, int t, int i0,
                                            int j0, int p, double2 *slot,
                                            int warp, int lane, int nwarps) {
  const int n = D.n;
  for (int r = warp; r < ROWS; r += nwarps) {
    const int j = j0 - 1 + r;
    const int rowlen = n + 1 - p - j;  // points i = 0..rowlen-1
    if (rowlen <= 0) continue;
    const long long kb = (long long)t * D.L + lbase(n, p, j);
    const double *krow = D.kc + kb;
    const double *vrow_lat = nullptr, *vint = nullptr, *vgh = nullptr;
    bool inner = false;
    if (SRC == SRC_LATTICE) {
      vrow_lat = D.u + kb;
    } else {
      inner = (p >= 1) && (j >= 1) && (p + j <= n - 2);
      if (inner)
        vint = D.u + D.vol_start[t] + lbase(n - 4, p - 1, j - 1) - 1;
      vgh = D.ghost + (long long)t * D.S + D.srow[p * (n + 1) + j];
    }
#pragma unroll
    for (int c0 = 0; c0 < VOL_COLS; c0 += 32) {
      const int c = c0 + lane;
      const int i = i0 - 1 + c;
      if (c < VOL_COLS && i < rowlen) {
        double2 *dst = slot + r * VOL_COLS + c;
        const double *vs;
        if (SRC == SRC_LATTICE) {
          vs = vrow_lat + i;
        } else if (inner) {
          vs = (i >= 1 && i <= rowlen - 2) ? vint + i
                                           : vgh + (i == 0 ? 0 : 1);
        } else {
          vs = vgh + i;
        }
        cp_async8(&dst->x, vs);
        cp_async8(&dst->y, krow + i);
      }
    }
  }
}

// per-thread register window of one plane: column i (C), i+1 (R), i-1 (L)
template <int B>
struct Win {
  double2 C[B + 2];  // rows j0w-1 .. j0w+B
  double2 R[B + 1];  // rows j0w-1 .. j0w+B-1
  double2 L[B + 1];  // rows j0w   .. j0w+B
};

template <int B>
__device__ __forceinline__ void load_win(Win<B> &w, const double2 *slot,
                                         int r0, int c) {
#pragma unroll
  for (int m = 0; m < B + 2; ++m) w.C[m] = slot[(r0 - 1 + m) * VOL_COLS + c];
#pragma unroll
  for (int m = 0; m < B + 1; ++m) w.R[m] = slot[(r0 - 1 + m) * VOL_COLS + c + 1];
#pragma unroll
  for (int m = 0; m < B + 1; ++m) w.L[m] = slot[(r0 + m) * VOL_COLS + c - 1];
}

// gather the 14 neighbours of output row s from below / mid / above windows
// in stencil direction order (DIRS_3D)
template <int B>
__device__ __forceinline__ void neighbours(const Win<B> &lo, const Win<B> &mi,
                                           const Win<B> &hi, int s,
                                           double2 (&q)[14]) {
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

template <int VAR, bool FAST, int B>
struct RowOp;

template <bool FAST, int B>
struct RowOp<0, FAST, B> {  // scaling
  double sh[14];
  __device__ void init(const VolDesc &D, int t, double *) {
#pragma unroll
    for (int d = 0; d < 14; ++d) sh[d] = __ldg(D.coef + (long long)t * D.coef_stride + d);
  }
  __device__ __forceinline__ double operator()(double v0, double k0,
                                               const double2 (&q)[14],
                                               long long) const {
    return FAST ? scaling_row_fast(v0, k0, q, sh) : scaling_row_exact(v0, k0, q, sh);
  }
};

template <bool FAST, int B>
struct RowOp<1, FAST, B> {  // nodal integration, factors broadcast from smem
  const double *fac;
  __device__ void init(const VolDesc &D, int t, double *sfac) {
    for (int e = threadIdx.x; e < 72; e += blockDim.x)
      sfac[e] = D.coef[(long long)t * D.coef_stride + e];
    fac = sfac;
  }
  __device__ __forceinline__ double operator()(double v0, double k0,
                                               const double2 (&q)[14],
                                               long long) const {
    return nodal_row_exact(v0, k0, q, fac);
  }
};

template <bool FAST, int B>
struct RowOp<2, FAST, B> {  // constant coefficient: c0 v0 + sum s_d v_q
  double s[15];
  __device__ void init(const VolDesc &D, int t, double *) {
#pragma unroll
    for (int d = 0; d < 15; ++d) s[d] = __ldg(D.coef + (long long)t * D.coef_stride + d);
  }
  __device__ __forceinline__ double operator()(double v0, double, const double2 (&q)[14],
                                               long long) const {
    double acc = dmul(s[14], v0);
#pragma unroll
    for (int d = 0; d < 14; ++d) acc = dadd(acc, dmul(s[d], q[d].x));
    return acc;
  }
};

template <bool FAST, int B>
struct RowOp<3, FAST, B> {  // stored stencils w[c] = (diag, s_0..s_13)
  const double *w;
  __device__ void init(const VolDesc &D, int t, double *) {
    w = D.w + (long long)t * D.nvol * 15;
  }
  __device__ __forceinline__ double operator()(double v0, double, const double2 (&q)[14],
                                               long long c) const {
    const double *wc = w + c * 15;
    double acc = dmul(__ldg(wc), v0);
#pragma unroll
    for (int d = 0; d < 14; ++d) acc = dadd(acc, dmul(__ldg(wc + 1 + d), q[d].x));
    return acc;
  }
};

template <int VAR, int SRC, bool RES, bool FAST, int B, int W, int NS>
__global__ void __launch_bounds__(32 * W, 1)
volume_kernel(VolDesc D) {
  constexpr int ROWS = W * B + 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2 *ring = reinterpret_cast<double2 *>(smem_raw);
  double *sfac = reinterpret_cast<double *>(ring + NS * ROWS * VOL_COLS);

  const int4 tile = D.tiles[blockIdx.x];
  const int t = tile.x, i0 = tile.y, j0 = tile.z, kmax = tile.w;
  const int n = D.n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  RowOp<VAR, FAST, B> op;
  op.init(D, t, sfac);

  // prologue: planes 0 .. NS-2 in flight
#pragma unroll
  for (int p = 0; p < NS - 1; ++p) {
    if (p <= kmax + 1)
      stage_plane<SRC, ROWS>(D, t, i0, j0, p, ring + (p % NS) * ROWS * VOL_COLS,
                             warp, lane, W);
    cp_async_commit();
  }

  const int r0 = 1 + warp * B;  // first tile row of this thread
  const int c = 1 + lane;
  const int i = i0 + lane;
  const int jw = j0 + warp * B;
  const long long vbase = (SRC == SRC_SPLIT) ? D.vol_start[t] : (long long)t * D.nvol;

  Win<B> X0, X1, X2;

  auto step = [&](int q, Win<B> &lo, Win<B> &mi, Win<B> &hi) {
    // plane q has landed for this thread; make everyone's copies visible
    cp_async_wait<NS - 2>();
    __syncthreads();
    const int pf = q + NS - 1;
    if (pf <= kmax + 1)
      stage_plane<SRC, ROWS>(D, t, i0, j0, pf, ring + (pf % NS) * ROWS * VOL_COLS,
                             warp, lane, W);
    cp_async_commit();
    load_win<B>(hi, ring + (q % NS) * ROWS * VOL_COLS, r0, c);
    if (q >= 2) {
      const int kk = q - 1;
      const int lim = n - 1 - kk;  // valid outputs: i + j <= lim
#pragma unroll
      for (int s = 0; s < B; ++s) {
        const int j = jw + s;
        if (i + j <= lim) {
          double2 nb[14];
          neighbours<B>(lo, mi, hi, s, nb);
          const long long cidx = lbase(n - 4, kk - 1, j - 1) + (i - 1);
          const double2 ctr = mi.C[s + 1];
          double val = op(ctr.x, ctr.y, nb, cidx);
          const long long g = vbase + cidx;
          if (RES) val = dsub(__ldg(D.f + g), val);
          D.out[g] = val;
        }
      }
    }
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

}  // namespace hhg
