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

struct VolDesc {
  int n, ntets;
  long long L, nvol, S;
  const long long *vol_start;  // global layout: first volume id per tet
  const int *srow;             // shell row offsets (host checks; kernels use srow32)
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

template <int B>
__device__ __forceinline__ void load_win(Win<B> &w, const double2 *slot, int r0, int c) {
  const double2 *base = slot + (r0 - 1) * VOL_COLS + c;
#pragma unroll
  for (int m = 0; m < B + 2; ++m) w.C[m] = base[m * VOL_COLS];
#pragma unroll
  for (int m = 0; m < B + 1; ++m) w.R[m] = base[m * VOL_COLS + 1];
#pragma unroll
  for (int m = 0; m < B + 1; ++m) w.L[m] = base[(m + 1) * VOL_COLS - 1];
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
    return nodal_row_exact(v0, k0, q, fac);
  }
};

template <bool FAST>
struct RowOp<2, FAST> {  // constant coefficient: c0 v0 + sum s_d v_q
  double s[15];
  __device__ void init(const VolDesc &D, int t, double *) {
#pragma unroll
    for (int d = 0; d < 15; ++d) s[d] = __ldg(D.coef + (long long)t * D.coef_stride + d);
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

template <int VAR, int SRC, bool RES, bool FAST, int B, int W, int NS>
__global__ void __launch_bounds__(32 * W, 1)
volume_kernel(VolDesc D) {
  constexpr int ROWS = W * B + 2;
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

  auto stage = [&](int p) {
    const PlaneConst P = plane_const(n, p);
    const unsigned off = (unsigned)(p % NS) * PLANE_BYTES;
#pragma unroll
    for (int m = 0; m < NSLOT; ++m) stage_slot<SRC>(T, slots[m], P, n, p, off);
  };

  // prologue: planes 0 .. NS-2 in flight
#pragma unroll
  for (int p = 0; p < NS - 1; ++p) {
    if (p <= kmax + 1) stage(p);
    cp_async_commit();
  }

  const int r0 = 1 + warp * B;  // first tile row of this thread
  const int c = 1 + lane;
  const int i = i0 + lane;
  const int jw = j0 + warp * B;
  const int m4 = n - 4;
  // per output row s: -(jj)(jj-1)/2 + i - 1 with jj = j - 1
  int oterm[B];
#pragma unroll
  for (int s = 0; s < B; ++s) {
    const int jj = jw + s - 1;
    oterm[s] = -jj * (jj - 1) / 2 + i - 1;
  }

  Win<B> X0, X1, X2;

  auto step = [&](int q, Win<B> &lo, Win<B> &mi, Win<B> &hi) {
    // plane q has landed for this thread; make everyone's copies visible
    cp_async_wait<NS - 2>();
    __syncthreads();
    const int pf = q + NS - 1;
    if (pf <= kmax + 1) stage(pf);
    cp_async_commit();
    load_win<B>(hi, ring + (q % NS) * ROWS * VOL_COLS, r0, c);
    if (q >= 2) {
      const int kk = q - 1;
      const int lim = n - 1 - kk;  // valid outputs: i + j <= lim
      // volume rank of (i, j, kk): inner-lattice row (kk-1, j-1) + i - 1
      const int iplane = tetra32(m4) - tetra32(m4 - (kk - 1));
      const int rowi = m4 + 2 - kk;
#pragma unroll
      for (int s = 0; s < B; ++s) {
        double2 nb[14];
        neighbours<B>(lo, mi, hi, s, nb);
        const double2 ctr = mi.C[s + 1];
        const int cidx = iplane + (jw + s - 1) * rowi + oterm[s];
        // invalid lanes compute on stale shared data; only the store is
        // predicated (no divergent branch around the arithmetic)
        const bool valid = i + jw + s <= lim;
        double val = 0.0;
        if (VAR != 3 || valid) val = op(ctr.x, ctr.y, nb, cidx);  // stored reads w[cidx]
        if (valid) {
          if (RES) val = dsub(__ldg(at(T.f, cidx)), val);
          *at(T.o, cidx) = val;
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
