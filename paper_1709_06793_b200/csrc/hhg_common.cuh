// Shared device helpers: lattice arithmetic, patch tables, fp64 ops.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

// Bounds-checked debug build (-DHHG_DEBUG_BOUNDS=1; tools/bounds_check.sh):
// compute-sanitizer is closed on this GPU pool, so the hot kernels assert
// every global index they form against the extent of its array and trap
// with the offending value.  Compiled out (no code) in product builds.
#ifndef HHG_DEBUG_BOUNDS
#define HHG_DEBUG_BOUNDS 0
#endif
#if HHG_DEBUG_BOUNDS
#include <cstdio>
#define HHG_BOUND(idx, lo, hi, what)                                                   \
  do {                                                                                 \
    const long long _i = (long long)(idx), _lo = (long long)(lo), _hi = (long long)(hi); \
    if (_i < _lo || _i >= _hi) {                                                       \
      printf("hhg bounds: %s = %lld outside [%lld, %lld) (block %d, thread %d)\n", what, \
             _i, _lo, _hi, (int)blockIdx.x, (int)threadIdx.x);                         \
      __trap();                                                                        \
    }                                                                                  \
  } while (0)
#else
#define HHG_BOUND(idx, lo, hi, what) ((void)0)
#endif

namespace hhg {

// ---------------------------------------------------------------------------
// lattice arithmetic (mesh.py: SimplexLattice, closed form of base[k, j])
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ long long tetra(long long m) {
  // points of a size-m tetrahedral lattice, 0 for m < 0
  return m < 0 ? 0 : (m + 1) * (m + 2) * (m + 3) / 6;
}
__host__ __device__ __forceinline__ long long lbase(int n, int k, int j) {
  return tetra(n) - tetra(n - k) + (long long)j * (n + 1 - k) -
         (long long)j * (j - 1) / 2;
}

// 32-bit forms for lattice-local offsets (exact for n <= 1000)
__host__ __device__ __forceinline__ int tetra32(int m) {
  return m < 0 ? 0 : (m + 1) * (m + 2) * (m + 3) / 6;
}
__host__ __device__ __forceinline__ int lbase32(int n, int k, int j) {
  return tetra32(n) - tetra32(n - k) + j * (n + 1 - k) - j * (j - 1) / 2;
}
// offset of lattice row (k, j) inside the compact ghost shell of an element:
// plane 0 is stored whole; plane k >= 1 stores its row j = 0, the two end
// points of rows 1 .. n-k-1 and its last row (3 (n-k) points, 1 for k = n)
__host__ __device__ __forceinline__ int srow32(int n, int k, int j) {
  if (k == 0) return j * (n + 1) - j * (j - 1) / 2;
  const int plane = (n + 1) * (n + 2) / 2 + 3 * ((k - 1) * n - (k - 1) * k / 2);
  return plane + (j == 0 ? 0 : (n - k + 1) + 2 * (j - 1));
}
__host__ __device__ __forceinline__ long long shell_size(int n) {
  return (long long)(n + 1) * (n + 2) / 2 + 3LL * n * (n - 1) / 2 + 1;
}

// the 14 stencil directions (di, dj, dk), mesh.py:44-48
__constant__ int8_t c_dirs[14][3] = {
    {1, 0, 0},  {0, 1, 0},  {0, 0, 1},  {1, -1, 0},  {1, 0, -1},
    {0, 1, -1}, {1, -1, 1}, {-1, 0, 0}, {0, -1, 0},  {0, 0, -1},
    {-1, 1, 0}, {-1, 0, 1}, {0, -1, 1}, {-1, 1, -1}};

// the same directions as compile-time constants (for unrolled loops)
__host__ __device__ constexpr int c_dirs_h(int d, int c) {
  constexpr int a[14][3] = {{1, 0, 0},  {0, 1, 0},  {0, 0, 1},  {1, -1, 0},  {1, 0, -1},
                            {0, 1, -1}, {1, -1, 1}, {-1, 0, 0}, {0, -1, 0},  {0, 0, -1},
                            {-1, 1, 0}, {-1, 0, 1}, {0, -1, 1}, {-1, 1, -1}};
  return a[d][c];
}

// patch tables (reference_stencils.py:48-75 and Environment.term_*):
// term t of direction d (t in [TPTR[d], TPTR[d+1])) reads element sum slot
// 31 + TELEM[t].
#define HHG_TPTR {0, 6, 10, 16, 22, 26, 32, 36, 42, 46, 52, 58, 62, 68, 72}
#define HHG_TELEM                                                            \
  {18, 19, 20, 21, 22, 23, 10, 11, 18, 20, 6,  7,  10, 14, 18, 19, 12, 13,   \
   15, 17, 22, 23, 16, 17, 21, 23, 8,  9,  11, 16, 20, 21, 14, 15, 19, 22,   \
   0,  1,  2,  3,  4,  5,  4,  5,  12, 13, 3,  5,  9,  13, 16, 17, 0,  2,    \
   6,  8,  10, 11, 0,  1,  6,  7,  1,  4,  7,  12, 14, 15, 2,  3,  8,  9}
#define HHG_CSE                                                              \
  {{15, 0, 1},   {16, 0, 10},  {17, 0, 11},  {18, 0, 13},  {19, 8, 12},      \
   {20, 8, 14},  {21, 8, 9},   {22, 3, 12},  {23, 6, 14},  {24, 2, 3},       \
   {25, 2, 6},   {26, 4, 9},   {27, 3, 7},   {28, 4, 7},   {29, 5, 6},       \
   {30, 4, 5},   {31, 17, 19}, {32, 18, 19}, {33, 17, 20}, {34, 16, 20},     \
   {35, 18, 21}, {36, 16, 21}, {37, 17, 22}, {38, 18, 22}, {39, 17, 23},     \
   {40, 16, 23}, {41, 17, 24}, {42, 17, 25}, {43, 18, 26}, {44, 16, 26},     \
   {45, 18, 27}, {46, 18, 28}, {47, 16, 29}, {48, 16, 30}, {49, 15, 24},     \
   {50, 15, 27}, {51, 15, 25}, {52, 15, 29}, {53, 15, 28}, {54, 15, 30}}

// compile-time accessors (indices are constants after full unrolling)
__host__ __device__ constexpr int pt_tptr(int d) {
  constexpr int a[15] = HHG_TPTR;
  return a[d];
}
__host__ __device__ constexpr int pt_telem(int t) {
  constexpr int a[72] = HHG_TELEM;
  return a[t];
}
__host__ __device__ constexpr int pt_cse(int r, int c) {
  constexpr int a[40][3] = HHG_CSE;
  return a[r][c];
}

// bitmask of stencil directions that stay inside the closed macro element
// for each of the 14 boundary classes (reference_stencils.class_element_masks)
__constant__ uint16_t c_cls_dirmask[14] = {16312, 4991, 11959, 7631, 4920,
                                           11952, 567,  7560,  4431, 3207,
                                           560,   4360, 3200,  7};

// ---------------------------------------------------------------------------
// fp64 arithmetic: the bitwise path uses explicit round-to-nearest ops so
// nvcc cannot contract mul+add into FMA (the reference runs numba without
// fastmath, kernels.py:10)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// scaled-stencil row, exact reference order:
//   acc = sum_d ((k0 + kq) * sh[d]) * (vq - v0), d = 0..13 left to right
__device__ __forceinline__ double scaling_row_exact(double v0, double k0,
                                                    const double2 (&q)[14],
                                                    const double (&sh)[14]) {
  double acc = dmul(dmul(dadd(k0, q[0].y), sh[0]), dsub(q[0].x, v0));
#pragma unroll
  for (int d = 1; d < 14; ++d)
    acc = dadd(acc, dmul(dmul(dadd(k0, q[d].y), sh[d]), dsub(q[d].x, v0)));
  return acc;
}

// reassociated form: mirror pairs (d, d+7) share a folded weight, FMAs
// (sh2[d] holds the pair weight, host checked |sh[d]-sh[d+7]| tiny)
__device__ __forceinline__ double scaling_row_fast(double v0, double k0,
                                                   const double2 (&q)[14],
                                                   const double (&sh)[14]) {
  double acc = 0.0;
#pragma unroll
  for (int d = 0; d < 7; ++d) {
    double m = (k0 + q[d].y) * (q[d].x - v0);
    m = fma(k0 + q[d + 7].y, q[d + 7].x - v0, m);
    acc = fma(sh[d], m, acc);
  }
  return acc;
}

// Patch tables as static constexpr members: every index below is a template
// argument, so the 55-slot element-sum buffer stays in registers (indexing a
// constexpr array with a loop variable made nvcc materialise the tables in
// local memory).
struct Patch {
  static constexpr int tptr[15] = HHG_TPTR;
  static constexpr int telem[72] = HHG_TELEM;
  static constexpr int cse[40][3] = HHG_CSE;
};

template <int R>
__device__ __forceinline__ void cse_steps(double (&b)[55]) {
  if constexpr (R < 40) {
    constexpr int dst = Patch::cse[R][0], a = Patch::cse[R][1], c = Patch::cse[R][2];
    b[dst] = dadd(b[a], b[c]);
    cse_steps<R + 1>(b);
  }
}

// s_d = sum over the terms t of direction d of buf[31 + telem[t]] * fac[t],
// left to right (kernels.py:172-177)
template <int T, int END, class FAC>
__device__ __forceinline__ double dir_terms(double s, const double (&b)[55], const FAC &fac) {
  if constexpr (T < END) {
    constexpr int slot = 31 + Patch::telem[T];
    return dir_terms<T + 1, END>(dadd(s, dmul(b[slot], fac[T])), b, fac);
  } else {
    return s;
  }
}

template <int D, class FAC>
__device__ __forceinline__ double dir_sum(const double (&b)[55], const FAC &fac) {
  constexpr int t0 = Patch::tptr[D], t1 = Patch::tptr[D + 1];
  constexpr int slot = 31 + Patch::telem[t0];
  return dir_terms<t0 + 1, t1>(dmul(b[slot], fac[t0]), b, fac);
}

// acc = s_0 (v_0 - v0) + s_1 (v_1 - v0) + ... in direction order
template <int D, class FAC>
__device__ __forceinline__ double nodal_acc(double acc, double v0, const double2 (&q)[14],
                                            const double (&b)[55], const FAC &fac) {
  if constexpr (D < 14) {
    const double term = dmul(dir_sum<D>(b, fac), dsub(q[D].x, v0));
    return nodal_acc<D + 1>(D == 0 ? term : dadd(acc, term), v0, q, b, fac);
  } else {
    return acc;
  }
}

__device__ __forceinline__ void nodal_buffer(double k0, const double2 (&q)[14],
                                             double (&b)[55]) {
  b[0] = k0;
#pragma unroll
  for (int d = 0; d < 14; ++d) b[1 + d] = q[d].y;
  cse_steps<0>(b);
}

// nodal-integration row, exact reference order (kernels.py:139-189)
template <class FAC>
__device__ __forceinline__ double nodal_row_exact(double v0, double k0,
                                                  const double2 (&q)[14],
                                                  const FAC &fac) {
  double b[55];
  nodal_buffer(k0, q, b);
  return nodal_acc<0>(0.0, v0, q, b, fac);
}

// FMA form of the nodal row (Operator(fast=True)): the same 40-add element
// sums, then s_d = fma(b, fac, s) over the terms and acc = fma(s_d,
// v_q - v0, acc): 140 instead of 211 FP64 operations per row, within 1e-12
// (max-norm relative) of the reference order
template <int T, int END, class FAC>
__device__ __forceinline__ double dir_terms_fma(double s, const double (&b)[55],
                                                const FAC &fac) {
  if constexpr (T < END) {
    constexpr int slot = 31 + Patch::telem[T];
    return dir_terms_fma<T + 1, END>(fma(b[slot], fac[T], s), b, fac);
  } else {
    return s;
  }
}

template <int D, class FAC>
__device__ __forceinline__ double nodal_acc_fma(double acc, double v0, const double2 (&q)[14],
                                                const double (&b)[55], const FAC &fac) {
  if constexpr (D < 14) {
    constexpr int t0 = Patch::tptr[D], t1 = Patch::tptr[D + 1];
    constexpr int slot = 31 + Patch::telem[t0];
    const double sd = dir_terms_fma<t0 + 1, t1>(b[slot] * fac[t0], b, fac);
    return nodal_acc_fma<D + 1>(fma(sd, q[D].x - v0, acc), v0, q, b, fac);
  } else {
    return acc;
  }
}

template <class FAC>
__device__ __forceinline__ double nodal_row_fast(double v0, double k0, const double2 (&q)[14],
                                                 const FAC &fac) {
  double b[55];
  nodal_buffer(k0, q, b);
  return nodal_acc_fma<0>(0.0, v0, q, b, fac);
}

// dump form (kernels.py:330-376): row[1 + d] = s_d, tot += s_d
template <int D, class FAC>
__device__ __forceinline__ void dump_nodal_terms(double &tot, double *row, const double (&b)[55],
                                                 const FAC &fac) {
  if constexpr (D < 14) {
    const double s = dir_sum<D>(b, fac);
    row[1 + D] = s;
    tot = dadd(tot, s);
    dump_nodal_terms<D + 1>(tot, row, b, fac);
  }
}

// GS form (kernels.py:553-600): acc += s_d u_d, diag -= s_d
template <int D, class FAC>
__device__ __forceinline__ void nodal_gs_terms(double &acc, double &diag,
                                               const double2 (&q)[14],
                                               const double (&b)[55], const FAC &fac,
                                               unsigned mask = 0x3fffu) {
  if constexpr (D < 14) {
    if (mask >> D & 1) {
      const double s = dir_sum<D>(b, fac);
      acc = dadd(acc, dmul(s, q[D].x));
      diag = dsub(diag, s);
    }
    nodal_gs_terms<D + 1>(acc, diag, q, b, fac, mask);
  }
}

}  // namespace hhg
