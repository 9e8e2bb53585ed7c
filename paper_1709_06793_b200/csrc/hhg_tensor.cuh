// Tensor-coefficient operators: M = 6 scalar component fields k_m, each
// riding on its own first-order operator (coefficients.py:120-200).
//
// Scaled rows (kernels.py:192-232, gs :603-640):
//   s_d = sum_m (k_m[p] + k_m[q_d]) * shm[m][d]          (m = 0..M-1)
//   row = sum_d s_d (v[q_d] - v[p])
// Nodal rows (kernels.py:235-286, gs :643-702): per component the 40-add
// element-sum schedule, then
//   s_d = sum_{t in terms(d)} sum_m esum_m[telem[t]] * fac[m][t]
// Both in the reference association order (bitwise, up to the sign of an
// exact zero: the reference seeds its sums with 0.0).
//
// These rows are FP64-bound (scaled ~300, nodal ~1150 ops per row against
// 64 B of streamed data), so the kernel is a plain thread-per-row layout:
// a warp owns 32 consecutive i of one lattice row, neighbour values come
// through L1 (the 15 points of a row's stencil sit on 3 planes x 3 rows that
// neighbouring warps of the CTA also read).  The nodal element sums of all
// components live in shared memory, one column per thread.
#pragma once
#include "hhg_common.cuh"
#include "hhg_smooth.cuh"
#include "hhg_surface.cuh"

namespace hhg {

constexpr int kTenM = 6;   // 3-D splitting (TENSOR_DIRS_3D)

struct TenDesc {
  int n, ntets;
  long long L, S, nvol;
  const long long *vol_start;  // SPLIT: first volume id per element
  const double *ghost;         // SPLIT: compact shells [ntets*S]
  const double *km;            // [ntets][M][L]
  const double *u;             // SPLIT: global vector; LATTICE: [ntets*L]
  const double *f;             // residual / GS rhs (global or [ntets*nvol])
  double *out;                 // apply: global or [ntets*nvol]
  const double *coef;          // shm [ntets][M][14] or fac [ntets][M][72]
  int lattice;
  double omega;
  const int *hp_ptr, *hp_code; // GS hyperplanes (hhg_smooth.cuh)
};

template <bool NODAL>
constexpr int ten_rows() { return NODAL ? 2 : 4; }   // lattice rows per CTA
template <bool NODAL>
constexpr int ten_threads() { return 32 * ten_rows<NODAL>(); }
template <bool NODAL>
constexpr int ten_ncoef() { return NODAL ? 72 : 14; }

// dynamic shared memory: coefficients of the element, then (nodal) the
// element sums [M*24][threads]
template <bool NODAL>
constexpr size_t ten_smem(int threads) {
  return sizeof(double) * (kTenM * ten_ncoef<NODAL>() +
                           (NODAL ? (size_t)kTenM * 24 * threads : 0));
}

// s_d of the nodal tensor row: terms t of direction d outer, components m
// inner (kernels.py:275-281); every index is a template constant
template <int T, int END>
__device__ __forceinline__ double ten_dir_terms(double s, const double *es, int nth, int tid,
                                                const double *sc) {
  if constexpr (T < END) {
    constexpr int e = Patch::telem[T];
#pragma unroll
    for (int m = 0; m < kTenM; ++m) s = dadd(s, dmul(es[(m * 24 + e) * nth + tid], sc[m * 72 + T]));
    return ten_dir_terms<T + 1, END>(s, es, nth, tid, sc);
  } else {
    return s;
  }
}

template <int D>
__device__ __forceinline__ double ten_dir_sum(const double *es, int nth, int tid,
                                              const double *sc) {
  constexpr int t0 = Patch::tptr[D], t1 = Patch::tptr[D + 1];
  constexpr int e = Patch::telem[t0];
  double s = dmul(es[e * nth + tid], sc[t0]);
#pragma unroll
  for (int m = 1; m < kTenM; ++m) s = dadd(s, dmul(es[(m * 24 + e) * nth + tid], sc[m * 72 + t0]));
  return ten_dir_terms<t0 + 1, t1>(s, es, nth, tid, sc);
}

template <int D, bool GS>
__device__ __forceinline__ void ten_nodal_acc(double &acc, double &diag, const double (&vq)[14],
                                              double v0, const double *es, int nth, int tid,
                                              const double *sc) {
  if constexpr (D < 14) {
    const double s = ten_dir_sum<D>(es, nth, tid, sc);
    if constexpr (GS) {
      acc = D == 0 ? dmul(s, vq[D]) : dadd(acc, dmul(s, vq[D]));
      diag = dsub(diag, s);
    } else {
      const double term = dmul(s, dsub(vq[D], v0));
      acc = D == 0 ? term : dadd(acc, term);
    }
    ten_nodal_acc<D + 1, GS>(acc, diag, vq, v0, es, nth, tid, sc);
  }
}

// one row of the tensor operator at interior point (i, j, k) of element t.
// GS=false: acc = sum_d s_d (v_d - v0).  GS=true: acc = sum_d s_d v_d and
// diag = -sum_d s_d.  `ut` / `gt`: value arrays (interior block or lattice,
// ghost shell), `kt`: the element's M component lattices.
template <bool NODAL, bool GS>
__device__ __forceinline__ void ten_row(const TenDesc &D, const IncPlanes &P, int i, int j,
                                        int k, const double *ut, const double *gt,
                                        const double *kt, const double *sc, double *es,
                                        int tid, int nth, double &acc, double &diag,
                                        double &v0) {
  const int n = D.n;
  const int L = (int)D.L;
  const int kp = inc_koff(P, 1, i, j);
  int ko[14];
  double vq[14];
#pragma unroll
  for (int d = 0; d < 14; ++d) {
    const int dk = c_dirs_h(d, 2);
    const int qi = i + c_dirs_h(d, 0), qj = j + c_dirs_h(d, 1);
    ko[d] = inc_koff(P, dk + 1, qi, qj);
    if (D.lattice) {
      vq[d] = ut[ko[d]];
    } else {
      int off;
      const bool in = inc_voff(P, dk + 1, n, qi, qj, k + dk, off);
      vq[d] = in ? ut[off] : gt[off];
    }
  }
  if (D.lattice) {
    v0 = ut[kp];
  } else {
    int off;
    inc_voff(P, 1, n, i, j, k, off);
    v0 = ut[off];
  }
  acc = 0.0;
  diag = 0.0;
  if constexpr (!NODAL) {
    double k0[kTenM];
#pragma unroll
    for (int m = 0; m < kTenM; ++m) k0[m] = __ldg(kt + m * L + kp);
#pragma unroll
    for (int d = 0; d < 14; ++d) {
      double s = dmul(dadd(k0[0], __ldg(kt + ko[d])), sc[d]);
#pragma unroll
      for (int m = 1; m < kTenM; ++m)
        s = dadd(s, dmul(dadd(k0[m], __ldg(kt + m * L + ko[d])), sc[m * 14 + d]));
      if constexpr (GS) {
        acc = d == 0 ? dmul(s, vq[d]) : dadd(acc, dmul(s, vq[d]));
        diag = dsub(diag, s);
      } else {
        const double term = dmul(s, dsub(vq[d], v0));
        acc = d == 0 ? term : dadd(acc, term);
      }
    }
  } else {
    // element sums of every component into this thread's smem column
#pragma unroll 1
    for (int m = 0; m < kTenM; ++m) {
      const double *km = kt + m * L;
      double b[55];
      b[0] = __ldg(km + kp);
#pragma unroll
      for (int d = 0; d < 14; ++d) b[1 + d] = __ldg(km + ko[d]);
      cse_steps<0>(b);
#pragma unroll
      for (int e = 0; e < 24; ++e) es[(m * 24 + e) * nth + tid] = b[31 + e];
    }
    ten_nodal_acc<0, GS>(acc, diag, vq, v0, es, nth, tid, sc);
  }
}

// apply / residual: grid (k - 1, j band, element), block (32, rows)
template <bool NODAL, bool RES>
__global__ void __launch_bounds__(ten_threads<NODAL>())
tensor_volume_kernel(TenDesc D) {
  extern __shared__ double ten_sm[];
  constexpr int NC = ten_ncoef<NODAL>();
  constexpr int NT = ten_threads<NODAL>();
  const int n = D.n;
  const int t = blockIdx.z;
  const int k = 1 + blockIdx.x;
  const int tid = threadIdx.y * 32 + threadIdx.x;
  double *sc = ten_sm;
  double *es = ten_sm + kTenM * NC;
  for (int e = tid; e < kTenM * NC; e += NT) sc[e] = D.coef[(long long)t * kTenM * NC + e];
  __syncthreads();
  const int j = 1 + blockIdx.y * ten_rows<NODAL>() + threadIdx.y;
  if (j > n - 2 - k) return;
  const IncPlanes P = inc_planes(n, k);
  const double *kt = D.km + (long long)t * kTenM * D.L;
  const double *ut = D.lattice ? D.u + (long long)t * D.L : D.u + D.vol_start[t];
  const double *gt = D.lattice ? nullptr : D.ghost + (long long)t * D.S;
  double *ot = D.lattice ? D.out + (long long)t * D.nvol : D.out + D.vol_start[t];
  const double *ft = D.f ? (D.lattice ? D.f + (long long)t * D.nvol : D.f + D.vol_start[t])
                         : nullptr;
  for (int i = 1 + threadIdx.x; i <= n - 1 - k - j; i += 32) {
    double acc, diag, v0;
    ten_row<NODAL, false>(D, P, i, j, k, ut, gt, kt, sc, es, tid, NT, acc, diag, v0);
    int c;
    inc_voff(P, 1, n, i, j, k, c);            // volume rank of (i, j, k)
    ot[c] = RES ? dsub(ft[c], acc) : acc;
  }
}

// forward Gauss-Seidel: one CTA per element walks the hyperplanes
// h = i + 2j + 3k (bitwise the lexicographic sweep, see hhg_smooth.cuh)
template <bool NODAL>
__global__ void __launch_bounds__(ten_threads<NODAL>())
tensor_gs_kernel(TenDesc D) {
  extern __shared__ double ten_sm[];
  constexpr int NC = ten_ncoef<NODAL>();
  constexpr int NT = ten_threads<NODAL>();
  const int n = D.n;
  const int t = blockIdx.x;
  const int tid = threadIdx.x;
  double *sc = ten_sm;
  double *es = ten_sm + kTenM * NC;
  for (int e = tid; e < kTenM * NC; e += NT) sc[e] = D.coef[(long long)t * kTenM * NC + e];
  __syncthreads();
  const double omega = D.omega;
  const double *kt = D.km + (long long)t * kTenM * D.L;
  double *ut = const_cast<double *>(D.lattice ? D.u + (long long)t * D.L
                                              : D.u + D.vol_start[t]);
  const double *gt = D.lattice ? nullptr : D.ghost + (long long)t * D.S;
  const double *ft = D.lattice ? D.f + (long long)t * D.nvol : D.f + D.vol_start[t];
  const int hmin = 6, hmax = 3 * n - 6;
  for (int h = hmin; h <= hmax; ++h) {
    const int ha = D.hp_ptr[h - hmin], hb = D.hp_ptr[h - hmin + 1];
    for (int e = ha + tid; e < hb; e += NT) {
      const int code = __ldg(D.hp_code + e);
      const int i = code & 1023, j = (code >> 10) & 1023, k = (code >> 20) & 1023;
      const IncPlanes P = inc_planes(n, k);
      double acc, diag, v0;
      ten_row<NODAL, true>(D, P, i, j, k, ut, gt, kt, sc, es, tid, NT, acc, diag, v0);
      if (diag == 0.0) atomicOr(&g_status, 1);
      int c;
      inc_voff(P, 1, n, i, j, k, c);
      const int pos = D.lattice ? inc_koff(P, 1, i, j) : c;
      ut[pos] = dadd(dmul(dsub(1.0, omega), v0), ddiv(dmul(omega, dsub(ft[c], acc)), diag));
    }
    __syncthreads();
  }
}

__constant__ int c_ten_tptr[15] = HHG_TPTR;
__constant__ int c_ten_telem[72] = HHG_TELEM;

// surface rows of the tensor operators, precomputed once (the tensor form
// of gs_surface_fill_kernel): per incidence and inside direction
//   scaled: w_d = sum_m (k_m0 + k_md) psh_m[cls][d]
//   nodal:  w_d = sum_{t in terms(d)} sum_m esum_m[telem[t]] pfac_m[cls][t]
// psh: [ntets][M][14][14], pfac: [ntets][M][14][72], km: [ntets][M][L]
__global__ void tensor_surface_fill_kernel(SurfGSDesc G, const double *km) {
  const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const SurfDesc &D = G.s;
  if (r >= D.nrows) return;
  const bool nodal = D.row_nodal[r] != 0;
  const long long L = D.L;
  double diag = 0.0;
  double *val = G.ent_val + G.ent_ptr[r];
  int *col = G.ent_col + G.ent_ptr[r];
  for (int x = D.inc_ptr[r]; x < D.inc_ptr[r + 1]; ++x) {
    const int t = D.inc_tet[x];
    const int code = D.inc_code[x];
    const int i = code & 1023, j = (code >> 10) & 1023, k = (code >> 20) & 1023;
    const int cls = D.inc_cls[x];
    const unsigned mask = c_cls_dirmask[cls];
    const double *kt = km + (long long)t * kTenM * L;
    const long long kp = lbase(D.n, k, j) + i;
    long long ko[14];
#pragma unroll
    for (int d = 0; d < 14; ++d) {
      ko[d] = kp;
      if (mask >> d & 1) {
        const int qi = i + c_dirs[d][0], qj = j + c_dirs[d][1], qk = k + c_dirs[d][2];
        ko[d] = lbase(D.n, qk, qj) + qi;
        *col++ = (int)point_gid(D, G.shell_gid, t, qi, qj, qk);
      }
    }
    if (!nodal) {
      for (int d = 0; d < 14; ++d) {
        if (!(mask >> d & 1)) continue;
        double s = 0.0;
        for (int m = 0; m < kTenM; ++m) {
          const double *sh = D.psh + (((long long)t * kTenM + m) * 14 + cls) * 14;
          const double x = dmul(dadd(kt[m * L + kp], kt[m * L + ko[d]]), sh[d]);
          s = m == 0 ? x : dadd(s, x);
        }
        *val++ = s;
        diag = dsub(diag, s);
      }
    } else {
      double es[kTenM][24];
      for (int m = 0; m < kTenM; ++m) {
        double b[55];
        b[0] = kt[m * L + kp];
        for (int d = 0; d < 14; ++d) b[1 + d] = kt[m * L + ko[d]];
        cse_steps<0>(b);
        for (int e = 0; e < 24; ++e) es[m][e] = b[31 + e];
      }
      for (int d = 0; d < 14; ++d) {
        if (!(mask >> d & 1)) continue;
        double s = 0.0;
        for (int T = c_ten_tptr[d]; T < c_ten_tptr[d + 1]; ++T)
          for (int m = 0; m < kTenM; ++m) {
            const double *fac = D.pfac + (((long long)t * kTenM + m) * 14 + cls) * 72;
            const double x = dmul(es[m][c_ten_telem[T]], fac[T]);
            s = (T == c_ten_tptr[d] && m == 0) ? x : dadd(s, x);
          }
        *val++ = s;
        diag = dsub(diag, s);
      }
    }
  }
  G.row_diag[r] = diag;
}

}  // namespace hhg
