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
#include "hhg_volume.cuh"

namespace hhg {

constexpr int kTenM = 6;   // 3-D splitting (TENSOR_DIRS_3D)

struct TenDesc {
  int n, ntets;
  long long L, S, nvol;
  const long long *vol_start;  // first volume id per element (split layout)
  const double *km;            // [ntets][L][M] (batched) or [M][L] (per element)
  const double *u;             // element lattices [ntets*L]
  const double *ghost;         // gather: compact shells [ntets*S]
  const double *f;             // residual / GS rhs (global or [ntets*nvol])
  double *out;                 // apply: global or [ntets*nvol]
  const double *coef;          // shm [ntets][M][14] or fac [ntets][M][72]
  int out_split;               // 1: rows / f addressed through vol_start
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

// component values of lattice point q: AOS = [L][M] (the batched device
// layout, one 48-byte record per point: 3 x 16-byte loads), else [M][L]
// (the reference's km layout, kept for the per-element ABI)
template <bool AOS>
__device__ __forceinline__ void ten_k6(const double *kt, int L, int q, double (&k)[kTenM]) {
  if constexpr (AOS) {
    const double2 *p = reinterpret_cast<const double2 *>(kt + kTenM * q);
#pragma unroll
    for (int h = 0; h < kTenM / 2; ++h) {
      const double2 v = __ldg(p + h);
      k[2 * h] = v.x;
      k[2 * h + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int m = 0; m < kTenM; ++m) k[m] = __ldg(kt + m * L + q);
  }
}

// one row of the tensor operator at interior point (i, j, k) of element t,
// all operands in the element's lattice arrays (`ut` values, `kt` the M
// component lattices): every neighbour address is affine in i, so the row
// constants hoist out of the i loop.  GS=false: acc = sum_d s_d (v_d - v0).
// GS=true: acc = sum_d s_d v_d and diag = -sum_d s_d.
template <bool NODAL, bool GS, bool AOS>
__device__ __forceinline__ void ten_row(const TenDesc &D, const IncPlanes &P, int i, int j,
                                        const double *ut, const double *kt, const double *sc,
                                        double *es, int tid, int nth, double &acc,
                                        double &diag, double &v0) {
  const int L = (int)D.L;
  const int kp = inc_koff(P, 1, i, j);
  int ko[14];
  double vq[14];
#pragma unroll
  for (int d = 0; d < 14; ++d) {
    ko[d] = inc_koff(P, c_dirs_h(d, 2) + 1, i + c_dirs_h(d, 0), j + c_dirs_h(d, 1));
    vq[d] = ut[ko[d]];
  }
  v0 = ut[kp];
  acc = 0.0;
  diag = 0.0;
  if constexpr (!NODAL) {
    double k0[kTenM];
    ten_k6<AOS>(kt, L, kp, k0);
#pragma unroll
    for (int d = 0; d < 14; ++d) {
      double kq[kTenM];
      ten_k6<AOS>(kt, L, ko[d], kq);
      double s = dmul(dadd(k0[0], kq[0]), sc[d]);
#pragma unroll
      for (int m = 1; m < kTenM; ++m) s = dadd(s, dmul(dadd(k0[m], kq[m]), sc[m * 14 + d]));
      if constexpr (GS) {
        acc = d == 0 ? dmul(s, vq[d]) : dadd(acc, dmul(s, vq[d]));
        diag = dsub(diag, s);
      } else {
        const double term = dmul(s, dsub(vq[d], v0));
        acc = d == 0 ? term : dadd(acc, term);
      }
    }
  } else {
    // element sums of every component into this thread's smem column;
    // per-point base pointers once, components at immediate offsets
    const double *pq[15];
    pq[0] = AOS ? kt + kTenM * kp : kt + kp;
#pragma unroll
    for (int d = 0; d < 14; ++d) pq[1 + d] = AOS ? kt + kTenM * ko[d] : kt + ko[d];
#pragma unroll 1
    for (int m = 0; m < kTenM; ++m) {
      const int mo = AOS ? m : m * L;
      double b[55];
#pragma unroll
      for (int x = 0; x < 15; ++x) b[x] = __ldg(pq[x] + mo);
      cse_steps<0>(b);
#pragma unroll
      for (int e = 0; e < 24; ++e) es[(m * 24 + e) * nth + tid] = b[31 + e];
    }
    ten_nodal_acc<0, GS>(acc, diag, vq, v0, es, nth, tid, sc);
  }
}

// apply / residual: grid (k - 1, j band, element), block (32, rows).
// Inputs: lattice values D.u [ntets*L]; rows written to the global vector
// (D.out_split: vol_start[t] + rank) or per element [ntets*nvol].
template <bool NODAL, bool RES, bool AOS>
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
  const double *ut = D.u + (long long)t * D.L;
  const long long o0 = D.out_split ? D.vol_start[t] : (long long)t * D.nvol;
  double *ot = D.out + o0;
  const double *ft = RES ? D.f + o0 : nullptr;
  // volume rank of (i, j, k): inner-lattice row (k-1, j-1) + i - 1
  const int c0 = P.ib[1] + (j - 1) * P.ri[1] - (j - 1) * (j - 2) / 2 - 1;
  for (int i = 1 + threadIdx.x; i <= n - 1 - k - j; i += 32) {
    double acc, diag, v0;
    ten_row<NODAL, false, AOS>(D, P, i, j, ut, kt, sc, es, tid, NT, acc, diag, v0);
    ot[c0 + i] = RES ? dsub(ft[c0 + i], acc) : acc;
  }
}

// ---------------------------------------------------------------------------
// Staged apply: a CTA owns a tile of 32 columns (i) x TR rows (j) of one
// element and marches the planes k upward.  Every plane of the tile plus a
// one-point halo (34 x (TR+2) points: value + 48-byte component record) is
// copied into a 4-slot shared-memory ring with cp.async, two planes ahead;
// each thread then forms one row of plane k from slots k-1, k, k+1.  Same
// arithmetic and order as ten_row (bitwise equal), but the 15 neighbour
// records come from shared memory instead of 15 scattered L1/L2 requests.
// ---------------------------------------------------------------------------
constexpr int kTenCols = 34;     // 32 + halo
constexpr int kTenNS = 4;        // ring slots (planes k-1, k, k+1, k+2)

template <bool NODAL>
constexpr int tt_rows() { return NODAL ? 2 : 4; }   // tile rows (j)
template <bool NODAL>
constexpr int tt_per() { return NODAL ? 1 : 2; }    // rows per thread
template <bool NODAL>
constexpr int tt_threads() { return 32 * tt_rows<NODAL>() / tt_per<NODAL>(); }
template <bool NODAL>
constexpr size_t tt_smem() {
  return sizeof(double) * ((size_t)kTenNS * (tt_rows<NODAL>() + 2) * kTenCols * (1 + kTenM) +
                           kTenM * ten_ncoef<NODAL>() +
                           (NODAL ? (size_t)kTenM * 24 * tt_threads<NODAL>() : 0));
}

template <bool NODAL, bool RES>
__global__ void __launch_bounds__(tt_threads<NODAL>())
tensor_tile_kernel(TenDesc D, const int4 *tiles) {
  constexpr int TR = tt_rows<NODAL>();
  constexpr int P = tt_per<NODAL>();
  constexpr int NT = tt_threads<NODAL>();
  constexpr int PTS = (TR + 2) * kTenCols;        // staged points per plane
  constexpr int NC = ten_ncoef<NODAL>();
  extern __shared__ __align__(16) double tt_sm[];
  double *sv = tt_sm;                              // [NS][PTS] values
  double *sk = sv + kTenNS * PTS;                  // [NS][PTS][M] records
  double *sc = sk + kTenNS * PTS * kTenM;          // coefficients
  double *es = sc + kTenM * NC;                    // nodal element sums
  const int4 tile = tiles[blockIdx.x];
  const int t = tile.x, i0 = tile.y, j0 = tile.z, kmax = tile.w;
  const int n = D.n;
  const int tid = threadIdx.x, lane = tid & 31, wr = tid >> 5;
  for (int e = tid; e < kTenM * NC; e += NT) sc[e] = D.coef[(long long)t * kTenM * NC + e];
  const double *ut = D.u + (long long)t * D.L;
  const double *kt = D.km + (long long)t * kTenM * D.L;

  auto stage = [&](int p) {
    if (p <= n) {
      const int slot = p % kTenNS;
      const int tn = n - p;                        // plane p is a size-(n-p) triangle
      const int pb = tetra32(n) - tetra32(n - p);  // lattice offset of plane p
#pragma unroll
      for (int r = 0; r < (PTS + NT - 1) / NT; ++r) {
        const int e = tid + r * NT;
        if (e < PTS) {
          const int rr = e / kTenCols, cc = e - rr * kTenCols;
          const int si = i0 - 1 + cc, sj = j0 - 1 + rr;
          if (si >= 0 && sj >= 0 && si + sj <= tn) {
            const int off = pb + sj * (tn + 1) - sj * (sj - 1) / 2 + si;
            cp_async8(sv + slot * PTS + e, ut + off);
            const double *src = kt + (long long)kTenM * off;
            double *dst = sk + ((long long)slot * PTS + e) * kTenM;
#pragma unroll
            for (int h = 0; h < kTenM / 2; ++h) {
              const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst + 2 * h));
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d),
                           "l"(src + 2 * h));
            }
          }
        }
      }
    }
    cp_async_commit();
  };

  stage(0);
  stage(1);
  stage(2);
  const int i = i0 + lane;
  const int lx = lane + 1;
  const long long o0 = D.out_split ? D.vol_start[t] : (long long)t * D.nvol;
  double *ot = D.out + o0;
  const double *ft = RES ? D.f + o0 : nullptr;
  const int m4 = n - 4;
  for (int k = 1; k <= kmax; ++k) {
    stage(k + 2);
    cp_async_wait<1>();                            // planes <= k + 1 have landed
    __syncthreads();
    const int s0 = ((k - 1) % kTenNS) * PTS, s1 = (k % kTenNS) * PTS,
              s2 = ((k + 1) % kTenNS) * PTS;
    // this thread's rows j = j0 + wr + q * (TR / P), q < P
    bool live[P];
    int pc[P];
    int po[P][14];
    double v0[P], acc[P];
#pragma unroll
    for (int q = 0; q < P; ++q) {
      const int ly = wr + q * (TR / P) + 1;
      live[q] = i + (j0 + ly - 1) + k <= n - 1;
      pc[q] = s1 + ly * kTenCols + lx;
      v0[q] = sv[pc[q]];
#pragma unroll
      for (int d = 0; d < 14; ++d) {
        const int dk = c_dirs_h(d, 2);
        const int sb = dk < 0 ? s0 : (dk > 0 ? s2 : s1);
        po[q][d] = sb + (ly + c_dirs_h(d, 1)) * kTenCols + lx + c_dirs_h(d, 0);
      }
    }
    bool any = false;
#pragma unroll
    for (int q = 0; q < P; ++q) any |= live[q];
    if (any) {
      if constexpr (!NODAL) {
        double k0[P][kTenM];
#pragma unroll
        for (int q = 0; q < P; ++q)
#pragma unroll
          for (int m = 0; m < kTenM; ++m) k0[q][m] = sk[pc[q] * kTenM + m];
#pragma unroll
        for (int d = 0; d < 14; ++d) {
          double cd[kTenM];                        // component weights of d, shared by the rows
#pragma unroll
          for (int m = 0; m < kTenM; ++m) cd[m] = sc[m * 14 + d];
#pragma unroll
          for (int q = 0; q < P; ++q) {
            const double *kq = sk + po[q][d] * kTenM;
            double s = dmul(dadd(k0[q][0], kq[0]), cd[0]);
#pragma unroll
            for (int m = 1; m < kTenM; ++m) s = dadd(s, dmul(dadd(k0[q][m], kq[m]), cd[m]));
            const double term = dmul(s, dsub(sv[po[q][d]], v0[q]));
            acc[q] = d == 0 ? term : dadd(acc[q], term);
          }
        }
      } else {
        // P == 1
#pragma unroll 1
        for (int m = 0; m < kTenM; ++m) {
          double b[55];
          b[0] = sk[pc[0] * kTenM + m];
#pragma unroll
          for (int d = 0; d < 14; ++d) b[1 + d] = sk[po[0][d] * kTenM + m];
          cse_steps<0>(b);
#pragma unroll
          for (int e = 0; e < 24; ++e) es[(m * 24 + e) * NT + tid] = b[31 + e];
        }
        double vq[14], diag = 0.0;
#pragma unroll
        for (int d = 0; d < 14; ++d) vq[d] = sv[po[0][d]];
        ten_nodal_acc<0, false>(acc[0], diag, vq, v0[0], es, NT, tid, sc);
      }
#pragma unroll
      for (int q = 0; q < P; ++q)
        if (live[q]) {
          const int j = j0 + wr + q * (TR / P);
          // volume rank of (i, j, k): inner-lattice row (k-1, j-1) + i - 1
          const int c = tetra32(m4) - tetra32(m4 - (k - 1)) + (j - 1) * (n - 2 - k) -
                        (j - 1) * (j - 2) / 2 + i - 1;
          ot[c] = RES ? dsub(ft[c], acc[q]) : acc[q];
        }
    }
    __syncthreads();                               // slot (k-1) % NS is refilled next
  }
  cp_async_wait<0>();
}

// forward Gauss-Seidel on the lattice arrays: one CTA per element walks
// the hyperplanes h = i + 2j + 3k (bitwise the lexicographic sweep, see
// hhg_smooth.cuh); f is global (D.out_split) or per element
template <bool NODAL, bool AOS>
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
  double *ut = const_cast<double *>(D.u) + (long long)t * D.L;
  const double *ft = D.f + (D.out_split ? D.vol_start[t] : (long long)t * D.nvol);
  const int hmin = 6, hmax = 3 * n - 6;
  for (int h = hmin; h <= hmax; ++h) {
    const int ha = D.hp_ptr[h - hmin], hb = D.hp_ptr[h - hmin + 1];
    for (int e = ha + tid; e < hb; e += NT) {
      const int code = __ldg(D.hp_code + e);
      const int i = code & 1023, j = (code >> 10) & 1023, k = (code >> 20) & 1023;
      const IncPlanes P = inc_planes(n, k);
      double acc, diag, v0;
      ten_row<NODAL, true, AOS>(D, P, i, j, ut, kt, sc, es, tid, NT, acc, diag, v0);
      if (diag == 0.0) atomicOr(&g_status, 1);
      const int c = P.ib[1] + (j - 1) * P.ri[1] - (j - 1) * (j - 2) / 2 + i - 1;
      ut[inc_koff(P, 1, i, j)] =
          dadd(dmul(dsub(1.0, omega), v0), ddiv(dmul(omega, dsub(ft[c], acc)), diag));
    }
    __syncthreads();
  }
}

// element lattices from the split global layout: interior points from the
// element's volume block, shell points from its compact ghost shell (the
// reference's u[elem_gidx[t]], operators.py:383).  grid (k, j band, element)
__global__ void __launch_bounds__(128)
lattice_gather_kernel(TenDesc D, double *lat) {
  const int n = D.n;
  const int t = blockIdx.z;
  const int k = blockIdx.x;
  const int j = blockIdx.y * 4 + threadIdx.y;
  if (j > n - k) return;
  const IncPlanes P = inc_planes(n, k);
  const double *vt = D.u + D.vol_start[t];
  const double *gt = D.ghost + (long long)t * D.S;
  double *lt = lat + (long long)t * D.L + inc_koff(P, 1, 0, j);
  for (int i = threadIdx.x; i <= n - k - j; i += 32) {
    int off;
    const bool in = inc_voff(P, 1, n, i, j, k, off);
    lt[i] = in ? vt[off] : gt[off];
  }
}

// interior values back into the global vector after a lattice GS sweep
// (operators.py:464-466); grid (k - 1, j band, element)
__global__ void __launch_bounds__(128)
lattice_scatter_kernel(TenDesc D, const double *lat, double *u) {
  const int n = D.n;
  const int t = blockIdx.z;
  const int k = 1 + blockIdx.x;
  const int j = 1 + blockIdx.y * 4 + threadIdx.y;
  if (j > n - 2 - k) return;
  const IncPlanes P = inc_planes(n, k);
  const double *lt = lat + (long long)t * D.L + inc_koff(P, 1, 0, j);
  double *vt = u + D.vol_start[t] + P.ib[1] + (j - 1) * P.ri[1] - (j - 1) * (j - 2) / 2 - 1;
  for (int i = 1 + threadIdx.x; i <= n - 1 - k - j; i += 32) vt[i] = lt[i];
}

__constant__ int c_ten_tptr[15] = HHG_TPTR;
__constant__ int c_ten_telem[72] = HHG_TELEM;

// surface rows of the tensor operators, precomputed once (the tensor form
// of gs_surface_fill_kernel): per incidence and inside direction
//   scaled: w_d = sum_m (k_m0 + k_md) psh_m[cls][d]
//   nodal:  w_d = sum_{t in terms(d)} sum_m esum_m[telem[t]] pfac_m[cls][t]
// psh: [ntets][M][14][14], pfac: [ntets][M][14][72], km: [ntets][L][M]
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
          const double x = dmul(dadd(kt[kTenM * kp + m], kt[kTenM * ko[d] + m]), sh[d]);
          s = m == 0 ? x : dadd(s, x);
        }
        *val++ = s;
        diag = dsub(diag, s);
      }
    } else {
      double es[kTenM][24];
      for (int m = 0; m < kTenM; ++m) {
        double b[55];
        b[0] = kt[kTenM * kp + m];
        for (int d = 0; d < 14; ++d) b[1 + d] = kt[kTenM * ko[d] + m];
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
