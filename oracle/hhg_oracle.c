/*
 * hhg_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's numba kernels
 * (/root/reference/pkg/src/hhgscale/kernels.py), used as the parity checker
 * for the CUDA path and as the CPU baseline of bench.py ("kind": "port").
 * Only tests/, __graft_entry__.smoke() and bench.py's reference/cpu_baseline
 * legs may load it.  The product (paper_1709_06793_b200) never does.
 *
 * Arithmetic follows the reference operation by operation (same
 * association, no FMA: build with -ffp-contract=off), so outputs are
 * bitwise those of the numba kernels; tests/test_oracle_golden.py pins that
 * against vectors produced by the reference itself.
 *
 * Lattice conventions (mesh.py:457-504): flat order k, j, i; base[k*(n+1)+j]
 * is the first index of row (k, j).  Volume rows are visited in (k, j, i)
 * order, k in [1, n-3], j in [1, n-2-k], i in [1, n-1-k-j]
 * (kernels.py:94-103), and written sequentially.
 */
#include <stdint.h>
#include <stddef.h>

#define ORACLE_OK 0
#define ORACLE_ZERO_DIAG (-3)

/* neighbour flat indices of lattice point (i, j, k) in DIRS_3D order
 * (mesh.py:44-48), through the seven row bases of kernels.py:96-102 */
static inline void neighbours(const int64_t *base, int64_t n1, int64_t k, int64_t j,
                              int64_t i, int64_t nb[14]) {
  const int64_t b = base[k * n1 + j], bju = base[k * n1 + j + 1];
  const int64_t bjd = base[k * n1 + j - 1], bku = base[(k + 1) * n1 + j];
  const int64_t bkd = base[(k - 1) * n1 + j], bkdju = base[(k - 1) * n1 + j + 1];
  const int64_t bkujd = base[(k + 1) * n1 + j - 1];
  const int64_t p = b + i;
  nb[0] = p + 1;         nb[1] = bju + i;      nb[2] = bku + i;
  nb[3] = bjd + i + 1;   nb[4] = bkd + i + 1;  nb[5] = bkdju + i;
  nb[6] = bkujd + i + 1; nb[7] = p - 1;        nb[8] = bjd + i;
  nb[9] = bkd + i;       nb[10] = bju + i - 1; nb[11] = bku + i - 1;
  nb[12] = bkujd + i;    nb[13] = bkdju + i - 1;
}

#define FOR_VOLUME(n)                                   \
  for (int64_t k = 1; k < (n) - 2; ++k)                 \
    for (int64_t j = 1; j < (n) - 1 - k; ++j)           \
      for (int64_t i = 1; i < (n) - k - j; ++i)

/* kernels.py:90-136 */
void oracle_apply_scaling_3d(int64_t n, const int64_t *base, const double *v,
                             const double *kc, const double *sh, double *out) {
  const int64_t n1 = n + 1;
  int64_t c = 0, nb[14];
  FOR_VOLUME(n) {
    const int64_t p = base[k * n1 + j] + i;
    neighbours(base, n1, k, j, i, nb);
    const double v0 = v[p], k0 = kc[p];
    double acc = (k0 + kc[nb[0]]) * sh[0] * (v[nb[0]] - v0);
    for (int d = 1; d < 14; ++d) acc += (k0 + kc[nb[d]]) * sh[d] * (v[nb[d]] - v0);
    out[c++] = acc;
  }
}

/* element-sum buffer of the nodal kernels (kernels.py:161-166) */
static inline void nodal_sums(const double *kc, int64_t p, const int64_t nb[14],
                              const int64_t *sched, int64_t nsched, double buf[55]) {
  buf[0] = kc[p];
  for (int d = 0; d < 14; ++d) buf[1 + d] = kc[nb[d]];
  for (int64_t r = 0; r < nsched; ++r)
    buf[sched[3 * r]] = buf[sched[3 * r + 1]] + buf[sched[3 * r + 2]];
}

static inline double dir_sum(const double buf[55], const int64_t *sums, const double *fac,
                             const int64_t *tptr, const int64_t *telem, int d) {
  int64_t t0 = tptr[d];
  double s = buf[sums[telem[t0]]] * fac[t0];
  for (int64_t t = t0 + 1; t < tptr[d + 1]; ++t) s += buf[sums[telem[t]]] * fac[t];
  return s;
}

/* kernels.py:139-189 */
void oracle_apply_nodal_3d(int64_t n, const int64_t *base, const double *v,
                           const double *kc, const int64_t *sched, int64_t nsched,
                           const int64_t *sums, const double *fac, const int64_t *tptr,
                           const int64_t *telem, double *out) {
  const int64_t n1 = n + 1;
  int64_t c = 0, nb[14];
  double buf[55];
  FOR_VOLUME(n) {
    const int64_t p = base[k * n1 + j] + i;
    neighbours(base, n1, k, j, i, nb);
    nodal_sums(kc, p, nb, sched, nsched, buf);
    const double v0 = v[p];
    double acc = dir_sum(buf, sums, fac, tptr, telem, 0) * (v[nb[0]] - v0);
    for (int d = 1; d < 14; ++d)
      acc += dir_sum(buf, sums, fac, tptr, telem, d) * (v[nb[d]] - v0);
    out[c++] = acc;
  }
}

/* kernels.py:22-53 */
void oracle_apply_const_3d(int64_t n, const int64_t *base, const double *v,
                           const double *s, double c0, double *out) {
  const int64_t n1 = n + 1;
  int64_t c = 0, nb[14];
  FOR_VOLUME(n) {
    const int64_t p = base[k * n1 + j] + i;
    neighbours(base, n1, k, j, i, nb);
    double acc = c0 * v[p];
    for (int d = 0; d < 14; ++d) acc += s[d] * v[nb[d]];
    out[c++] = acc;
  }
}

/* kernels.py:56-87; w is [nvol][15] */
void oracle_apply_stored_3d(int64_t n, const int64_t *base, const double *v,
                            const double *w, double *out) {
  const int64_t n1 = n + 1;
  int64_t c = 0, nb[14];
  FOR_VOLUME(n) {
    const int64_t p = base[k * n1 + j] + i;
    neighbours(base, n1, k, j, i, nb);
    const double *wc = w + 15 * c;
    double acc = wc[0] * v[p];
    for (int d = 0; d < 14; ++d) acc += wc[1 + d] * v[nb[d]];
    out[c++] = acc;
  }
}

/* kernels.py:510-550 (in place on the lattice array u) */
int oracle_gs_scaling_3d(int64_t n, const int64_t *base, double *u, const double *fv,
                         const double *kc, const double *sh, double omega) {
  const int64_t n1 = n + 1;
  int64_t c = 0, nb[14];
  FOR_VOLUME(n) {
    const int64_t p = base[k * n1 + j] + i;
    neighbours(base, n1, k, j, i, nb);
    const double k0 = kc[p];
    double acc = 0.0, diag = 0.0;
    for (int d = 0; d < 14; ++d) {
      const double sd = (k0 + kc[nb[d]]) * sh[d];
      acc += sd * u[nb[d]];
      diag -= sd;
    }
    if (diag == 0.0) return ORACLE_ZERO_DIAG;
    u[p] = (1.0 - omega) * u[p] + omega * (fv[c] - acc) / diag;
    ++c;
  }
  return ORACLE_OK;
}

/* kernels.py:553-600 */
int oracle_gs_nodal_3d(int64_t n, const int64_t *base, double *u, const double *fv,
                       const double *kc, const int64_t *sched, int64_t nsched,
                       const int64_t *sums, const double *fac, const int64_t *tptr,
                       const int64_t *telem, double omega) {
  const int64_t n1 = n + 1;
  int64_t c = 0, nb[14];
  double buf[55];
  FOR_VOLUME(n) {
    const int64_t p = base[k * n1 + j] + i;
    neighbours(base, n1, k, j, i, nb);
    nodal_sums(kc, p, nb, sched, nsched, buf);
    double acc = 0.0, diag = 0.0;
    for (int d = 0; d < 14; ++d) {
      const double s = dir_sum(buf, sums, fac, tptr, telem, d);
      acc += s * u[nb[d]];
      diag -= s;
    }
    if (diag == 0.0) return ORACLE_ZERO_DIAG;
    u[p] = (1.0 - omega) * u[p] + omega * (fv[c] - acc) / diag;
    ++c;
  }
  return ORACLE_OK;
}

/* ---- tensor coefficients: km is [M][L], shm [M][14], fac [M][72] ---- */

/* s_d of the scaled tensor row, kernels.py:224-228 */
static inline double tensor_scaled(const double *km, int64_t M, int64_t L, int64_t p,
                                   int64_t q, const double *shm, int d) {
  double s = 0.0;
  for (int64_t m = 0; m < M; ++m) s += (km[m * L + p] + km[m * L + q]) * shm[m * 14 + d];
  return s;
}

/* element sums of every component (kernels.py:268-274); es is [M][24] */
static void tensor_esums(const double *km, int64_t M, int64_t L, int64_t p,
                         const int64_t nb[14], const int64_t *sched, int64_t nsched,
                         const int64_t *sums, double *es) {
  double buf[55];
  for (int64_t m = 0; m < M; ++m) {
    nodal_sums(km + m * L, p, nb, sched, nsched, buf);
    for (int e = 0; e < 24; ++e) es[m * 24 + e] = buf[sums[e]];
  }
}

/* s_d of the nodal tensor row, kernels.py:277-281 (terms outer, m inner) */
static inline double tensor_nodal(const double *es, int64_t M, const double *fac,
                                  const int64_t *tptr, const int64_t *telem, int d) {
  double s = 0.0;
  for (int64_t t = tptr[d]; t < tptr[d + 1]; ++t)
    for (int64_t m = 0; m < M; ++m) s += es[m * 24 + telem[t]] * fac[m * 72 + t];
  return s;
}

#define ORACLE_MAXM 8

/* kernels.py:192-232 */
void oracle_apply_scaling_tensor_3d(int64_t n, const int64_t *base, const double *v,
                                    const double *km, int64_t M, const double *shm,
                                    double *out) {
  const int64_t n1 = n + 1, L = (n + 1) * (n + 2) * (n + 3) / 6;
  int64_t c = 0, nb[14];
  FOR_VOLUME(n) {
    const int64_t p = base[k * n1 + j] + i;
    neighbours(base, n1, k, j, i, nb);
    const double v0 = v[p];
    double acc = 0.0;
    for (int d = 0; d < 14; ++d)
      acc += tensor_scaled(km, M, L, p, nb[d], shm, d) * (v[nb[d]] - v0);
    out[c++] = acc;
  }
}

/* kernels.py:235-286 */
int oracle_apply_nodal_tensor_3d(int64_t n, const int64_t *base, const double *v,
                                 const double *km, int64_t M, const int64_t *sched,
                                 int64_t nsched, const int64_t *sums, const double *fac,
                                 const int64_t *tptr, const int64_t *telem, double *out) {
  if (M > ORACLE_MAXM) return -1;
  const int64_t n1 = n + 1, L = (n + 1) * (n + 2) * (n + 3) / 6;
  int64_t c = 0, nb[14];
  double es[ORACLE_MAXM * 24];
  FOR_VOLUME(n) {
    const int64_t p = base[k * n1 + j] + i;
    neighbours(base, n1, k, j, i, nb);
    tensor_esums(km, M, L, p, nb, sched, nsched, sums, es);
    const double v0 = v[p];
    double acc = 0.0;
    for (int d = 0; d < 14; ++d)
      acc += tensor_nodal(es, M, fac, tptr, telem, d) * (v[nb[d]] - v0);
    out[c++] = acc;
  }
  return ORACLE_OK;
}

/* kernels.py:603-640 */
int oracle_gs_scaling_tensor_3d(int64_t n, const int64_t *base, double *u, const double *fv,
                                const double *km, int64_t M, const double *shm,
                                double omega) {
  const int64_t n1 = n + 1, L = (n + 1) * (n + 2) * (n + 3) / 6;
  int64_t c = 0, nb[14];
  FOR_VOLUME(n) {
    const int64_t p = base[k * n1 + j] + i;
    neighbours(base, n1, k, j, i, nb);
    double acc = 0.0, diag = 0.0;
    for (int d = 0; d < 14; ++d) {
      const double s = tensor_scaled(km, M, L, p, nb[d], shm, d);
      acc += s * u[nb[d]];
      diag -= s;
    }
    if (diag == 0.0) return ORACLE_ZERO_DIAG;
    u[p] = (1.0 - omega) * u[p] + omega * (fv[c] - acc) / diag;
    ++c;
  }
  return ORACLE_OK;
}

/* kernels.py:643-702 */
int oracle_gs_nodal_tensor_3d(int64_t n, const int64_t *base, double *u, const double *fv,
                              const double *km, int64_t M, const int64_t *sched,
                              int64_t nsched, const int64_t *sums, const double *fac,
                              const int64_t *tptr, const int64_t *telem, double omega) {
  if (M > ORACLE_MAXM) return -1;
  const int64_t n1 = n + 1, L = (n + 1) * (n + 2) * (n + 3) / 6;
  int64_t c = 0, nb[14];
  double es[ORACLE_MAXM * 24];
  FOR_VOLUME(n) {
    const int64_t p = base[k * n1 + j] + i;
    neighbours(base, n1, k, j, i, nb);
    tensor_esums(km, M, L, p, nb, sched, nsched, sums, es);
    double acc = 0.0, diag = 0.0;
    for (int d = 0; d < 14; ++d) {
      const double s = tensor_nodal(es, M, fac, tptr, telem, d);
      acc += s * u[nb[d]];
      diag -= s;
    }
    if (diag == 0.0) return ORACLE_ZERO_DIAG;
    u[p] = (1.0 - omega) * u[p] + omega * (fv[c] - acc) / diag;
    ++c;
  }
  return ORACLE_OK;
}

/* kernels.py:979-992 */
/* 2-D scaling kernels with the MA2 gray-edge selector (kernels.py:750-782,
 * 906-937): triangle lattice, base[j] row starts, interior rows j in
 * [1, n-2], i in [1, n-1-j]; direction d (DIRS_2D, mesh.py:41-43) uses the
 * safeguarded coefficient kg when g[d] != 0, else kc */
static inline void neighbours_2d(const int64_t *base, int64_t j, int64_t i, int64_t nb[6]) {
  const int64_t b = base[j], bju = base[j + 1], bjd = base[j - 1], p = b + i;
  nb[0] = p + 1;         nb[1] = bju + i;  nb[2] = bjd + i + 1;
  nb[3] = p - 1;         nb[4] = bjd + i;  nb[5] = bju + i - 1;
}

void oracle_apply_scaling_2d(int64_t n, const int64_t *base, const double *v,
                             const double *kc, const double *kg, const uint8_t *g,
                             const double *sh, double *out) {
  int64_t c = 0, nb[6];
  for (int64_t j = 1; j < n - 1; ++j)
    for (int64_t i = 1; i < n - j; ++i) {
      const int64_t p = base[j] + i;
      neighbours_2d(base, j, i, nb);
      const double v0 = v[p];
      double sd = g[0] ? (kg[p] + kg[p + 1]) * sh[0] : (kc[p] + kc[p + 1]) * sh[0];
      double acc = sd * (v[p + 1] - v0);
      for (int d = 1; d < 6; ++d) {
        const int64_t q = nb[d];
        sd = g[d] ? (kg[p] + kg[q]) * sh[d] : (kc[p] + kc[q]) * sh[d];
        acc += sd * (v[q] - v0);
      }
      out[c++] = acc;
    }
}

int oracle_gs_scaling_2d(int64_t n, const int64_t *base, double *u, const double *fv,
                         const double *kc, const double *kg, const uint8_t *g,
                         const double *sh, double omega) {
  int64_t c = 0, nb[6];
  for (int64_t j = 1; j < n - 1; ++j)
    for (int64_t i = 1; i < n - j; ++i) {
      const int64_t p = base[j] + i;
      neighbours_2d(base, j, i, nb);
      double acc = 0.0, diag = 0.0;
      for (int d = 0; d < 6; ++d) {
        const int64_t q = nb[d];
        const double sd = g[d] ? (kg[p] + kg[q]) * sh[d] : (kc[p] + kc[q]) * sh[d];
        acc += sd * u[q];
        diag -= sd;
      }
      if (diag == 0.0) return ORACLE_ZERO_DIAG;
      u[p] = (1.0 - omega) * u[p] + omega * (fv[c] - acc) / diag;
      ++c;
    }
  return ORACLE_OK;
}

int oracle_csr_gs(int64_t nrows, const int64_t *rows, const int32_t *indptr,
                  const int32_t *indices, const double *data, const double *diag,
                  double *u, const double *f, double omega) {
  for (int64_t ri = 0; ri < nrows; ++ri) {
    const int64_t r = rows[ri];
    double acc = 0.0;
    for (int64_t e = indptr[r]; e < indptr[r + 1]; ++e)
      if (indices[e] != r) acc += data[e] * u[indices[e]];
    const double d0 = diag[r];
    if (d0 == 0.0) return ORACLE_ZERO_DIAG;
    u[r] = (1.0 - omega) * u[r] + omega * (f[r] - acc) / d0;
  }
  return ORACLE_OK;
}

/* CPU baseline: the scaling kernel over a batch of macro elements, one
 * element at a time per POSIX thread (the reference runs them serially in
 * one process; this is the all-cores version of the same kernel). */
#include <pthread.h>
#include <stdatomic.h>
#include <unistd.h>

struct batch_job {
  int64_t n, ntets, L, nv;
  const int64_t *base;
  const double *v, *kc, *sh;
  double *out;
  atomic_llong next;
};

static void *batch_worker(void *arg) {
  struct batch_job *J = (struct batch_job *)arg;
  for (;;) {
    const long long t = atomic_fetch_add(&J->next, 1);
    if (t >= J->ntets) break;
    oracle_apply_scaling_3d(J->n, J->base, J->v + t * J->L, J->kc + t * J->L,
                            J->sh + 14 * t, J->out + t * J->nv);
  }
  return NULL;
}

int oracle_num_threads(void) {
  long c = sysconf(_SC_NPROCESSORS_ONLN);
  return c < 1 ? 1 : (int)c;
}

void oracle_apply_scaling_3d_batch(int64_t n, const int64_t *base, int64_t ntets,
                                   const double *v, const double *kc, const double *sh,
                                   double *out, int64_t nthreads) {
  struct batch_job J;
  J.n = n;
  J.ntets = ntets;
  J.L = (n + 1) * (n + 2) * (n + 3) / 6;
  J.nv = n >= 4 ? (n - 1) * (n - 2) * (n - 3) / 6 : 0;
  J.base = base;
  J.v = v;
  J.kc = kc;
  J.sh = sh;
  J.out = out;
  atomic_init(&J.next, 0);
  if (nthreads < 1) nthreads = oracle_num_threads();
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  for (int64_t i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, batch_worker, &J);
  for (int64_t i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
}
