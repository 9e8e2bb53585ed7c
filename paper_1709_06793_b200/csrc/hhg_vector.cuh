// Vector kernels for CG and multigrid: deterministic dot products, ratio
// axpys that read their scalars from device memory (no host round trip per
// CG iteration), and CSR products for the grid transfers.
#pragma once
#include "hhg_common.cuh"
#include "hhg_transfer.cuh"

namespace hhg {

constexpr int DOT_BLOCKS = 1024;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-level tree sum; result valid in thread 0
__device__ __forceinline__ double block_sum(double v, double *sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  v = (threadIdx.x < (blockDim.x >> 5)) ? sh[l] : 0.0;
  if (w == 0) v = warp_sum(v);
  return v;
}

__global__ void dot_partial(long long n, const double *__restrict__ x,
                            const double *__restrict__ y, double *work) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    acc = fma(x[i], y[i], acc);
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) work[blockIdx.x] = acc;
}

__global__ void dot_final(int nb, const double *work, double *result) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) acc += work[i];
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) result[0] = acc;
}

// ---------------------------------------------------------------------------
// fused CG / PCG updates (multigrid.py:169-194): one pass per update with
// the next dot product's partials formed on the way.  Launched with the dot
// geometry (dot_blocks x 256, grid-stride), so every partial sum is formed
// in exactly the order dot_partial would form it: the iterates are bitwise
// those of the separate axpy / dot sequence.
// ---------------------------------------------------------------------------

// a = rs / pAp;  x += a p;  r -= a Ap;  work[block] = partial sum of r.r
// (over the entries with mask != 0 when a mask is given: sharded vectors)
__global__ void cg_update_kernel(long long n, const double *rs, const double *pAp,
                                 const double *__restrict__ p, const double *__restrict__ Ap,
                                 double *__restrict__ x, double *__restrict__ r,
                                 const unsigned char *__restrict__ mask, double *work) {
  __shared__ double sh[32];
  const double a = 1.0 * (rs[0] / pAp[0]);
  const double na = -1.0 * (rs[0] / pAp[0]);
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    x[i] += a * p[i];
    const double ri = r[i] + na * Ap[i];
    r[i] = ri;
    if (!mask || mask[i]) acc = fma(ri, ri, acc);
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) work[blockIdx.x] = acc;
}

// PCG: a = rz / pAp;  x += a p;  rn = r - a Ap;  work = partials of rn.rn
__global__ void pcg_update_kernel(long long n, const double *rz, const double *pAp,
                                  const double *__restrict__ p, const double *__restrict__ Ap,
                                  double *__restrict__ x, const double *__restrict__ r,
                                  double *__restrict__ rn, double *work) {
  __shared__ double sh[32];
  const double a = rz[0] / pAp[0];
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    x[i] += a * p[i];
    const double v = r[i] - a * Ap[i];
    rn[i] = v;
    acc = fma(v, v, acc);
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) work[blockIdx.x] = acc;
}

// two dots in one pass: work[b] = partial of (a - b).c, work[nb + b] = a.c
__global__ void dot2_partial(long long n, const double *__restrict__ a,
                             const double *__restrict__ b, const double *__restrict__ c,
                             double *work) {
  __shared__ double sh[32];
  double d1 = 0.0, d2 = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double ci = c[i], ai = a[i];
    d1 = fma(ai - b[i], ci, d1);
    d2 = fma(ai, ci, d2);
  }
  d1 = block_sum(d1, sh);
  __syncthreads();
  d2 = block_sum(d2, sh);
  if (threadIdx.x == 0) {
    work[blockIdx.x] = d1;
    work[gridDim.x + blockIdx.x] = d2;
  }
}

// owner-masked dot (sharded vectors: every shared node counted once)
__global__ void dot_masked_partial(long long n, const double *__restrict__ x,
                                   const double *__restrict__ y,
                                   const unsigned char *__restrict__ mask, double *work) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    if (mask[i]) acc = fma(x[i], y[i], acc);
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) work[blockIdx.x] = acc;
}

// final sums of k partial arrays of nb entries each: result[q] = sum work[q nb ..]
__global__ void dot_final_multi(int nb, int k, const double *work, double *result) {
  __shared__ double sh[32];
  for (int q = 0; q < k; ++q) {
    double acc = 0.0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) acc += work[q * nb + i];
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) result[q] = acc;
    __syncthreads();
  }
}

__global__ void axpy_ratio_kernel(long long n, const double *num, const double *den,
                                  double sign, const double *__restrict__ x,
                                  double *__restrict__ y) {
  const double a = sign * (num[0] / den[0]);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] += a * x[i];
}

__global__ void xpay_ratio_kernel(long long n, const double *num, const double *den,
                                  const double *__restrict__ r, double *__restrict__ p) {
  const double b = num[0] / den[0];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = r[i] + b * p[i];
}

// thread per row, stored column order: bitwise the scipy csr_matvec sum
__global__ void csr_spmv_kernel(long long nrows, const long long *indptr,
                                const long long *indices, const double *data,
                                const double *x, double *y, int accumulate) {
  const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  double s = 0.0;
  for (long long e = indptr[r]; e < indptr[r + 1]; ++e)
    s = dadd(s, dmul(data[e], x[indices[e]]));
  y[r] = accumulate ? dadd(y[r], s) : s;
}

// rows r of a row-listed CSR: y[rows[r]] (+)= sum_e val[e] x[col[e]] in
// stored order (the surface rows of the grid transfers)
__global__ void csr_rows_kernel(long long nrows, const long long *rows, const long long *ptr,
                                const long long *col, const double *val, const double *x,
                                double *y, int accumulate) {
  const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  double s = 0.0;
  for (long long e = ptr[r]; e < ptr[r + 1]; ++e) s = dadd(s, dmul(val[e], x[col[e]]));
  const long long g = rows[r];
  y[g] = accumulate ? dadd(y[g], s) : s;
}

__global__ void scatter_zero_kernel(long long n, const long long *ids, double *y) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e < n) y[ids[e]] = 0.0;
}

// interface exchange over NCCL (shard.exchange_partials): pack the
// one-sided interface rows, then complete them in rank order
__global__ void gather_kernel(long long n, const long long *ids, const double *x, double *y) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e < n) y[e] = x[ids[e]];
}
__global__ void interface_add_kernel(long long n, const long long *ids, const double *mine,
                                     const double *recv, int recv_first, double *out) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e < n) out[ids[e]] = recv_first ? dadd(recv[e], mine[e]) : dadd(mine[e], recv[e]);
}

}  // namespace hhg

extern "C" {

static inline int vec_grid(long long n) {
  long long b = (n + 255) / 256;
  if (b > 148 * 8) b = 148 * 8;
  return (int)(b < 1 ? 1 : b);
}

int hhg_dot(int64_t n, const double *x, const double *y, double *work, double *result,
            void *stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int nb = (int)((n + 255) / 256);
  if (nb > hhg::DOT_BLOCKS) nb = hhg::DOT_BLOCKS;
  if (nb < 1) nb = 1;
  hhg::dot_partial<<<nb, 256, 0, st>>>(n, x, y, work);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  hhg::dot_final<<<1, 1024, 0, st>>>(nb, work, result);
  return check("dot");
}

static inline int dot_blocks(long long n) {
  int nb = (int)((n + 255) / 256);
  if (nb > hhg::DOT_BLOCKS) nb = hhg::DOT_BLOCKS;
  return nb < 1 ? 1 : nb;
}

int hhg_cg_update(int64_t n, const double *rs, const double *pAp, const double *p,
                  const double *Ap, double *x, double *r, const uint8_t *mask, double *work,
                  double *rs_new, void *stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int nb = dot_blocks(n);
  hhg::cg_update_kernel<<<nb, 256, 0, st>>>(n, rs, pAp, p, Ap, x, r, mask, work);
  int rc = check("cg_update_kernel");
  if (rc) return rc;
  hhg::dot_final<<<1, 1024, 0, st>>>(nb, work, rs_new);
  return check("dot_final");
}

int hhg_pcg_update(int64_t n, const double *rz, const double *pAp, const double *p,
                   const double *Ap, double *x, const double *r, double *r_new, double *work,
                   double *rr_new, void *stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int nb = dot_blocks(n);
  hhg::pcg_update_kernel<<<nb, 256, 0, st>>>(n, rz, pAp, p, Ap, x, r, r_new, work);
  int rc = check("pcg_update_kernel");
  if (rc) return rc;
  hhg::dot_final<<<1, 1024, 0, st>>>(nb, work, rr_new);
  return check("dot_final");
}

int hhg_dot2(int64_t n, const double *a, const double *b, const double *c, double *work,
             double *result, void *stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int nb = dot_blocks(n);
  hhg::dot2_partial<<<nb, 256, 0, st>>>(n, a, b, c, work);
  int rc = check("dot2_partial");
  if (rc) return rc;
  hhg::dot_final_multi<<<1, 1024, 0, st>>>(nb, 2, work, result);
  return check("dot_final_multi");
}

int hhg_dot_masked(int64_t n, const double *x, const double *y, const uint8_t *mask,
                   double *work, double *result, void *stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int nb = dot_blocks(n);
  hhg::dot_masked_partial<<<nb, 256, 0, st>>>(n, x, y, mask, work);
  int rc = check("dot_masked_partial");
  if (rc) return rc;
  hhg::dot_final<<<1, 1024, 0, st>>>(nb, work, result);
  return check("dot_final");
}

int hhg_axpy_ratio(int64_t n, const double *num, const double *den, double sign,
                   const double *x, double *y, void *stream) {
  hhg::axpy_ratio_kernel<<<vec_grid(n), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      n, num, den, sign, x, y);
  return check("vector kernel");
}

int hhg_xpay_ratio(int64_t n, const double *num, const double *den, const double *r,
                   double *p, void *stream) {
  hhg::xpay_ratio_kernel<<<vec_grid(n), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      n, num, den, r, p);
  return check("vector kernel");
}

int hhg_csr_spmv(int64_t nrows, const int64_t *indptr, const int64_t *indices,
                 const double *data, const double *x, double *y, int accumulate,
                 void *stream) {
  if (nrows <= 0) return HHG_OK;
  hhg::csr_spmv_kernel<<<(int)((nrows + 255) / 256), 256, 0,
                         reinterpret_cast<cudaStream_t>(stream)>>>(
      nrows, reinterpret_cast<const long long *>(indptr),
      reinterpret_cast<const long long *>(indices), data, x, y, accumulate);
  return check("vector kernel");
}

int hhg_prolongate(const hhg_transfer *T, const double *xc, double *yf, int accumulate,
                   void *stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (T->nf >= 4 && T->ntets > 0) {
    hhg::prolong_volume_kernel<<<dim3(T->nf - 3, T->ntets), 256, 0, st>>>(*T, xc, yf,
                                                                          accumulate);
    int rc = check("prolong_volume_kernel");
    if (rc) return rc;
  }
  if (T->p_nrows > 0) {
    hhg::csr_rows_kernel<<<(int)((T->p_nrows + 255) / 256), 256, 0, st>>>(
        T->p_nrows, reinterpret_cast<const long long *>(T->p_rows),
        reinterpret_cast<const long long *>(T->p_ptr),
        reinterpret_cast<const long long *>(T->p_col), T->p_val, xc, yf, accumulate);
    return check("csr_rows_kernel");
  }
  return HHG_OK;
}

int hhg_restrict(const hhg_transfer *T, const double *xf, double *yc, void *stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (T->nc >= 4 && T->ntets > 0) {
    hhg::restrict_volume_kernel<<<dim3(T->nc - 3, T->ntets), 128, 0, st>>>(*T, xf, yc);
    int rc = check("restrict_volume_kernel");
    if (rc) return rc;
  }
  if (T->r_nrows > 0) {
    hhg::csr_rows_kernel<<<(int)((T->r_nrows + 255) / 256), 256, 0, st>>>(
        T->r_nrows, reinterpret_cast<const long long *>(T->r_rows),
        reinterpret_cast<const long long *>(T->r_ptr),
        reinterpret_cast<const long long *>(T->r_col), T->r_val, xf, yc, 0);
    int rc = check("csr_rows_kernel");
    if (rc) return rc;
  }
  if (T->ndir > 0) {
    hhg::scatter_zero_kernel<<<(int)((T->ndir + 255) / 256), 256, 0, st>>>(
        T->ndir, reinterpret_cast<const long long *>(T->c_dir_ids), yc);
    return check("scatter_zero_kernel");
  }
  return HHG_OK;
}

int hhg_gather(int64_t n, const int64_t *ids, const double *x, double *y, void *stream) {
  if (n <= 0) return HHG_OK;
  if (!ids || !x || !y) return HHG_ERR_ARG;
  hhg::gather_kernel<<<(int)((n + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      n, reinterpret_cast<const long long *>(ids), x, y);
  return check("gather_kernel");
}

int hhg_interface_add(int64_t n, const int64_t *ids, const double *mine, const double *recv,
                      int recv_first, double *out, void *stream) {
  if (n <= 0) return HHG_OK;
  if (!ids || !mine || !recv || !out) return HHG_ERR_ARG;
  hhg::interface_add_kernel<<<(int)((n + 255) / 256), 256, 0,
                              reinterpret_cast<cudaStream_t>(stream)>>>(
      n, reinterpret_cast<const long long *>(ids), mine, recv, recv_first, out);
  return check("interface_add_kernel");
}

int hhg_scatter_zero(int64_t n, const int64_t *ids, double *y, void *stream) {
  if (n <= 0) return HHG_OK;
  hhg::scatter_zero_kernel<<<(int)((n + 255) / 256), 256, 0,
                             reinterpret_cast<cudaStream_t>(stream)>>>(
      n, reinterpret_cast<const long long *>(ids), y);
  return check("vector kernel");
}

}  // extern "C"
