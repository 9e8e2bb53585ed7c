// Vector kernels for CG and multigrid: deterministic dot products, ratio
// axpys that read their scalars from device memory (no host round trip per
// CG iteration), and CSR products for the grid transfers.
#pragma once
#include "hhg_common.cuh"

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

__global__ void scatter_zero_kernel(long long n, const long long *ids, double *y) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e < n) y[ids[e]] = 0.0;
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

int hhg_scatter_zero(int64_t n, const int64_t *ids, double *y, void *stream) {
  if (n <= 0) return HHG_OK;
  hhg::scatter_zero_kernel<<<(int)((n + 255) / 256), 256, 0,
                             reinterpret_cast<cudaStream_t>(stream)>>>(
      n, reinterpret_cast<const long long *>(ids), y);
  return check("vector kernel");
}

}  // extern "C"
