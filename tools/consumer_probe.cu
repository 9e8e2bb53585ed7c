// Consumer-side microbenchmark of the volume kernel (no staging): the
// shared-memory plane ring is filled once, then every CTA walks planes as
// the FMA edge-flux consumer does - window loads, fma_step, one coalesced
// 8-byte store per output row - for as many rows as config 5 has (2.62e8).
//   variant 1: the shipped consumer, one column x 3 rows per thread
//              (8 x 4 lanes, 13 window loads per 3 rows)
//   variant 2: two adjacent columns x 3 rows per thread sharing the window
//              (4 col-pairs x 8 row groups per warp, 18 loads per 6 rows)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//        --expt-relaxed-constexpr -Xptxas -v tools/consumer_probe.cu -o consumer_probe
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1709_06793_b200/csrc/hhg_volume.cuh"

using namespace hhg;
constexpr int NS = 6, B = 3;

template <int VARIANT>
struct Geo;
template <>
struct Geo<1> {                 // 32 x 12 outputs per CTA
  static constexpr int ROWS = 4 * B + 2, COLS = 34, OUT = 128 * B;
};
template <>
struct Geo<2> {                 // 32 x 24 outputs per CTA, odd row stride
  static constexpr int ROWS = 8 * B + 2, COLS = 35, OUT = 128 * 2 * B;
};

template <int VARIANT>
__global__ void __launch_bounds__(128, 2) consumer(long long steps, double *out, double sh0) {
  using G = Geo<VARIANT>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2 *ring = reinterpret_cast<double2 *>(smem_raw);
  for (int e = threadIdx.x; e < NS * G::ROWS * G::COLS; e += blockDim.x)
    ring[e] = make_double2(1.0 + 1e-3 * ((e * 7919) % 1000), 2.0 + 1e-3 * ((e * 104729) % 997));
  __syncthreads();
  double sh[7];
#pragma unroll
  for (int d = 0; d < 7; ++d) sh[d] = sh0 * (d + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double *o = out + (long long)blockIdx.x * G::OUT;
  if constexpr (VARIANT == 1) {
    const int li = lane & 7, lj = lane >> 3;
    const int r0 = 1 + lj * B, c = 1 + warp * 8 + li;
    Win<B> X0, X1;
    double P[B];
    load_win<B, G::COLS>(X0, ring, r0, c);
    fma_seed<B>(X0, X0, sh, P);
    for (long long q = 0; q < steps; q += 2) {
      double v[B];
      load_win<B, G::COLS>(X1, ring + ((q + 1) % NS) * G::ROWS * G::COLS, r0, c);
      fma_step<B>(X0, X1, sh, P, v);
#pragma unroll
      for (int s = 0; s < B; ++s) __stcs(o + (s * 128 + threadIdx.x), v[s]);
      load_win<B, G::COLS>(X0, ring + ((q + 2) % NS) * G::ROWS * G::COLS, r0, c);
      fma_step<B>(X1, X0, sh, P, v);
#pragma unroll
      for (int s = 0; s < B; ++s) __stcs(o + (s * 128 + threadIdx.x), v[s]);
    }
  } else {
    // lanes 0-3: col-pairs 0-3 of row group 2k, lanes 4-7: row group 2k+1, ...
    const int li = lane & 3, lj = lane >> 2;
    const int r0 = 1 + lj * B, c = 1 + warp * 8 + 2 * li;
    struct W2 { double2 C0[B + 2], C1[B + 2], L[B + 1], R[B + 1]; };
    auto load2 = [&](W2 &w, const double2 *slot) {
      const double2 *b = slot + (r0 - 1) * G::COLS + c;
#pragma unroll
      for (int m = 0; m < B + 2; ++m) { w.C0[m] = b[m * G::COLS]; w.C1[m] = b[m * G::COLS + 1]; }
#pragma unroll
      for (int m = 0; m < B + 1; ++m) { w.L[m] = b[(m + 1) * G::COLS - 1]; w.R[m] = b[m * G::COLS + 2]; }
    };
    auto view0 = [&](const W2 &w) {   // column c: R = column c+1, L = column c-1
      Win<B> v;
#pragma unroll
      for (int m = 0; m < B + 2; ++m) v.C[m] = w.C0[m];
#pragma unroll
      for (int m = 0; m < B + 1; ++m) { v.R[m] = w.C1[m]; v.L[m] = w.L[m]; }
      return v;
    };
    auto view1 = [&](const W2 &w) {   // column c+1: R = column c+2, L = column c
      Win<B> v;
#pragma unroll
      for (int m = 0; m < B + 2; ++m) v.C[m] = w.C1[m];
#pragma unroll
      for (int m = 0; m < B + 1; ++m) { v.R[m] = w.R[m]; v.L[m] = w.C0[m + 1]; }
      return v;
    };
    W2 X0, X1;
    double P0[B], P1[B];
    load2(X0, ring);
    fma_seed<B>(view0(X0), view0(X0), sh, P0);
    fma_seed<B>(view1(X0), view1(X0), sh, P1);
    for (long long q = 0; q < steps; q += 2) {
      double v0[B], v1[B];
      load2(X1, ring + ((q + 1) % NS) * G::ROWS * G::COLS);
      fma_step<B>(view0(X0), view0(X1), sh, P0, v0);
      fma_step<B>(view1(X0), view1(X1), sh, P1, v1);
#pragma unroll
      for (int s = 0; s < B; ++s) {
        __stcs(o + (2 * s * 128 + 2 * threadIdx.x), v0[s]);
        __stcs(o + (2 * s * 128 + 2 * threadIdx.x + 1), v1[s]);
      }
      load2(X0, ring + ((q + 2) % NS) * G::ROWS * G::COLS);
      fma_step<B>(view0(X1), view0(X0), sh, P0, v0);
      fma_step<B>(view1(X1), view1(X0), sh, P1, v1);
#pragma unroll
      for (int s = 0; s < B; ++s) {
        __stcs(o + (2 * s * 128 + 2 * threadIdx.x), v0[s]);
        __stcs(o + (2 * s * 128 + 2 * threadIdx.x + 1), v1[s]);
      }
    }
  }
}

template <int VARIANT>
static void run(double *out) {
  using G = Geo<VARIANT>;
  const long long rows = 262188960LL;
  const int ctas = 148 * 2;
  const long long steps = (rows / ctas + G::OUT - 1) / G::OUT;   // planes per CTA
  const size_t smem = sizeof(double2) * NS * G::ROWS * G::COLS;
  cudaFuncSetAttribute(consumer<VARIANT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  consumer<VARIANT><<<ctas, 128, smem>>>(steps & ~1LL, out, 0.1);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) consumer<VARIANT><<<ctas, 128, smem>>>(steps & ~1LL, out, 0.1);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("variant %d: %.3f ms per 2.62e8 rows (%lld planes per CTA, smem %zu B) %s\n", VARIANT,
         ms / 5, steps, smem, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double *out;
  cudaMalloc(&out, sizeof(double) * 148 * 2 * 128 * 2 * B);
  run<1>(out);
  run<2>(out);
  run<1>(out);
  run<2>(out);
  return 0;
}
