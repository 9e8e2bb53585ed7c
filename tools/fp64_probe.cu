// FP64 throughput probe: independent DADD / DMUL / DFMA chains, many warps.
#include <cuda_runtime.h>
#include <cstdio>
template <int OP>
__global__ void probe(int iters, double *out, double seed) {
  double a[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) a[c] = seed + threadIdx.x * 1e-9 + c;
  const double b = 1.0000001, d = 1e-12;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (OP == 0) a[c] = __dadd_rn(a[c], d);
      else if (OP == 1) a[c] = __dmul_rn(a[c], b);
      else a[c] = fma(a[c], b, d);
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += a[c];
  if (s == 12345.0) out[0] = s;
}
int main() {
  double *out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096;
  for (int op = 0; op < 3; ++op)
    for (int warps : {4, 8, 16, 32}) {
      dim3 grid(148 * 4), block(32 * warps / 4);
      auto k = op == 0 ? probe<0> : op == 1 ? probe<1> : probe<2>;
      k<<<grid, block>>>(iters, out, 1.0);
      cudaEventRecord(e0);
      k<<<grid, block>>>(iters, out, 1.0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)grid.x * block.x * iters * 8;
      printf("op=%s warps/SM=%2d  %.1f Gop/s  = %.1f ops/clk/SM @1.965GHz\n",
             op == 0 ? "DADD" : op == 1 ? "DMUL" : "DFMA", warps, ops / ms / 1e6,
             ops / (ms * 1e-3) / 148 / 1.965e9);
    }
  // dependent chain latency: 1 warp per SM
  return 0;
}
