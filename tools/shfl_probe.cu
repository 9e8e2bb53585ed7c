// SHFL throughput probe: independent shuffle chains, many warps per SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void probe(int iters, double *out) {
  double a[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) a[c] = threadIdx.x + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = __shfl_down_sync(0xffffffffu, a[c], 1);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += a[c];
  if (s == 123.0) out[0] = s;
}
int main() {
  double *o;
  cudaMalloc(&o, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    dim3 grid(148 * 4), block(32 * warps / 4);
    probe<8><<<grid, block>>>(iters, o);
    cudaEventRecord(e0);
    probe<8><<<grid, block>>>(iters, o);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // one double shuffle = 2 SHFL.32 warp instructions
    double shfl = 2.0 * grid.x * (block.x / 32) * iters * 8;
    printf("warps/SM=%2d: %.2f SHFL warp-instr/clk/SM @1.965GHz\n", warps,
           shfl / (ms * 1e-3) / 148 / 1.965e9);
  }
  return 0;
}
