#include <cstdio>
#include <cuda_runtime.h>
template <int OP, int CH>
__global__ void lat(int iters, double *out, long long *cyc, double seed) {
  double a[CH];
  for (int c = 0; c < CH; ++c) a[c] = seed + c + threadIdx.x;
  const double b = 1.0000001, d = 1e-12;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = OP == 0 ? __dadd_rn(a[c], d) : __dmul_rn(a[c], b);
  }
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < CH; ++c) s += a[c];
  if (s == 1234.5) out[0] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double *o; long long *c; cudaMalloc(&o, 8); cudaMalloc(&c, 8);
  int iters = 1 << 14;
  auto run = [&](auto k, const char *name, int ch, int warps) {
    k<<<1, 32 * warps>>>(iters, o, c, 1.0); cudaDeviceSynchronize();
    k<<<1, 32 * warps>>>(iters, o, c, 1.0);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%s chains=%d warps=%d: %.2f cycles per dependent op (per chain), %.3f warp-instr/clk\n",
           name, ch, warps, (double)h / iters, (double)ch * warps / ((double)h / iters));
  };
  run(lat<0, 1>, "DADD", 1, 1);
  run(lat<1, 1>, "DMUL", 1, 1);
  run(lat<0, 2>, "DADD", 2, 1);
  run(lat<0, 4>, "DADD", 4, 1);
  run(lat<0, 8>, "DADD", 8, 1);
  run(lat<0, 16>, "DADD", 16, 1);
  run(lat<0, 8>, "DADD", 8, 4);
  run(lat<0, 4>, "DADD", 4, 8);
  return 0;
}
