// PCIe: does an SM-driven write stream into mapped pinned host memory get
// more device->host bandwidth beside a concurrent host->device copy than the
// copy engine does?  (the e2e apply's D2H leg runs at ~44 GB/s next to the
// H2D, 57 GB/s alone).  2.16 GB each way, like one config-5 apply.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void write_host(double *__restrict__ host, const double *__restrict__ dev, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    host[i] = dev[i];
}

int main() {
  const long long n = 270000000LL;
  const size_t bytes = n * sizeof(double);
  double *h_in, *h_out, *d_in, *d_out;
  cudaHostAlloc(&h_in, bytes, cudaHostAllocMapped);
  cudaHostAlloc(&h_out, bytes, cudaHostAllocMapped);
  cudaMalloc(&d_in, bytes);
  cudaMalloc(&d_out, bytes);
  cudaMemset(d_out, 0, bytes);
  for (long long i = 0; i < n; i += 4096) h_in[i] = 1.0;
  double *h_out_dev;
  cudaHostGetDevicePointer(&h_out_dev, h_out, 0);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](const char *name, auto body) {
    for (int w = 0; w < 2; ++w) {
      cudaDeviceSynchronize();
      cudaEventRecord(a, s1);
      cudaStreamWaitEvent(s2, a, 0);
      body();
      cudaEvent_t e2;
      cudaEventCreate(&e2);
      cudaEventRecord(e2, s2);
      cudaStreamWaitEvent(s1, e2, 0);
      cudaEventRecord(b, s1);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (w) printf("%-44s %8.2f ms\n", name, ms);
    }
  };
  for (int grid : {148, 296, 592, 1184}) {
    char nm[64];
    snprintf(nm, sizeof nm, "D2H kernel alone (grid %d)", grid);
    timeit(nm, [&] { write_host<<<grid, 256, 0, s2>>>(h_out_dev, d_out, n); });
  }
  timeit("D2H copy engine alone", [&] { cudaMemcpyAsync(h_out, d_out, bytes, cudaMemcpyDeviceToHost, s2); });
  timeit("H2D copy engine alone", [&] { cudaMemcpyAsync(d_in, h_in, bytes, cudaMemcpyHostToDevice, s1); });
  timeit("H2D + D2H copy engines", [&] {
    cudaMemcpyAsync(d_in, h_in, bytes, cudaMemcpyHostToDevice, s1);
    cudaMemcpyAsync(h_out, d_out, bytes, cudaMemcpyDeviceToHost, s2);
  });
  for (int grid : {148, 296, 592}) {
    char nm[64];
    snprintf(nm, sizeof nm, "H2D copy engine + D2H kernel (grid %d)", grid);
    timeit(nm, [&] {
      cudaMemcpyAsync(d_in, h_in, bytes, cudaMemcpyHostToDevice, s1);
      write_host<<<grid, 256, 0, s2>>>(h_out_dev, d_out, n);
    });
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
