// Standalone check of 1-D TMA row copies (tools/, not product code):
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tma_unit.cu -o /tmp/tma_unit
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

struct Maps {
  CUtensorMap a;
};

__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void expect(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma1d(unsigned dst, const void *map, int c0, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2}], [%3];\n" ::"r"(dst),
      "l"(map), "r"(c0), "r"(bar)
      : "memory");
}

// MODE 0: lane 0 issues all rows; MODE 1: lane r issues row r (divergent);
// map from the grid-constant parameter (P) or a global pointer (G)
template <int MODE, bool GLOBAL>
__global__ void kern(const __grid_constant__ Maps M, const CUtensorMap *gm, int nrows, int stride,
                     int pitch, int off, double *out) {
  extern __shared__ __align__(128) unsigned char sm[];
  double *rows = reinterpret_cast<double *>(sm);
  __shared__ __align__(8) unsigned long long bar;
  const unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
  const unsigned base = (unsigned)__cvta_generic_to_shared(rows);
  const CUtensorMap *map = GLOBAL ? gm : &M.a;
  if (threadIdx.x == 0) {
    mbar_init(b, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) expect(b, nrows * 34 * 8);
    __syncwarp();
    if (MODE == 0) {
      if (threadIdx.x == 0)
        for (int r = 0; r < nrows; ++r) tma1d(base + r * pitch * 8, map, r * stride + off, b);
    } else {
      const int r = threadIdx.x;
      if (r < nrows) tma1d(base + r * pitch * 8, map, r * stride + off, b);
    }
  }
  mbar_wait(b, 0);
  for (int e = threadIdx.x; e < nrows * 34; e += blockDim.x)
    out[e] = rows[(e / 34) * pitch + e % 34];
}

int main(int argc, char **argv) {
  const int N = 10000, nrows = 14;
  const int stride = argc > 2 ? atoi(argv[2]) : 101, off = argc > 3 ? atoi(argv[3]) : 3;
  const int which = argc > 1 ? atoi(argv[1]) : 0;
  std::vector<double> h(N);
  for (int i = 0; i < N; ++i) h[i] = i;
  double *d, *o;
  cudaMalloc(&d, N * 8);
  cudaMalloc(&o, nrows * 34 * 8);
  cudaMemcpy(d, h.data(), N * 8, cudaMemcpyHostToDevice);
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  Maps M;
  cuuint64_t dim[1] = {(cuuint64_t)N}, str[1] = {(cuuint64_t)N * 8};
  cuuint32_t box[1] = {34}, es[1] = {1};
  CUresult r = enc(&M.a, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, d, dim, str, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode rc %d\n", (int)r);
  CUtensorMap *gm;
  cudaMalloc(&gm, sizeof(CUtensorMap));
  cudaMemcpy(gm, &M.a, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  auto run = [&](const char *name, auto k, int pitch) {
    cudaMemset(o, 0, nrows * 34 * 8);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    k<<<1, 128, nrows * pitch * 8>>>(M, gm, nrows, stride, pitch, off, o);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<double> ho(nrows * 34);
    cudaMemcpy(ho.data(), o, ho.size() * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int rr = 0; rr < nrows; ++rr)
      for (int c = 0; c < 34; ++c) bad += ho[rr * 34 + c] != rr * stride + off + c;
    printf("%-28s pitch %3d: %s bad=%d\n", name, pitch, cudaGetErrorString(e), bad);
    return e == cudaSuccess;
  };
  bool ok = true;
  switch (which) {
    case 0: ok = run("lane0 param", kern<0, false>, 48); break;
    case 1: ok = run("lane0 global", kern<0, true>, 48); break;
    case 2: ok = run("divergent global", kern<1, true>, 48); break;
    case 3: ok = run("divergent param", kern<1, false>, 48); break;
    case 4: ok = run("lane0 param pitch36", kern<0, false>, 36); break;
    case 5: ok = run("lane0 param pitch34", kern<0, false>, 34); break;
  }
  return ok ? 0 : 1;
}
