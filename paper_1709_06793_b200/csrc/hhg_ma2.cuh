// 2-D scaled-stencil kernels with the uniform-ellipticity (MA2) gray-edge
// selector: kernels.apply_scaling_2d / gs_scaling_2d
// (pkg/src/hhgscale/kernels.py:750-782, 906-937).  On a triangle lattice of
// size n (row j starts at base[j] = j (n+1) - j (j-1)/2), an interior point
// p = (i, j) has six neighbours in DIRS_2D order (mesh.py:41-43); direction
// d takes the mean of the safeguarded coefficient kg when gray[d] is set
// (the reference's g array: the gray pair of a marked obtuse element,
// operators.py:88-129), else of kc.  Same operation order as the numba
// kernels: bitwise.
#pragma once
#include "hhg_common.cuh"

namespace hhg {

__device__ __forceinline__ int base2d(int n, int j) { return j * (n + 1) - j * (j - 1) / 2; }

__device__ __forceinline__ void nb2d(int n, int i, int j, int (&q)[6]) {
  const int b = base2d(n, j), bju = base2d(n, j + 1), bjd = base2d(n, j - 1), p = b + i;
  q[0] = p + 1;
  q[1] = bju + i;
  q[2] = bjd + i + 1;
  q[3] = p - 1;
  q[4] = bjd + i;
  q[5] = bju + i - 1;
}

// one thread per interior point; out in the reference's (j, i) order
__global__ void apply_scaling_2d_kernel(int n, const double *__restrict__ v,
                                        const double *__restrict__ kc,
                                        const double *__restrict__ kg, unsigned gray,
                                        const double *__restrict__ sh, double *__restrict__ out) {
  const int j = 1 + blockIdx.y;
  const int i = 1 + blockIdx.x * blockDim.x + threadIdx.x;
  if (j > n - 2 || i > n - 1 - j) return;
  int q[6];
  nb2d(n, i, j, q);
  const int p = base2d(n, j) + i;
  const double v0 = v[p];
  double acc = 0.0;
#pragma unroll
  for (int d = 0; d < 6; ++d) {
    const double sd = (gray >> d & 1) ? dmul(dadd(kg[p], kg[q[d]]), sh[d])
                                      : dmul(dadd(kc[p], kc[q[d]]), sh[d]);
    const double term = dmul(sd, dsub(v[q[d]], v0));
    acc = d == 0 ? term : dadd(acc, term);
  }
  out[(j - 1) * (n - 1) - (j - 1) * j / 2 + i - 1] = acc;
}

// forward Gauss-Seidel in (j, i) order as wavefronts h = i + 2j (every
// direction changes h with the sign of its lexicographic order), one CTA,
// block barrier between wavefronts: bitwise the sequential sweep
__global__ void gs_scaling_2d_kernel(int n, double *u, const double *__restrict__ fv,
                                     const double *__restrict__ kc,
                                     const double *__restrict__ kg, unsigned gray,
                                     const double *__restrict__ sh, double omega) {
  for (int h = 3; h <= 2 * n - 3; ++h) {
    // points of the wavefront: j in [1, n-2], i = h - 2j in [1, n-1-j]
    for (int j = 1 + threadIdx.x; j <= n - 2; j += blockDim.x) {
      const int i = h - 2 * j;
      if (i < 1 || i > n - 1 - j) continue;
      int q[6];
      nb2d(n, i, j, q);
      const int p = base2d(n, j) + i;
      double acc = 0.0, diag = 0.0;
#pragma unroll
      for (int d = 0; d < 6; ++d) {
        const double sd = (gray >> d & 1) ? dmul(dadd(kg[p], kg[q[d]]), sh[d])
                                          : dmul(dadd(kc[p], kc[q[d]]), sh[d]);
        acc = dadd(acc, dmul(sd, u[q[d]]));
        diag = dsub(diag, sd);
      }
      if (diag == 0.0) atomicOr(&g_status, 1);
      const int c = (j - 1) * (n - 1) - (j - 1) * j / 2 + i - 1;
      u[p] = dadd(dmul(dsub(1.0, omega), u[p]), ddiv(dmul(omega, dsub(fv[c], acc)), diag));
    }
    __syncthreads();
  }
}

}  // namespace hhg
