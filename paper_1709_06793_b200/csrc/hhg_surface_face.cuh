// Face rows of the surface, tiled per macro face (the default apply path).
//
// A free macro-face point's row is the sum, over the (one or two) incident
// macro elements in ascending element order, of the one-sided partial
// stencil of that element (operators.py:329-365 assembled element-wise;
// hhg_surface.cuh).  Instead of one thread per stored incidence (two passes
// through a partial-sum array) or the precomputed weights of
// surface_csr_kernel (~400 B per row), one thread owns one face point and
// forms both partial rows from the lattices directly: the point's
// coordinates in each incident element are affine in the face-local (a, b)
// (host-built per face: hhg_face), neighbours come from the element's volume
// block / ghost shell and coefficient lattice (inc_gather).  Tiles are 32 x 8
// face points, a running along the fastest lattice direction of the first
// element, so its reads are coalesced and the second element's cover a
// compact parallelogram.  Same IEEE operations and order as the other two
// surface paths: results are bitwise theirs.
//
// Rows on macro edges and vertices (few) stay on surface_csr_kernel through
// a row sub-list.
#pragma once
#include "../../include/hhg_b200.h"
#include "hhg_smooth.cuh"

namespace hhg {

constexpr int FACE_TA = 32, FACE_TB = 8;   // face tile: 32 (a) x 8 (b) points

template <bool RES, bool MIXED>
__global__ void __launch_bounds__(FACE_TA * FACE_TB)
surface_face_kernel(SurfGSDesc G, const hhg_face *faces, const int4 *tiles, double *out,
                    SurfPush push) {
  const SurfDesc &D = G.s;
  const int4 tl = tiles[blockIdx.x];
  const hhg_face &F = faces[tl.x];
  const int n = D.n;
  const int a = tl.y + (threadIdx.x % FACE_TA), b = tl.z + (threadIdx.x / FACE_TA);
  if (a < 1 || b < 1 || a + b > n - 1) return;
  double row = 0.0, v0 = 0.0;
  long long gid = 0;
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int t = F.tet[e];
    if (t < 0) break;
    const int i = F.c[e][0] + F.A[e][0] * a + F.A[e][1] * b;
    const int j = F.c[e][1] + F.A[e][2] * a + F.A[e][3] * b;
    const int k = F.c[e][2] + F.A[e][4] * a + F.A[e][5] * b;
    const int cls = F.cls[e];
    const unsigned mask = c_cls_dirmask[cls];
    if (e == 0) {
      const IncPlanes P = inc_planes(n, k);
      int off;
      inc_voff(P, 1, n, i, j, k, off);            // a boundary point: shell offset
      const long long s = (long long)t * D.S + off;
      v0 = D.ghost[s];
      gid = G.shell_gid[s];
    }
    double2 q[14];
    double k0;
    inc_gather(D, t, i, j, k, mask, v0, q, k0);
    double part;
    if (!MIXED || !F.nodal) {
      const double *sh = D.psh + ((long long)t * 14 + cls) * 14;
      part = 0.0;
#pragma unroll
      for (int d = 0; d < 14; ++d)
        if (mask >> d & 1)
          part = dadd(part, dmul(dmul(dadd(k0, q[d].y), __ldg(sh + d)), dsub(q[d].x, v0)));
    } else {
      const double *fac = D.pfac + ((long long)t * 14 + cls) * 72;
      part = nodal_row_exact(v0, k0, q, fac);
    }
    row = dadd(row, part);
  }
  if (RES) row = dsub(D.f[gid], row);
  out[gid] = row;
  if (!RES && push.slot) {
    const int sl = __ldg(push.slot + (F.rbase + (gid - F.fs)));
    if (sl >= 0) {
      if (sl < push.split) push.dst0[sl] = row;
      else push.dst1[sl - push.split] = row;
    }
  }
}

}  // namespace hhg
