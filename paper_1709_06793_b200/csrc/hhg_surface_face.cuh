// Face rows of the surface, tiled per macro face.
//
// A free macro-face point's row is the sum, over the (one or two) incident
// macro elements in ascending element order, of the one-sided partial
// stencil of that element (operators.py:329-365 assembled element-wise;
// hhg_surface.cuh).  Instead of one thread per stored incidence (two passes
// through a partial-sum array) or the precomputed weights of
// surface_csr_kernel (~400 B per row), one thread owns one face point and
// forms both partial rows from three face-parallel layers: the face itself
// and each incident element's lattice layer next to it, indexed by the
// face-local (a, b) of the reference's face numbering.  The coefficients of
// those layers never change, so they (and the global id of every layer
// point) are stored once per face in face-local order (hhg_surface.face_k /
// face_g); an apply streams them and gathers u through the ids.  A CTA owns
// 32 x 8 face points: it stages the three layers over the tile plus a
// one-point halo into shared memory, then every thread forms its row
// through the per-face direction -> layer offset table.  Same IEEE
// operations and order as the other two surface paths: results are bitwise
// theirs.
//
// Rows on macro edges and vertices (few) stay on surface_csr_kernel through
// a row sub-list.
#pragma once
#include "../../include/hhg_b200.h"
#include "hhg_smooth.cuh"

namespace hhg {

#ifndef HHG_FACE_TB
#define HHG_FACE_TB 8
#endif
constexpr int FACE_TA = 32, FACE_TB = HHG_FACE_TB;   // face tile: 32 (a) x TB (b) points
constexpr int FACE_W = FACE_TA + 2, FACE_H = FACE_TB + 2;   // staged region (halo 1)

template <bool RES, bool MIXED>
__global__ void __launch_bounds__(FACE_TA * FACE_TB)
surface_face_kernel(SurfGSDesc G, const hhg_surface s, double *out, SurfPush push) {
  // layer 0: the face points (shared by both elements); layer 1 + e: the
  // layer of element e next to the face; (v, k) pairs over the tile + halo
  constexpr int AREA = FACE_H * FACE_W;
  __shared__ double2 Ls[3 * AREA];
  __shared__ hhg_face F;
  __shared__ int offs[2][14];      // direction -> Ls offset relative to the point
  constexpr int NONE = -(1 << 20);   // direction leaving the element
  const SurfDesc &D = G.s;
  const int4 tl = reinterpret_cast<const int4 *>(s.face_tiles)[blockIdx.x];
  HHG_BOUND(tl.x, 0, s.nfaces, "face tile: face index");
  if (threadIdx.x < sizeof(hhg_face) / 4)
    reinterpret_cast<int *>(&F)[threadIdx.x] =
        reinterpret_cast<const int *>(s.faces + tl.x)[threadIdx.x];
  __syncthreads();
  const int n = D.n, a0 = tl.y, b0 = tl.z, sq = s.face_sq;
  const int ne = F.tet[1] >= 0 ? 2 : 1;
  if (threadIdx.x < 28) {
    const int e = threadIdx.x / 14, d = threadIdx.x % 14;
    const int l = F.dl[e][d];
    offs[e][d] = l < 0 ? NONE : (l == 0 ? 0 : 1 + e) * AREA + F.db[e][d] * FACE_W + F.da[e][d];
  }
  // stage: static k and global ids of the layers, u gathered through them.
  // All of a thread's id and k loads are issued first, then all its u
  // gathers: two dependent round trips per thread instead of two per point.
  const long long layer0 = (long long)tl.x * 3 * sq * sq;
  constexpr int NT = FACE_TA * FACE_TB, NIT = (3 * AREA + NT - 1) / NT;
  const int nx = (1 + ne) * AREA;
  const unsigned *gbase = reinterpret_cast<const unsigned *>(s.face_g) + layer0;
  const double *kbase = s.face_k + layer0;
  unsigned sg[NIT];
  double kv[NIT];
  int li[NIT];                                  // layer-local square index, -1: zero slot
#pragma unroll
  for (int it = 0; it < NIT; ++it) {
    const int x = threadIdx.x + it * NT;
    const int l = x / AREA, rem = x - l * AREA;
    const int rb = rem / FACE_W, ra = rem - rb * FACE_W;
    // square index of (a, b) = (a0 - 1 + ra, b0 - 1 + rb): (b + 1) sq + a + 1;
    // slots past the face's (n+3)^2 square stay zero
    li[it] = (x < nx && a0 + ra < sq && b0 + rb < sq) ? l * sq * sq + (b0 + rb) * sq + (a0 + ra) : -1;
    if (li[it] >= 0) {
      HHG_BOUND(li[it], 0, 3LL * sq * sq, "face staging: layer index");
      sg[it] = __ldg(gbase + li[it]);
      kv[it] = __ldg(kbase + li[it]);
    }
  }
#pragma unroll
  for (int it = 0; it < NIT; ++it) {
    const int x = threadIdx.x + it * NT;
    if (li[it] >= 0) Ls[x] = make_double2(__ldg(D.u + sg[it]), kv[it]);
    else if (x < nx) Ls[x] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  const int ta = threadIdx.x % FACE_TA, tb = threadIdx.x / FACE_TA;
  const int a = a0 + ta, b = b0 + tb;
  if (a < 1 || b < 1 || a + b > n - 1) return;
  const int ctr = (tb + 1) * FACE_W + (ta + 1);
  const double2 c0 = Ls[ctr];
  const double v0 = c0.x;
  double row = 0.0;
  for (int e = 0; e < ne; ++e) {
    const int t = F.tet[e], cls = F.cls[e];
    const unsigned mask = c_cls_dirmask[cls];
    double part;
    if (!MIXED || !F.nodal) {
      // only the directions of the one-sided stencil are read (all of them
      // stay inside the element, so their offsets are never NONE)
      const double *sh = D.psh + ((long long)t * 14 + cls) * 14;
      part = 0.0;
#pragma unroll
      for (int d = 0; d < 14; ++d)
        if (mask >> d & 1) {
          const int o = offs[e][d];
          HHG_BOUND(ctr + o, 0, 3 * AREA, "face row: staged neighbour");
          const double2 q = Ls[ctr + o];
          part = dadd(part, dmul(dmul(dadd(c0.y, q.y), __ldg(sh + d)), dsub(q.x, v0)));
        }
    } else {
      double2 q[14];
#pragma unroll
      for (int d = 0; d < 14; ++d) {
        const int o = offs[e][d];
        if (o != NONE) HHG_BOUND(ctr + o, 0, 3 * AREA, "face row: staged neighbour");
        q[d] = o == NONE ? make_double2(v0, 0.0) : Ls[ctr + o];
      }
      const double *fac = D.pfac + ((long long)t * 14 + cls) * 72;
      part = nodal_row_exact(v0, c0.y, q, fac);
    }
    row = dadd(row, part);
  }
  // interior face points are numbered fs + base2(b - 1) + a - 1 (face-local
  // (a, b) = the barycentrics of the face's 2nd and 3rd sorted vertices)
  const long long off = (long long)(b - 1) * (n - 2) - (long long)(b - 1) * (b - 2) / 2 + a - 1;
  const long long gid = F.fs + off;
  HHG_BOUND(off, 0, (long long)(n - 2) * (n - 1) / 2, "face row: face-local offset");
  if (RES) row = dsub(D.f[gid], row);
  out[gid] = row;
  if (!RES && push.slot) {
    const int sl = __ldg(push.slot + (F.rbase + off));
    if (sl >= 0) {
      if (sl < push.split) push.dst0[sl] = row;
      else push.dst1[sl - push.split] = row;
    }
  }
}

}  // namespace hhg
