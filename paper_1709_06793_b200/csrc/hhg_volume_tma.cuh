// Volume stencil kernel with TMA row staging (default scaling apply /
// residual of the batched operator, kernels.apply_scaling_3d semantics,
// pkg/src/hhgscale/kernels.py:90-136).
//
// Same work decomposition as volume_kernel_mirror (tiles of 32 i-columns x
// 4B j-rows of one macro element marching the k planes; hhg_grid.mtiles)
// but the plane ring is filled by the tensor-memory accelerator: per plane,
// one warp issues one 1-D TMA copy per lattice row and array (lane r: u row
// r, lane ROWS + r: k row r, one lane: the shell end-point strip), so the
// staging costs ~2 warp instructions per plane instead of ~30 8-byte
// cp.async plus their address arithmetic, and the LSU path is left to the
// window loads.
//
//  * u rows of the interior come straight from the caller's global vector
//    (the element's contiguous volume block, HHG numbering): a 34-wide box
//    starting at column i0-1 of row (j, p).  Its two shell end points
//    (i = 0 and i = n-p-j) are not in the volume block - the box carries the
//    neighbouring rows' values there - so after the plane has landed each
//    warp overwrites the shell slots it will read with the values of the
//    ghost-layer end-point strip (the ghost shell stores the end points of
//    consecutive rows next to each other, one TMA box per plane).
//  * u rows j = 0 and the whole plane p = 0 are shell rows: copied from the
//    ghost layer directly.
//  * k is complete per element (library-owned lattice layout): plain rows.
//
// TMA tile copies need a 16-byte-aligned global start and a 128-byte-aligned
// shared destination: every row is copied from the even element index at or
// below its first column (box of 36 doubles), so its data lands shifted by
// 0 or 1 slot; the producing warp publishes the shift bits of a plane (v
// rows, k rows, strip) in one word next to the slot's mbarriers and the
// consumers add them to their row addresses.  Shared rows are 48 doubles
// (384 B); v and k in separate rows; warps are 16 (i) x 2 (row groups) lane
// patches so a window load of one row touches 16 consecutive doubles per
// half-warp (two conflict-free wavefronts per 64-bit load).
//
// Arithmetic: MODE 0 = bitwise the reference order (mirror_step of
// hhg_volume.cuh); MODE 1 = FMA edge-flux form (each edge shared by two rows
// of a thread evaluated once, mirror pairs folded, down-plane terms
// pre-summed into one carry per row; ~48 instead of ~60 FP64 operations
// per row, within 1e-12 of the reference order).
#pragma once
#include <cudaTypedefs.h>

#include "hhg_volume.cuh"

// ablation switch for tools/tma_probe.py (0 in every product build):
// 1 = k rows not copied, 2 = u rows not copied, 3 = no arithmetic
#ifndef HHG_TMA_EXPT
#define HHG_TMA_EXPT 0
#endif
#ifndef HHG_TMA_PRODUCER_REGS
#define HHG_TMA_PRODUCER_REGS 24
#endif
#ifndef HHG_TMA_CONSUMER_REGS
#define HHG_TMA_CONSUMER_REGS 232
#endif

namespace hhg {

struct TmaMaps {
  CUtensorMap u;   // global vector, 1-D, box TMA_BOX doubles
  CUtensorMap g;   // ghost shells of all elements [ntets * S]
  CUtensorMap k;   // coefficient lattices of all elements [ntets * L]
};

constexpr int TMA_BOX = 36;     // 32 tile columns + 2 halo columns + alignment shift
constexpr int TMA_PITCH = 48;   // doubles per shared row (384 B)

__device__ __forceinline__ void tma_load_1d(unsigned dst, const CUtensorMap *map, int c0,
                                            unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2}], [%3];\n" ::"r"(dst),
      "l"(map), "r"(c0), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// --------------------------------------------------------------------------
// the kernel: 4 warps (2 along i x 2 along j), 16 x 2 lanes per warp, B rows
// per lane; tile = 32 columns x 4B rows (same tile list as the mirror kernel)
// --------------------------------------------------------------------------
template <int B>
struct TmaGeom {
  static constexpr int ROWS = 4 * B + 2;
  static constexpr int SLOT = (2 * ROWS + 1) * TMA_PITCH;   // doubles: v rows, k rows, strip
  static constexpr unsigned SLOT_BYTES = SLOT * sizeof(double);
  // NS slots, then NS full + NS empty mbarriers, then 3 NS shift words
  template <int NS>
  static constexpr unsigned smem_bytes() { return NS * SLOT_BYTES + 2 * NS * 8 + 3 * NS * 4; }
};

// Warp-specialised: warps 0-3 consume (fix-ups, windows, arithmetic,
// stores), warpgroup 1 produces - warp 4 the u rows, warp 5 the k rows,
// warp 6 the end-point strip - with setmaxnreg moving the producers'
// registers to the consumers; 2 CTAs per SM.
template <bool RES, int MODE, int B, int NS, int MINB>
__global__ void __launch_bounds__(256, MINB)
volume_kernel_tma(const __grid_constant__ TmaMaps M, VolDesc D) {
  constexpr int NW = 4;
  constexpr int ROWS = TmaGeom<B>::ROWS;
  constexpr int SLOT = TmaGeom<B>::SLOT;
  static_assert(ROWS <= 32, "one lane per staged row");
  static_assert(2 * B + 2 <= 16, "fix-up lanes cover the window rows of a warp");
  // dynamic shared memory only (the ring must start 128-byte aligned):
  // NS slots, then the full / empty mbarriers, then 3 shift words per slot
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double *ring = reinterpret_cast<double *>(smem_raw);
  const unsigned ring_s = static_cast<unsigned>(__cvta_generic_to_shared(ring));
  const unsigned full0 = ring_s + NS * TmaGeom<B>::SLOT_BYTES;
  const unsigned empty0 = full0 + NS * 8;
  // shift words of slot s: [3s] bit r = v row r, [3s+1] k row r, [3s+2] strip
  const unsigned *shiftw = reinterpret_cast<const unsigned *>(smem_raw + NS * TmaGeom<B>::SLOT_BYTES +
                                                              2 * NS * 8);
  const unsigned shift_s = full0 + 2 * NS * 8;

  const int4 tile = D.mtiles[blockIdx.x];
  const int t = tile.x, i0 = tile.y, j0 = tile.z, kmax = tile.w;
  const int n = D.n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int b = 0; b < NS; ++b) {
      mbar_init(full0 + 8 * b, 3);
      mbar_init(empty0 + 8 * b, NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp >= NW) {
    // ---------------- producers ----------------
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(HHG_TMA_PRODUCER_REGS) : "memory");
    const int pw = warp - NW;   // 0: u rows, 1: k rows, 2: strip
    if (pw > 2) return;
    const int vcoord = static_cast<int>(D.vol_start[t]);
    const int gcoord = t * static_cast<int>(D.S);
    const int kcoord = t * static_cast<int>(D.L);
    const int t2n = (n + 1) * (n + 2) / 2;
    const int jr = j0 - 1 + lane;
    for (int p = 0; p <= kmax + 1; ++p) {
      const int sl = p % NS;
      if (p >= NS) mbar_wait(empty0 + 8 * sl, ((p / NS) - 1) & 1);
      const int gpl = t2n + 3 * ((p - 1) * n - (p - 1) * p / 2);   // ghost plane p >= 1
      bool act;
      const CUtensorMap *map = &M.g;
      int want = 0;
      if (pw == 2) {
        act = lane == 0 && p >= 1;
        want = gcoord + gpl + (n - p + 1) + 2 * (j0 - 2);
      } else {
        act = lane < ROWS && jr <= n - p && (i0 - 1) + jr + p <= n;
        if (pw == 1) {
          map = &M.k;
          want = kcoord + lbase32(n, p, jr) + i0 - 1;
        } else if (p == 0) {
          want = gcoord + jr * (n + 1) - jr * (jr - 1) / 2 + i0 - 1;
        } else if (jr == 0) {
          want = gcoord + gpl + i0 - 1;
        } else {
          // inner-lattice offset of (i0-1, jr, p): iplane + (jr-1) rowi - (jr-1)(jr-2)/2 + i - 1
          const int m4 = n - 4;
          const int iplane = tetra32(m4) - tetra32(m4 - (p - 1));
          map = &M.u;
          want = vcoord + iplane + (jr - 1) * (n - 2 - p) - (jr - 1) * (jr - 2) / 2 + i0 - 2;
        }
      }
      const unsigned live = __ballot_sync(0xffffffffu, act);
      const unsigned shifts = __ballot_sync(0xffffffffu, act && (want & 1));
      if (lane == 0) {
        asm volatile("st.shared.u32 [%0], %1;\n" ::"r"(shift_s + 4 * (3 * sl + pw)), "r"(shifts)
                     : "memory");
        mbar_arrive_expect_tx(full0 + 8 * sl, __popc(live) * TMA_BOX * 8u);
      }
      __syncwarp();
      if (act) {
        const int row_off = pw == 2 ? 2 * ROWS : pw * ROWS + lane;
        tma_load_1d(ring_s + (unsigned)(sl * SLOT + row_off * TMA_PITCH) * 8u, map, want & ~1,
                    full0 + 8 * sl);
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(HHG_TMA_CONSUMER_REGS) : "memory");
  double sh[7];
#pragma unroll
  for (int d = 0; d < 7; ++d) sh[d] = __ldg(D.coef + (long long)t * D.coef_stride + d);
  double *To = opaque(D.out + D.vol_start[t]);
  const double *Tf = RES ? opaque(D.f + D.vol_start[t]) : nullptr;

  // lanes: 16 columns x 2 row groups per warp, warps 2 (i) x 2 (j)
  const int li = lane & 15, lj = lane >> 4;
  const int wi = warp & 1, wj = warp >> 1;
  const int cw0 = 1 + wi * 16;               // first tile column of the warp
  const int rw0 = 1 + wj * 2 * B;            // first tile row of the warp
  const int c = cw0 + li;
  const int r0 = rw0 + lj * B;
  const int i = i0 - 1 + c;
  const int jw = j0 - 1 + r0;
  const int warp_min_ij = i0 - 1 + cw0 + j0 - 1 + rw0;
  const int m4 = n - 4;
  int oterm[B];
#pragma unroll
  for (int s = 0; s < B; ++s) {
    const int jj = jw + s - 1;
    oterm[s] = -jj * (jj - 1) / 2 + i - 1;
  }
  // the warp's window: tile columns cw0-1 .. cw0+16, rows rw0-1 .. rw0+2B
  const bool fix_left = (i0 == 1) && (wi == 0);
  const int win_ij0 = (i0 - 1 + cw0 - 1) + (j0 - 1 + rw0 - 1);   // min i + j of the window

  // overwrite the shell slots of the warp's window (rows from the volume
  // block) with the end-point strip; lanes 0-15 left ends, 16-31 diagonal
  auto fixup = [&](int q, double *slot, unsigned sw, unsigned sws) {
    if (q < 1) return;
    const bool diag = win_ij0 + q <= n && n <= win_ij0 + q + 17 + 2 * B + 1;
    if (!fix_left && !diag) return;
    const int rr = lane & 15;
    const int r = rw0 - 1 + rr;
    const int jr = j0 - 1 + r;
    bool ok = rr < 2 * B + 2 && jr >= 1 && jr <= n - q;
    int col;
    if (lane < 16) {
      ok = ok && fix_left;
      col = 0;
    } else {
      const int id = n - q - jr;
      col = id - i0 + 1;
      ok = ok && id >= 1 && col >= cw0 - 1 && col <= cw0 + 16;
    }
    if (ok)
      slot[r * TMA_PITCH + col + ((sw >> r) & 1)] =
          slot[2 * ROWS * TMA_PITCH + 2 * r + (lane >> 4) + (sws & 1)];
    fence_proxy_async_smem();
    __syncwarp();
  };

  auto fetch = [&](int q, Win<B> &w) {
    const int sl = q % NS;
    mbar_wait(full0 + 8 * sl, (q / NS) & 1);
    double *slot = ring + sl * SLOT;
    const unsigned sw = shiftw[3 * sl];
    fixup(q, slot, sw, shiftw[3 * sl + 2]);
    const double *sv = slot + (r0 - 1) * TMA_PITCH + c;
    const double *sk = sv + ROWS * TMA_PITCH;
    const unsigned svw = sw >> (r0 - 1), skw = shiftw[3 * sl + 1] >> (r0 - 1);
#pragma unroll
    for (int m = 0; m < B + 2; ++m) {
      const double *pv = sv + m * TMA_PITCH + ((svw >> m) & 1);
      const double *pk = sk + m * TMA_PITCH + ((skw >> m) & 1);
      w.C[m] = make_double2(pv[0], pk[0]);
      if (m < B + 1) w.R[m] = make_double2(pv[1], pk[1]);
      if (m >= 1) w.L[m - 1] = make_double2(pv[-1], pk[-1]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * sl);
  };
  auto emit = [&](int kk, const double (&vals)[B]) {
    const int lim = n - 1 - kk;
    const int iplane = tetra32(m4) - tetra32(m4 - (kk - 1));
    const int rowi = m4 + 2 - kk;
#pragma unroll
    for (int s = 0; s < B; ++s)
      if (i + jw + s <= lim) {
        const int cidx = iplane + (jw + s - 1) * rowi + oterm[s];
        double val = vals[s];
        if (RES) val = dsub(__ldg(at(Tf, cidx)), val);
        __stcs(at(To, cidx), val);
      }
  };

  Win<B> X0, X1, X2;
  MirrorCarry<B> carry;   // MODE 0
  double P[B];            // MODE 1
  auto step = [&](int q, Win<B> &mi, Win<B> &hi) {
    fetch(q, hi);
    if (warp_min_ij <= n - q) {   // some lane of the warp is valid
      double vals[B];
      if constexpr (HHG_TMA_EXPT == 3) {
#pragma unroll
        for (int s = 0; s < B; ++s) vals[s] = hi.C[s + 1].x + mi.R[s].y + mi.L[s + 1].x;
      } else if constexpr (MODE == 0) {
        mirror_step<B>(mi, hi, sh, carry, vals);
      } else {
        fma_step<B>(mi, hi, sh, P, vals);
      }
      emit(q - 1, vals);
    }
  };

  if (kmax >= 1) {
    fetch(0, X0);
    fetch(1, X1);
    if (warp_min_ij <= n - 2) {
      if constexpr (MODE == 0) mirror_seed<B>(X0, X1, sh, carry);
      else fma_seed<B>(X0, X1, sh, P);
    }
    step(2, X1, X2);
    for (int q = 3; q <= kmax + 1; q += 3) {
      step(q, X2, X0);
      if (q + 1 > kmax + 1) break;
      step(q + 1, X0, X1);
      if (q + 2 > kmax + 1) break;
      step(q + 2, X1, X2);
    }
  }
  // every issued copy was consumed (each plane 0..kmax+1 is fetched): no
  // TMA can still be writing this CTA's shared memory
}

}  // namespace hhg
