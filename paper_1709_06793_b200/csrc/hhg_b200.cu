// libhhg_b200: extern "C" entry points (include/hhg_b200.h) over the sm_100a
// kernels in hhg_volume.cuh / hhg_surface.cuh / hhg_smooth.cuh.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <set>
#include <tuple>
#include <vector>

#include "../../include/hhg_b200.h"
#include "hhg_common.cuh"
#include "hhg_smooth.cuh"
#include "hhg_ma2.cuh"
#include "hhg_surface.cuh"
#include "hhg_surface_face.cuh"
#include "hhg_tensor.cuh"
#include "hhg_volume.cuh"
#ifndef HHG_VOLUME_TMA
#define HHG_VOLUME_TMA 0   // experimental TMA-staged kernel (profiles/README.md, round 2)
#endif
#if HHG_VOLUME_TMA
#include "hhg_volume_tma.cuh"
#endif

using namespace hhg;

#ifndef HHG_VOL_B
#define HHG_VOL_B 3
#endif
#ifndef HHG_VOL_W
#define HHG_VOL_W 4
#endif
#ifndef HHG_VOL_NS
#define HHG_VOL_NS 6
#endif

#ifndef HHG_VOL_MINB
#define HHG_VOL_MINB 2
#endif

static constexpr int kB = HHG_VOL_B, kW = HHG_VOL_W, kNS = HHG_VOL_NS;

static inline cudaStream_t S(void *s) { return reinterpret_cast<cudaStream_t>(s); }
// dynamic shared-memory opt-in of a kernel, once per (device, kernel)
static std::mutex g_attr_mu;
static int smem_optin(const void *kern, int bytes) {
  static std::set<std::pair<int, const void *>> done;
  std::lock_guard<std::mutex> lock(g_attr_mu);
  int dev = 0;
  cudaGetDevice(&dev);
  if (done.count({dev, kern})) return HHG_OK;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) !=
      cudaSuccess)
    return HHG_ERR_CUDA;
  done.insert({dev, kern});
  return HHG_OK;
}

// every kernel launch of the library goes through check(): it also counts
// them (hhg_launch_count, bench.py's gpu_launches)
static std::atomic<long long> g_launches{0};
static inline int check(const char *what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "hhg_b200: %s: %s\n", what, cudaGetErrorString(e));
    return HHG_ERR_CUDA;
  }
  return HHG_OK;
}

// ---------------------------------------------------------------------------
// volume kernel dispatch
// ---------------------------------------------------------------------------
// tile geometry: every variant covers kW*kB rows per tile (the host tile
// list depends only on that product); the nodal kernel keeps one output row
// per thread (its 55-slot element-sum buffer needs the registers)
template <int VAR>
struct VolGeom {
  static constexpr int B = (VAR == 1) ? 1 : kB;
  static constexpr int W = (VAR == 1) ? kW * kB : kW;
};
// tile = 32 columns x (W * B) rows; warps are 8 x 4 lane patches
static_assert(kW % 4 == 0, "tile width is 4 warps of 8 columns");

template <int VAR, int SRC, bool RES, bool FAST, bool MIRROR = false>
static int launch_volume(const VolDesc &D, cudaStream_t st) {
  if (D.ntiles <= 0) return HHG_OK;
  constexpr int B = VolGeom<VAR>::B, W = VolGeom<VAR>::W;
  static_assert(B * W == kB * kW, "tile rows must not depend on the variant");
  constexpr int ROWS = W * B + 2;
  const size_t smem = sizeof(double2) * kNS * ROWS * VOL_COLS + 72 * sizeof(double);
  constexpr int MINB = (VAR == 1) ? 1 : HHG_VOL_MINB;
  auto kern = volume_kernel<VAR, SRC, RES, FAST, B, W, kNS, MINB, MIRROR>;
  if (smem_optin((const void *)kern, (int)smem)) return HHG_ERR_CUDA;
  kern<<<D.ntiles, 32 * W, smem, st>>>(D);
  return check("volume_kernel");
}

#ifndef HHG_MIRROR_NW
#define HHG_MIRROR_NW 4          // warps per CTA = tile columns / 8
#endif
#ifndef HHG_MIRROR_MINB
#define HHG_MIRROR_MINB (8 / HHG_MIRROR_NW)
#endif
#ifndef HHG_MIRROR_FMA_MINB
#define HHG_MIRROR_FMA_MINB HHG_MIRROR_MINB
#endif

template <int SRC, bool RES, int MODE = 0>
static int launch_mirror(const VolDesc &D, cudaStream_t st) {
  if (D.nmtiles <= 0) return D.ntiles > 0 ? HHG_ERR_ARG : HHG_OK;
  static_assert(kW == 4, "the mirror kernel uses 8x4-lane warps of 4B rows");
  constexpr int NW = HHG_MIRROR_NW;
  constexpr int ROWS = 4 * kB + 2;
  const size_t smem = sizeof(double2) * kNS * ROWS *
                      (HHG_VOL_SOA ? HHG_VOL_CS : 8 * NW + 2);
#ifndef HHG_VOLUME_WS
#define HHG_VOLUME_WS 0          // warp-specialised producer / consumer form
#endif
  if (HHG_VOLUME_WS && NW == 4) {
    auto kern = volume_kernel_ws<SRC, RES, kB, kNS, MODE>;
    if (smem_optin((const void *)kern, (int)smem)) return HHG_ERR_CUDA;
    kern<<<D.nmtiles, 256, smem, st>>>(D);
    return check("volume_kernel_ws");
  }
  constexpr int MB = MODE == 1 ? HHG_MIRROR_FMA_MINB : HHG_MIRROR_MINB;
  auto kern = volume_kernel_mirror<SRC, RES, kB, kNS, MB, NW, MODE>;
  if (smem_optin((const void *)kern, (int)smem)) return HHG_ERR_CUDA;
  kern<<<D.nmtiles, 32 * NW, smem, st>>>(D);
  return check("volume_kernel_mirror");
}

#if HHG_VOLUME_TMA
// ---------------------------------------------------------------------------
// TMA-staged scaling kernel (hhg_volume_tma.cuh): 1-D tensor maps over the
// global vector, the ghost shells and the coefficient lattices, encoded per
// call (host-side, ~1 us each; the u pointer changes between calls)
// ---------------------------------------------------------------------------
#ifndef HHG_TMA_NS
#define HHG_TMA_NS 6
#endif
#ifndef HHG_TMA_MINB
#define HHG_TMA_MINB 2
#endif
#ifndef HHG_TMA_L2PROMO
#define HHG_TMA_L2PROMO 2        // CU_TENSOR_MAP_L2_PROMOTION_L2_128B
#endif

static PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

static bool tma_map_1d(CUtensorMap *m, const void *base, long long len) {
  auto enc = tma_encoder();
  if (!enc || len <= 0) return false;
  cuuint64_t dim[1] = {(cuuint64_t)len};
  cuuint64_t stride[1] = {(cuuint64_t)len * 8};   // unused for rank 1
  cuuint32_t box[1] = {(cuuint32_t)TMA_BOX}, es[1] = {1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, const_cast<void *>(base), dim, stride, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             (CUtensorMapL2promotion)HHG_TMA_L2PROMO,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// TMA coordinates are 32-bit element indices
static bool tma_fits(const VolDesc &D) {
  const long long lim = (1LL << 31) - 64;
  return D.n_nodes > 0 && D.n_nodes < lim && (long long)D.ntets * D.L < lim &&
         (long long)D.ntets * D.S < lim && D.n >= 8 && D.nmtiles > 0;
}

template <bool RES, int MODE>
static int launch_tma(const VolDesc &D, cudaStream_t st) {
  static_assert(HHG_MIRROR_NW == 4, "the TMA kernel uses the 32-column mirror tiles");
  TmaMaps M;
  if (!tma_map_1d(&M.u, D.u, D.n_nodes) || !tma_map_1d(&M.g, D.ghost, (long long)D.ntets * D.S) ||
      !tma_map_1d(&M.k, D.kc, (long long)D.ntets * D.L))
    return HHG_ERR_CUDA;
  constexpr unsigned smem = TmaGeom<kB>::smem_bytes<HHG_TMA_NS>();
  auto kern = volume_kernel_tma<RES, MODE, kB, HHG_TMA_NS, HHG_TMA_MINB>;
  if (smem_optin((const void *)kern, (int)smem)) return HHG_ERR_CUDA;
  kern<<<D.nmtiles, 256, smem, st>>>(M, D);
  return check("volume_kernel_tma");
}
#else
static bool tma_fits(const VolDesc &) { return false; }
template <bool RES, int MODE>
static int launch_tma(const VolDesc &, cudaStream_t) { return HHG_ERR_ARG; }
#endif

template <int SRC>
static int dispatch_volume(const VolDesc &D, int variant, int flags, cudaStream_t st) {
  const bool res = flags & HHG_FLAG_RESIDUAL;
  const bool fast = flags & HHG_FLAG_FAST;
  const bool mirror = flags & HHG_FLAG_MIRROR;
#ifdef HHG_SCALING_ONLY  // tuning builds (tools/tune_volume.py)
  if (variant != HHG_VAR_SCALING || res || SRC != SRC_SPLIT) return HHG_ERR_ARG;
  if (mirror && HHG_VOLUME_TMA && tma_fits(D))
    return fast ? launch_tma<false, 1>(D, st) : launch_tma<false, 0>(D, st);
  if (mirror && fast) return launch_mirror<SRC, false, 1>(D, st);
  if (fast) return launch_volume<0, SRC, false, true>(D, st);
  return mirror ? launch_mirror<SRC, false>(D, st)
                : launch_volume<0, SRC, false, false>(D, st);
#endif
  switch (variant) {
    case HHG_VAR_SCALING:
      if (SRC == SRC_SPLIT && mirror && HHG_VOLUME_TMA && tma_fits(D)) {
        if (fast) return res ? launch_tma<true, 1>(D, st) : launch_tma<false, 1>(D, st);
        return res ? launch_tma<true, 0>(D, st) : launch_tma<false, 0>(D, st);
      }
      if (mirror && fast) return res ? launch_mirror<SRC, true, 1>(D, st)
                                     : launch_mirror<SRC, false, 1>(D, st);
      if (fast) return res ? launch_volume<0, SRC, true, true>(D, st)
                           : launch_volume<0, SRC, false, true>(D, st);
      if (mirror) return res ? launch_mirror<SRC, true>(D, st)
                             : launch_mirror<SRC, false>(D, st);
      return res ? launch_volume<0, SRC, true, false>(D, st)
                 : launch_volume<0, SRC, false, false>(D, st);
    case HHG_VAR_NODAL:
      if (fast) return res ? launch_volume<1, SRC, true, true>(D, st)
                           : launch_volume<1, SRC, false, true>(D, st);
      return res ? launch_volume<1, SRC, true, false>(D, st)
                 : launch_volume<1, SRC, false, false>(D, st);
    case HHG_VAR_CONST:
      return res ? launch_volume<2, SRC, true, false>(D, st)
                 : launch_volume<2, SRC, false, false>(D, st);
    case HHG_VAR_STORED:
      return res ? launch_volume<3, SRC, true, false>(D, st)
                 : launch_volume<3, SRC, false, false>(D, st);
  }
  return HHG_ERR_ARG;
}

// tiles of the macro elements: 32 i-columns x (W*B) j-rows, k-march up to
// kmax; (j-band, element, i) order as in device.volume_tiles
static std::vector<int4> make_tiles(int n, int ntets) {
  std::vector<int4> tl;
  const int TJ = kW * kB;
  for (int j0 = 1; j0 <= n - 3; j0 += TJ)
    for (int t = 0; t < ntets; ++t)
      for (int i0 = 1; i0 + j0 <= n - 2; i0 += 32)
        tl.push_back(make_int4(t, i0, j0, n - 1 - i0 - j0));
  return tl;
}

// Small host-built tables (tile lists, hyperplane point lists) are uploaded
// once per parameter set and kept for the process lifetime: never freed, so
// kernels queued earlier on any stream can still read them (a multigrid
// cycle alternates levels, so a single-entry cache would rebuild and free
// a table per sweep).
template <class T>
static int upload(const std::vector<T> &v, T **dev) {
  *dev = nullptr;
  if (v.empty()) return HHG_OK;
  if (cudaMalloc(dev, v.size() * sizeof(T)) != cudaSuccess) return HHG_ERR_CUDA;
  return cudaMemcpy(*dev, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice) == cudaSuccess
             ? HHG_OK
             : HHG_ERR_CUDA;
}

// per-element ABI: one macro element, lattice layout (tiles per n)
struct ElemTiles {
  int4 *dev = nullptr;
  int count = 0;
};

// process-lifetime caches are keyed by the current device as well (device
// pointers of one GPU are not valid on another) and guarded by one mutex
// (ctypes releases the GIL around these calls)
static std::mutex g_cache_mu;
static int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

static int elem_tiles(int n, const int4 **tiles, int *count) {
  static std::map<std::pair<int, int>, ElemTiles> cache;
  std::lock_guard<std::mutex> lock(g_cache_mu);
  const auto key = std::make_pair(current_device(), n);
  auto it = cache.find(key);
  if (it == cache.end()) {
    std::vector<int4> tl = make_tiles(n, 1);
    ElemTiles e;
    int rc = upload(tl, &e.dev);
    if (rc) return rc;
    e.count = (int)tl.size();
    it = cache.emplace(key, e).first;
  }
  *tiles = it->second.dev;
  *count = it->second.count;
  return HHG_OK;
}

static VolDesc elem_desc(int64_t n, const double *v, const double *kc,
                         const double *coef, int stride, double *out) {
  VolDesc D{};
  D.n = (int)n;
  D.ntets = 1;
  D.L = tetra(n);
  D.nvol = n >= 4 ? tetra(n - 4) : 0;
  D.kc = kc;
  D.u = v;
  D.out = out;
  D.coef = coef;
  D.coef_stride = stride;
  return D;
}

static bool tables_match(const int64_t *sched, int64_t nsched, const int64_t *sums,
                         const int64_t *tptr, const int64_t *telem) {
  if (nsched != 40) return false;
  for (int r = 0; r < 40; ++r)
    for (int c = 0; c < 3; ++c)
      if (sched[r * 3 + c] != pt_cse(r, c)) return false;
  for (int e = 0; e < 24; ++e)
    if (sums[e] != 31 + e) return false;
  for (int d = 0; d < 15; ++d)
    if (tptr[d] != pt_tptr(d)) return false;
  for (int t = 0; t < 72; ++t)
    if (telem[t] != pt_telem(t)) return false;
  return true;
}

// Volume Gauss-Seidel of all elements: cpt co-resident CTAs per element
// (cooperative launch, grid barrier per hyperplane) when the device can hold
// at least two per element, else one CTA per element (block barrier).
// co-resident CTAs of a kernel on the current device (cached per device)
template <class K>
static int device_capacity(K kern, int threads, std::map<int, int> &cache) {
  std::lock_guard<std::mutex> lock(g_cache_mu);
  const int dev = current_device();
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int sms = 0, per = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, threads, 0);
  const int cap = sms * (per > 0 ? per : 1);
  cache.emplace(dev, cap);
  return cap;
}

#ifndef HHG_GS_CLUSTER
#define HHG_GS_CLUSTER 4         // CTAs per element of the cluster sweeps (0: off)
#endif

#ifndef HHG_GS_CLUSTER_MAX
#define HHG_GS_CLUSTER_MAX 16    // most CTAs per element of the hyperplane-major sweep
#endif

// CTAs per element of the cluster volume sweeps (HHG_GS_CLUSTER_N overrides;
// > 8 needs the non-portable opt-in)
static int gs_cluster() {
  static const int v = [] {
    const char *e = getenv("HHG_GS_CLUSTER_N");
    return e ? atoi(e) : HHG_GS_CLUSTER;
  }();
  return v;
}

template <int VAR>
static int launch_gs_volume(GSDesc G, cudaStream_t st) {
  if (gs_cluster() > 0 && G.n >= 16) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G.ntets * gs_cluster());
    cfg.blockDim = dim3(gs_cluster_threads<VAR>());
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = gs_cluster();
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    G.cpt = gs_cluster();
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaLaunchKernelEx(&cfg, gs_volume_cluster_kernel<VAR>, G);
    if (e != cudaSuccess) {
      fprintf(stderr, "hhg_b200: gs_volume_cluster_kernel: %s\n", cudaGetErrorString(e));
      return HHG_ERR_CUDA;
    }
    return HHG_OK;
  }
  static std::map<int, int> caps;
  const int capacity = device_capacity(gs_volume_kernel<VAR, true>,
                                       gs_volume_threads<VAR, true>(), caps);
  // enough CTAs per element to give each thread about one point per
  // hyperplane, within the co-residency limit; the grid barrier (~2 us per
  // hyperplane) and L1-bypassing loads do not pay for narrow hyperplanes
  // (level 6: one CTA per element with L1-cached loads is faster)
  constexpr int TC = gs_volume_threads<VAR, true>();
  const long long avg = G.nvol / (3LL * G.n - 11);
  const int cpt = G.ntets > 0 ? capacity / G.ntets : 1;
  if (avg < 3LL * TC || cpt < 2) {
    G.cpt = 1;
    gs_volume_kernel<VAR, false><<<G.ntets, gs_volume_threads<VAR, false>(), 0, st>>>(G);
    return check("gs_volume_kernel");
  }
  G.cpt = cpt;
  void *args[] = {(void *)&G};
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaLaunchCooperativeKernel((void *)gs_volume_kernel<VAR, true>,
                                              G.ntets * cpt, TC, args, 0, st);
  if (e != cudaSuccess) {
    fprintf(stderr, "hhg_b200: gs_volume_kernel (cooperative): %s\n", cudaGetErrorString(e));
    return HHG_ERR_CUDA;
  }
  return HHG_OK;
}

extern "C" {

int hhg_apply_scaling_3d(int64_t n, const int64_t *, const double *v, const double *kc,
                         const double *sh, double *out, void *stream) {
  if (n > HHG_MAX_N) return HHG_ERR_ARG;   // 32-bit lattice forms, 10-bit point codes
  if (n < 4) return HHG_OK;
  VolDesc D = elem_desc(n, v, kc, sh, 14, out);
  int rc = elem_tiles((int)n, &D.tiles, &D.ntiles);
  if (rc) return rc;
  return dispatch_volume<SRC_LATTICE>(D, HHG_VAR_SCALING, 0, S(stream));
}

int hhg_apply_nodal_3d(int64_t n, const int64_t *, const double *v, const double *kc,
                       const int64_t *sched, int64_t nsched, const int64_t *sums,
                       const double *fac, const int64_t *tptr, const int64_t *telem,
                       double *out, void *stream) {
  if (n > HHG_MAX_N) return HHG_ERR_ARG;   // 32-bit lattice forms, 10-bit point codes
  if (!tables_match(sched, nsched, sums, tptr, telem)) return HHG_ERR_TABLE;
  if (n < 4) return HHG_OK;
  VolDesc D = elem_desc(n, v, kc, fac, 72, out);
  int rc = elem_tiles((int)n, &D.tiles, &D.ntiles);
  if (rc) return rc;
  return dispatch_volume<SRC_LATTICE>(D, HHG_VAR_NODAL, 0, S(stream));
}

int hhg_apply_const_3d(int64_t n, const int64_t *, const double *v, const double *s,
                       double c0, double *out, void *stream) {
  if (n > HHG_MAX_N) return HHG_ERR_ARG;   // 32-bit lattice forms, 10-bit point codes
  // s: the 14 neighbour weights (device), c0: the diagonal weight (by value),
  // exactly kernels.apply_const_3d(n, base, v, s, c0, out)
  if (n < 4) return HHG_OK;
  VolDesc D = elem_desc(n, v, v, s, 14, out);
  D.c0 = c0;
  int rc = elem_tiles((int)n, &D.tiles, &D.ntiles);
  if (rc) return rc;
  return dispatch_volume<SRC_LATTICE>(D, HHG_VAR_CONST, 0, S(stream));
}

int hhg_apply_stored_3d(int64_t n, const int64_t *, const double *v, const double *w,
                        double *out, void *stream) {
  if (n > HHG_MAX_N) return HHG_ERR_ARG;   // 32-bit lattice forms, 10-bit point codes
  if (n < 4) return HHG_OK;
  VolDesc D = elem_desc(n, v, v, nullptr, 0, out);
  D.w = w;
  int rc = elem_tiles((int)n, &D.tiles, &D.ntiles);
  if (rc) return rc;
  return dispatch_volume<SRC_LATTICE>(D, HHG_VAR_STORED, 0, S(stream));
}

// interior points of each hyperplane h = i + 2j + 3k (host-built once per n)
struct Hyperplanes {
  int *ptr = nullptr, *code = nullptr;
  // the whole (n+1)-lattice (interior + boundary points) in hyperplane
  // order - h = i + 2j + 3k (0 .. 3n), then k, then j: position of (i, j, k)
  // = xstart[h (n + 1) + k] + j; xcode = the point codes in that order
  int *xstart = nullptr, *xcode = nullptr;
  // the boundary (ghost) points: code and position in that order
  int *bcode = nullptr, *bpos = nullptr;
  int nb = 0;
  // interior points in volume-block (k, j, i) order (the scatter back to u)
  int *icode = nullptr;
};

static int hyperplanes(int n, const int **ptr, const int **code, const int **xstart = nullptr,
                       const int **xcode = nullptr, const int **bcode = nullptr,
                       const int **bpos = nullptr, int *nb = nullptr,
                       const int **icode = nullptr) {
  static std::map<std::pair<int, int>, Hyperplanes> cache;
  std::lock_guard<std::mutex> lock(g_cache_mu);
  const auto key = std::make_pair(current_device(), n);
  auto it = cache.find(key);
  if (it == cache.end()) {
    const int hmin = 6, hmax = 3 * n - 6;
    std::vector<int> p(std::max(hmax - hmin + 2, 1), 0), c;
    for (int h = hmin; h <= hmax; ++h) {
      p[h - hmin] = (int)c.size();
      for (int k = 1; k <= n - 3; ++k)
        for (int j = 1; j <= n - 2 - k; ++j) {
          const int i = h - 2 * j - 3 * k;
          if (i >= 1 && i + j + k <= n - 1) c.push_back(i | (j << 10) | (k << 20));
        }
    }
    if (hmax >= hmin) p[hmax - hmin + 1] = (int)c.size();
    std::vector<int> ic;
    for (int k = 1; k <= n - 3; ++k)
      for (int j = 1; j <= n - 2 - k; ++j)
        for (int i = 1; i <= n - 1 - j - k; ++i) ic.push_back(i | (j << 10) | (k << 20));
    std::vector<int> xs((3 * n + 1) * (n + 1), 0), xc, bc, bp;
    for (int h = 0; h <= 3 * n; ++h)
      for (int k = 0; k <= n; ++k) {
        int jmin = -1;
        for (int j = 0; j <= n - k; ++j) {
          const int i = h - 2 * j - 3 * k;
          if (i >= 0 && i + j + k <= n) {
            if (jmin < 0) {
              jmin = j;
              xs[h * (n + 1) + k] = (int)xc.size() - j;
            }
            if (!(i >= 1 && j >= 1 && k >= 1 && i + j + k <= n - 1)) {
              bc.push_back(i | (j << 10) | (k << 20));
              bp.push_back((int)xc.size());
            }
            xc.push_back(i | (j << 10) | (k << 20));
          }
        }
      }
    Hyperplanes hp;
    int rc = upload(p, &hp.ptr);
    if (!rc) rc = upload(c, &hp.code);
    if (!rc) rc = upload(xs, &hp.xstart);
    if (!rc) rc = upload(xc, &hp.xcode);
    if (!rc) rc = upload(bc, &hp.bcode);
    if (!rc) rc = upload(bp, &hp.bpos);
    if (!rc) rc = upload(ic, &hp.icode);
    if (rc) return rc;
    hp.nb = (int)bc.size();
    it = cache.emplace(key, hp).first;
  }
  *ptr = it->second.ptr;
  *code = it->second.code;
  if (xstart) *xstart = it->second.xstart;
  if (xcode) *xcode = it->second.xcode;
  if (bcode) *bcode = it->second.bcode;
  if (bpos) *bpos = it->second.bpos;
  if (nb) *nb = it->second.nb;
  if (icode) *icode = it->second.icode;
  return HHG_OK;
}

static int gs_elem(int var, int64_t n, double *u, const double *fv, const double *kc,
                   const double *coef, int stride, double omega, cudaStream_t st) {
  if (n < 4) return HHG_OK;
  GSDesc G{};
  G.n = (int)n;
  G.ntets = 1;
  G.L = tetra(n);
  G.nvol = tetra(n - 4);
  G.kc = kc;
  G.u = u;
  G.f = fv;
  G.coef = coef;
  G.coef_stride = stride;
  G.omega = omega;
  G.lattice = 1;
  int rc = hyperplanes((int)n, &G.hp_ptr, &G.hp_code);
  if (rc) return rc;
  G.cpt = 1;
  if (var == 0) gs_volume_kernel<0, false><<<1, gs_volume_threads<0, false>(), 0, st>>>(G);
  else gs_volume_kernel<1, false><<<1, gs_volume_threads<1, false>(), 0, st>>>(G);
  return check("gs_volume_kernel");
}

int hhg_csr_gs(int64_t nrows_list, const int64_t *rows, const int64_t *indptr,
               const int64_t *indices, const double *data, const double *diag, double *u,
               const double *f, double omega, void *stream) {
  if (nrows_list <= 0) return HHG_OK;
  if (!rows || !indptr || !indices || !data || !diag || !u || !f) return HHG_ERR_ARG;
  csr_gs_kernel<<<1, 32, 0, S(stream)>>>(
      nrows_list, reinterpret_cast<const long long *>(rows),
      reinterpret_cast<const long long *>(indptr), reinterpret_cast<const long long *>(indices),
      data, diag, u, f, omega);
  return check("csr_gs_kernel");
}

// 2-D scaling with the MA2 gray-edge selector (hhg_ma2.cuh); gray: 6 host
// flags (the reference's g), base: the canonical row table (or NULL)
static unsigned gray_bits(const uint8_t *g) {
  unsigned b = 0;
  for (int d = 0; d < 6; ++d)
    if (g && g[d]) b |= 1u << d;
  return b;
}

int hhg_apply_scaling_2d(int64_t n, const int64_t *, const double *v, const double *kc,
                         const double *kg, const uint8_t *g, const double *sh, double *out,
                         void *stream) {
  if (n > 1 << 15) return HHG_ERR_ARG;
  if (n < 3) return HHG_OK;
  const dim3 grid((unsigned)((n - 3 + 127) / 128), (unsigned)(n - 2));
  apply_scaling_2d_kernel<<<grid, 128, 0, S(stream)>>>((int)n, v, kc, kg, gray_bits(g), sh, out);
  return check("apply_scaling_2d_kernel");
}

int hhg_gs_scaling_2d(int64_t n, const int64_t *, double *u, const double *fv, const double *kc,
                      const double *kg, const uint8_t *g, const double *sh, double omega,
                      void *stream) {
  if (n > 1 << 15) return HHG_ERR_ARG;
  if (n < 3) return HHG_OK;
  gs_scaling_2d_kernel<<<1, 256, 0, S(stream)>>>((int)n, u, fv, kc, kg, gray_bits(g), sh,
                                                 omega);
  return check("gs_scaling_2d_kernel");
}

int hhg_gs_scaling_3d(int64_t n, const int64_t *, double *u, const double *fv,
                      const double *kc, const double *sh, double omega, void *stream) {
  if (n > HHG_MAX_N) return HHG_ERR_ARG;   // 32-bit lattice forms, 10-bit point codes
  return gs_elem(0, n, u, fv, kc, sh, 14, omega, S(stream));
}

int hhg_gs_nodal_3d(int64_t n, const int64_t *, double *u, const double *fv,
                    const double *kc, const int64_t *sched, int64_t nsched,
                    const int64_t *sums, const double *fac, const int64_t *tptr,
                    const int64_t *telem, double omega, void *stream) {
  if (n > HHG_MAX_N) return HHG_ERR_ARG;   // 32-bit lattice forms, 10-bit point codes
  if (!tables_match(sched, nsched, sums, tptr, telem)) return HHG_ERR_TABLE;
  return gs_elem(1, n, u, fv, kc, fac, 72, omega, S(stream));
}

// ---------------------------------------------------------------------------
// batched operator entry points
// ---------------------------------------------------------------------------
static VolDesc grid_desc(const hhg_grid *g) {
  VolDesc D{};
  D.n = g->n;
  D.ntets = g->ntets;
  D.L = g->lat_size;
  D.nvol = g->nvol;
  D.S = g->shell_size;
  D.vol_start = reinterpret_cast<const long long *>(g->vol_start);
  D.srow = g->srow;
  D.ghost = g->ghost;
  D.kc = g->kc;
  D.tiles = reinterpret_cast<const int4 *>(g->tiles);
  D.ntiles = g->ntiles;
  D.mtiles = reinterpret_cast<const int4 *>(g->mtiles);
  D.nmtiles = g->nmtiles;
  D.n_nodes = g->n_nodes;
  return D;
}

int hhg_dump_stencils(const hhg_grid *g, int variant, const double *coef, double *w,
                      void *stream) {
  if (g->n > HHG_MAX_N) return HHG_ERR_ARG;
  if (g->n < 4 || g->ntets == 0) return HHG_OK;
  if (variant != HHG_VAR_SCALING && variant != HHG_VAR_NODAL) return HHG_ERR_ARG;
  const dim3 grid(g->n - 3, g->ntets);
  if (variant == HHG_VAR_NODAL)
    dump_stencils_kernel<1><<<grid, 128, 0, S(stream)>>>(g->n, g->lat_size, g->nvol, g->kc,
                                                         coef, 72, w);
  else
    dump_stencils_kernel<0><<<grid, 128, 0, S(stream)>>>(g->n, g->lat_size, g->nvol, g->kc,
                                                         coef, 14, w);
  return check("dump_stencils_kernel");
}

int hhg_ghost_update(const hhg_grid *g, const double *u, void *stream) {
  if (g->n > HHG_MAX_N) return HHG_ERR_ARG;   // 32-bit lattice forms, 10-bit point codes
  const long long total = (long long)g->ntets * g->shell_size;
  if (total == 0) return HHG_OK;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  ghost_kernel<<<blocks, 256, 0, S(stream)>>>(
      total, reinterpret_cast<const long long *>(g->shell_gid), u, g->ghost);
  return check("ghost_kernel");
}

int hhg_volume_apply(const hhg_grid *g, int variant, int flags, const double *coef,
                     const double *w, const double *u, const double *f, double *out,
                     void *stream) {
  if (g->n > HHG_MAX_N) return HHG_ERR_ARG;   // 32-bit lattice forms, 10-bit point codes
  if (g->n < 4 || g->ntiles == 0) return HHG_OK;
  VolDesc D = grid_desc(g);
  D.u = u;
  D.f = f;
  D.out = out;
  D.coef = coef;
  D.coef_stride = variant == HHG_VAR_NODAL ? 72 : (variant == HHG_VAR_CONST ? 15 : 14);
  D.w = w;
  return dispatch_volume<SRC_SPLIT>(D, variant, flags, S(stream));
}

static SurfDesc surf_desc(const hhg_grid *g, const hhg_surface *s) {
  SurfDesc D{};
  D.n = g->n;
  D.L = g->lat_size;
  D.S = g->shell_size;
  D.nrows = s->nrows;
  D.vol_start = reinterpret_cast<const long long *>(g->vol_start);
  D.srow = g->srow;
  D.ghost = g->ghost;
  D.kc = g->kc;
  D.rows = reinterpret_cast<const long long *>(s->rows);
  D.row_nodal = s->row_nodal;
  D.inc_ptr = s->inc_ptr;
  D.inc_tet = s->inc_tet;
  D.inc_code = s->inc_code;
  D.inc_cls = s->inc_cls;
  D.psh = s->psh;
  D.pfac = s->pfac;
  D.ninc = s->ninc;
  D.p_tet = s->p_tet;
  D.p_code = s->p_code;
  D.p_cls = s->p_cls;
  D.p_nodal = s->p_nodal;
  D.row_inc = s->row_inc;
  D.partial = s->partial;
  return D;
}

int hhg_surface_apply(const hhg_grid *g, const hhg_surface *s, int, int flags,
                      const double *u, const double *f, double *out, void *stream) {
  if (g->n > HHG_MAX_N) return HHG_ERR_ARG;   // 32-bit lattice forms, 10-bit point codes
  const bool res = flags & HHG_FLAG_RESIDUAL;
  SurfDesc D = surf_desc(g, s);
  D.u = u;
  D.f = f;
  D.out = out;
  if (s->nrows > 0) {
    const bool mixed = s->pfac != nullptr;
    const int pblocks = (int)((s->ninc + 127) / 128);
    if (mixed) surface_partial_kernel<true><<<pblocks, 128, 0, S(stream)>>>(D);
    else surface_partial_kernel<false><<<pblocks, 128, 0, S(stream)>>>(D);
    int rc = check("surface_partial_kernel");
    if (rc) return rc;
    const int rblocks = (int)((s->nrows + 255) / 256);
    if (res) surface_reduce_kernel<true><<<rblocks, 256, 0, S(stream)>>>(D);
    else surface_reduce_kernel<false><<<rblocks, 256, 0, S(stream)>>>(D);
    rc = check("surface_reduce_kernel");
    if (rc) return rc;
  }
  if (s->ndir > 0) {
    const int blocks = (int)((s->ndir + 255) / 256);
    const long long *ids = reinterpret_cast<const long long *>(s->dir_ids);
    if (res) dirichlet_kernel<true><<<blocks, 256, 0, S(stream)>>>(s->ndir, ids, u, out);
    else dirichlet_kernel<false><<<blocks, 256, 0, S(stream)>>>(s->ndir, ids, u, out);
    return check("dirichlet_kernel");
  }
  return HHG_OK;
}

// smoother: surface rows level by level, then refresh the ghost layer, then
// the volume wavefronts of all macro elements (one CTA each)
int hhg_smooth_surface_level(const hhg_grid *g, const hhg_surface *s,
                             const int64_t *level_rows, int64_t count, double omega,
                             double *u, const double *f, void *stream) {
  if (g->n > HHG_MAX_N) return HHG_ERR_ARG;   // 32-bit lattice forms, 10-bit point codes
  if (count <= 0) return HHG_OK;
  SurfGSDesc G{};
  G.s = surf_desc(g, s);
  G.s.u = u;
  G.s.f = f;
  G.shell_gid = reinterpret_cast<const long long *>(g->shell_gid);
  G.level_rows = reinterpret_cast<const long long *>(level_rows);
  G.count = count;
  G.omega = omega;
  gs_surface_kernel<<<(int)((count + 127) / 128), 128, 0, S(stream)>>>(G);
  return check("gs_surface_kernel");
}

// surface rows of the smoother, precomputed once: weights + diagonals
int hhg_smooth_surface_prepare(const hhg_grid *g, const hhg_surface *s,
                               const hhg_surface_gs *gs, void *stream) {
  if (g->n > HHG_MAX_N) return HHG_ERR_ARG;   // 32-bit lattice forms, 10-bit point codes
  if (s->nrows <= 0) return HHG_OK;
  SurfGSDesc G{};
  G.s = surf_desc(g, s);
  G.shell_gid = reinterpret_cast<const long long *>(g->shell_gid);
  G.ent_ptr = reinterpret_cast<const long long *>(gs->ent_ptr);
  G.ent_col = gs->ent_col;
  G.ent_val = gs->ent_val;
  G.row_diag = gs->row_diag;
  gs_surface_fill_kernel<<<(int)((s->nrows + 127) / 128), 128, 0, S(stream)>>>(G);
  return check("gs_surface_fill_kernel");
}

// surface rows of apply / residual from the precomputed rows (+ Dirichlet)
static int surface_csr(const hhg_grid *g, const hhg_surface *s, const hhg_surface_gs *gs,
                       int flags, const double *u, const double *f, double *out,
                       const SurfPush &push, void *stream);

int hhg_surface_apply_csr(const hhg_grid *g, const hhg_surface *s, const hhg_surface_gs *gs,
                          int flags, const double *u, const double *f, double *out,
                          void *stream) {
  return surface_csr(g, s, gs, flags, u, f, out, SurfPush{}, stream);
}

int hhg_surface_apply_csr_push(const hhg_grid *g, const hhg_surface *s,
                               const hhg_surface_gs *gs, const double *u, double *out,
                               const int32_t *push_slot, double *dst0, double *dst1,
                               int64_t split, void *stream) {
  if (!push_slot) return HHG_ERR_ARG;
  SurfPush p{push_slot, dst0, dst1, (long long)split};
  return surface_csr(g, s, gs, 0, u, nullptr, out, p, stream);
}

int hhg_p2p_signal(unsigned long long *remote_flag, void *stream) {
  if (!remote_flag) return HHG_ERR_ARG;
  p2p_signal_kernel<<<1, 1, 0, S(stream)>>>(remote_flag);
  return check("p2p_signal_kernel");
}

int hhg_p2p_pull(double *out, const int64_t *ids, int64_t count, const double *recv,
                 const unsigned long long *flag, unsigned long long target, int recv_first,
                 int *err, void *stream) {
  if (count <= 0) return HHG_OK;
  if (!out || !ids || !recv || !flag || !err) return HHG_ERR_ARG;
  p2p_wait_kernel<<<1, 32, 0, S(stream)>>>(flag, target, err);
  int rc = check("p2p_wait_kernel");
  if (rc) return rc;
  const int blocks = (int)std::min<int64_t>((count + 255) / 256, 64);
  p2p_add_kernel<<<blocks, 256, 0, S(stream)>>>(out, reinterpret_cast<const long long *>(ids),
                                                count, recv, recv_first, err);
  return check("p2p_add_kernel");
}

int hhg_device_alloc(int64_t bytes, void **ptr) {
  if (bytes <= 0 || !ptr) return HHG_ERR_ARG;
  if (cudaMalloc(ptr, (size_t)bytes) != cudaSuccess) return HHG_ERR_CUDA;
  return cudaMemset(*ptr, 0, (size_t)bytes) == cudaSuccess ? HHG_OK : HHG_ERR_CUDA;
}

int hhg_device_free(void *ptr) { return cudaFree(ptr) == cudaSuccess ? HHG_OK : HHG_ERR_CUDA; }

int hhg_ipc_get_handle(const void *ptr, void *handle) {
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, const_cast<void *>(ptr)) != cudaSuccess) return HHG_ERR_CUDA;
  memcpy(handle, &h, sizeof h);
  return HHG_OK;
}

int hhg_ipc_open_handle(const void *handle, void **ptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof h);
  return cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess
             ? HHG_OK
             : HHG_ERR_CUDA;
}

int hhg_ipc_close_handle(void *ptr) {
  return cudaIpcCloseMemHandle(ptr) == cudaSuccess ? HHG_OK : HHG_ERR_CUDA;
}

}  // extern "C"

static int surface_csr(const hhg_grid *g, const hhg_surface *s, const hhg_surface_gs *gs,
                       int flags, const double *u, const double *f, double *out,
                       const SurfPush &push, void *stream) {
  if (g->n > HHG_MAX_N) return HHG_ERR_ARG;   // 32-bit lattice forms, 10-bit point codes
  const bool res = flags & HHG_FLAG_RESIDUAL;
  SurfGSDesc G{};
  G.s = surf_desc(g, s);
  G.s.u = u;
  G.s.f = f;
  G.ent_ptr = reinterpret_cast<const long long *>(gs->ent_ptr);
  G.ent_col = gs->ent_col;
  G.ent_val = gs->ent_val;
  G.shell_gid = reinterpret_cast<const long long *>(g->shell_gid);
#ifndef HHG_FUSE_DIRICHLET
#define HHG_FUSE_DIRICHLET 0
#endif
  const long long *ids = reinterpret_cast<const long long *>(s->dir_ids);
  const long long nd = HHG_FUSE_DIRICHLET ? s->ndir : 0;
  const bool faced = s->nfaces > 0 && s->nface_tiles > 0;
  if (faced) {   // face rows tiled per macro face, edge / vertex rows below
    const int nb = (int)s->nface_tiles, nt = FACE_TA * FACE_TB;
    const bool mixed = s->pfac != nullptr;
    if (!s->face_k || !s->face_g) return HHG_ERR_ARG;
    if (res) {
      if (mixed) surface_face_kernel<true, true><<<nb, nt, 0, S(stream)>>>(G, *s, out, push);
      else surface_face_kernel<true, false><<<nb, nt, 0, S(stream)>>>(G, *s, out, push);
    } else {
      if (mixed) surface_face_kernel<false, true><<<nb, nt, 0, S(stream)>>>(G, *s, out, push);
      else surface_face_kernel<false, false><<<nb, nt, 0, S(stream)>>>(G, *s, out, push);
    }
    int rc = check("surface_face_kernel");
    if (rc) return rc;
  }
  const int *sub = faced ? s->sub_rows : nullptr;
  const long long nsub = faced ? s->nsub : 0;
  const long long total = (faced ? nsub : s->nrows) + nd;   // rows (then Dirichlet rows)
  if (total > 0) {
    const int blocks = (int)((total + 127) / 128);
    if (res) surface_csr_kernel<true><<<blocks, 128, 0, S(stream)>>>(G, out, nd, ids, SurfPush{}, sub, nsub);
    else surface_csr_kernel<false><<<blocks, 128, 0, S(stream)>>>(G, out, nd, ids, push, sub, nsub);
    int rc = check("surface_csr_kernel");
    if (rc) return rc;
  }
  if (!HHG_FUSE_DIRICHLET && s->ndir > 0) {
    const int blocks = (int)((s->ndir + 255) / 256);
    if (res) dirichlet_kernel<true><<<blocks, 256, 0, S(stream)>>>(s->ndir, ids, u, out);
    else dirichlet_kernel<false><<<blocks, 256, 0, S(stream)>>>(s->ndir, ids, u, out);
    return check("dirichlet_kernel");
  }
  return HHG_OK;
}

extern "C" {

// sharded surface sweep pieces (rows of one level of the global schedule)
static SurfGSDesc surf_gs_desc(const hhg_grid *g, const hhg_surface *s, const hhg_surface_gs *gs,
                               double omega, double *u, const double *f) {
  SurfGSDesc G{};
  G.s = surf_desc(g, s);
  G.s.u = u;
  G.s.f = f;
  G.shell_gid = reinterpret_cast<const long long *>(g->shell_gid);
  G.omega = omega;
  G.ent_ptr = reinterpret_cast<const long long *>(gs->ent_ptr);
  G.ent_col = gs->ent_col;
  G.ent_val = gs->ent_val;
  G.row_diag = gs->row_diag;
  G.level_rows = reinterpret_cast<const long long *>(gs->level_rows);
  G.nslots = gs->nslots;
  G.slot_gid = reinterpret_cast<const long long *>(gs->slot_gid);
  G.slot_cnt = gs->slot_cnt;
  G.slot_col = gs->slot_col;
  G.slot_diag = gs->slot_diag;
  G.slot_val = gs->slot_val;
  G.slot_dyn = gs->slot_dyn;
  return G;
}

int hhg_smooth_surface_slots(const hhg_grid *g, const hhg_surface *s, const hhg_surface_gs *gs,
                             const int32_t *gid_level, int64_t nlv, void *stream) {
  if (gs->nslots <= 0) return HHG_OK;
  if (!gs->slot_gid || !gs->slot_cnt || !gs->slot_diag || !gs->slot_col || !gs->slot_val ||
      !gs->slot_dyn || !gs->level_rows || !gid_level)
    return HHG_ERR_ARG;
  SurfGSDesc G = surf_gs_desc(g, s, gs, 1.0, nullptr, nullptr);
  surface_slots_kernel<<<(int)((gs->nslots + 255) / 256), 256, 0, S(stream)>>>(
      G, reinterpret_cast<long long *>(gs->slot_gid), gs->slot_cnt, gs->slot_diag, gs->slot_col,
      gs->slot_val, gs->slot_dyn, gid_level, nlv);
  return check("surface_slots_kernel");
}

int hhg_smooth_surface_rows(const hhg_grid *g, const hhg_surface *s, const hhg_surface_gs *gs,
                            const int64_t *rows, int64_t count, double omega, double *u,
                            const double *f, void *stream) {
  if (count <= 0) return HHG_OK;
  SurfGSDesc G = surf_gs_desc(g, s, gs, omega, u, f);
  gs_surface_rows_kernel<<<(int)((count + 127) / 128), 128, 0, S(stream)>>>(
      G, reinterpret_cast<const long long *>(rows), count);
  return check("gs_surface_rows_kernel");
}

int hhg_smooth_surface_partial(const hhg_grid *g, const hhg_surface *s,
                               const hhg_surface_gs *gs, const int64_t *rows, int64_t count,
                               const double *u, double *acc, double *diag, void *stream) {
  if (count <= 0) return HHG_OK;
  SurfGSDesc G = surf_gs_desc(g, s, gs, 1.0, const_cast<double *>(u), nullptr);
  gs_surface_partial_kernel<<<(int)((count + 127) / 128), 128, 0, S(stream)>>>(
      G, reinterpret_cast<const long long *>(rows), count, acc, diag);
  return check("gs_surface_partial_kernel");
}

int hhg_smooth_surface_finish(const hhg_grid *g, const hhg_surface *s,
                              const hhg_surface_gs *gs, const int64_t *rows, int64_t count,
                              const double *acc, const double *diag, double omega, double *u,
                              const double *f, void *stream) {
  if (count <= 0) return HHG_OK;
  SurfGSDesc G = surf_gs_desc(g, s, gs, omega, u, f);
  gs_surface_finish_kernel<<<(int)((count + 127) / 128), 128, 0, S(stream)>>>(
      G, reinterpret_cast<const long long *>(rows), count, acc, diag);
  return check("gs_surface_finish_kernel");
}

// every level of the surface sweep in one cooperative launch; the grid is
// sized to the mean level width (a narrow sweep syncs few blocks)
int hhg_smooth_surface_all(const hhg_grid *g, const hhg_surface *s, const hhg_surface_gs *gs,
                           double omega, double *u, const double *f, void *stream) {
  if (g->n > HHG_MAX_N) return HHG_ERR_ARG;   // 32-bit lattice forms, 10-bit point codes
  if (gs->nlev <= 0) return HHG_OK;
  SurfGSDesc G = surf_gs_desc(g, s, gs, omega, u, f);
  const long long *lp = reinterpret_cast<const long long *>(gs->level_ptr);
  int nl = (int)gs->nlev;
  // narrow sweeps (mean level width <= 512 rows: level 6 grids): one
  // 16-CTA thread-block cluster walks the levels, a cluster barrier between
  // them; wider sweeps need the memory parallelism of many SMs: a
  // cooperative grid with a split software barrier.  Both from the
  // level-ordered slots, prefetching each thread's next row across the
  // barrier.  HHG_SURF_CLUSTER overrides: CTAs per cluster (> 8 needs the
  // non-portable opt-in), 0 = grid; HHG_SURF_LEGACY=1: the round-1 grid
  // kernel (cooperative groups grid.sync, no slots).
  static const int env_cl = [] {
    const char *e = getenv("HHG_SURF_CLUSTER");
    return e ? atoi(e) : -1;
  }();
  static const bool legacy = [] {
    const char *e = getenv("HHG_SURF_LEGACY");
    return e && atoi(e) != 0;
  }();
  const long long mean_width = (s->nrows + gs->nlev - 1) / gs->nlev;
  const int ncl = env_cl >= 0 ? env_cl : (mean_width <= 512 ? 16 : 0);   // -1: auto
  const bool slots = gs->slot_gid && gs->slot_dyn && gs->sweep_bar && gs->nslots == s->nrows &&
                     !legacy;
  if (slots && ncl > 0) {
    if (ncl > 8)
      cudaFuncSetAttribute(gs_surface_slots_kernel<false>,
                           cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ncl);
    cfg.blockDim = dim3(HHG_SURF_CT);
    cfg.stream = S(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = ncl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    unsigned *nobar = nullptr;
    cudaError_t e = cudaLaunchKernelEx(&cfg, gs_surface_slots_kernel<false>, G, lp, nl, nobar);
    if (e != cudaSuccess) {
      fprintf(stderr, "hhg_b200: gs_surface_slots_kernel: %s\n", cudaGetErrorString(e));
      return HHG_ERR_CUDA;
    }
    return HHG_OK;
  }
  if (slots) {
    static std::map<int, int> gcaps;
    const int cap = device_capacity(gs_surface_slots_kernel<true>, HHG_SURF_GRID_CT, gcaps);
    int blocks = (int)std::min<long long>((mean_width + HHG_SURF_GRID_RPB - 1) / HHG_SURF_GRID_RPB,
                                          cap);
    if (blocks < 8) blocks = std::min(8, cap);
    unsigned *bar = gs->sweep_bar;
    cudaError_t e = cudaMemsetAsync(bar, 0, sizeof(unsigned), S(stream));
    if (e == cudaSuccess) {
      void *args[] = {(void *)&G, (void *)&lp, (void *)&nl, (void *)&bar};
      g_launches.fetch_add(1, std::memory_order_relaxed);
      e = cudaLaunchCooperativeKernel((void *)gs_surface_slots_kernel<true>, blocks,
                                      HHG_SURF_GRID_CT, args, 0, S(stream));
    }
    if (e != cudaSuccess) {
      fprintf(stderr, "hhg_b200: gs_surface_slots_kernel<grid>: %s\n", cudaGetErrorString(e));
      return HHG_ERR_CUDA;
    }
    return HHG_OK;
  }
  static std::map<int, int> caps;
  const int max_blocks = device_capacity(gs_surface_all_kernel, 64, caps);
  // spread each level over many SMs (a single SM's outstanding-miss limit
  // bounds a level to ~15 us); ~8 rows per 64-thread block
  int blocks = (int)((mean_width + 7) / 8);
  if (blocks < 8) blocks = 8;
  if (blocks > max_blocks) blocks = max_blocks;
  void *args[] = {(void *)&G, (void *)&lp, (void *)&nl};
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaLaunchCooperativeKernel((void *)gs_surface_all_kernel, blocks, 64, args,
                                              0, S(stream));
  if (e != cudaSuccess) {
    fprintf(stderr, "hhg_b200: gs_surface_all_kernel: %s\n", cudaGetErrorString(e));
    return HHG_ERR_CUDA;
  }
  return HHG_OK;
}

int hhg_smooth_volume(const hhg_grid *g, int variant, const double *coef, double omega,
                      double *u, const double *f, void *stream) {
  if (g->n > HHG_MAX_N) return HHG_ERR_ARG;   // 32-bit lattice forms, 10-bit point codes
  if (g->n < 4) return HHG_OK;
  GSDesc G{};
  G.n = g->n;
  G.ntets = g->ntets;
  G.L = g->lat_size;
  G.S = g->shell_size;
  G.nvol = g->nvol;
  G.vol_start = reinterpret_cast<const long long *>(g->vol_start);
  G.srow = g->srow;
  G.ghost = g->ghost;
  G.kc = g->kc;
  G.u = u;
  G.f = f;
  G.coef = coef;
  G.coef_stride = variant == HHG_VAR_NODAL ? 72 : 14;
  G.omega = omega;
  G.lattice = 0;
  int rc = hyperplanes(g->n, &G.hp_ptr, &G.hp_code);
  if (rc) return rc;
  return variant == HHG_VAR_NODAL ? launch_gs_volume<1>(G, S(stream))
                                  : launch_gs_volume<0>(G, S(stream));
}

// skewed (hyperplane-major) volume sweep: u and f gathered into the
// hyperplane order, the sweep, u scattered back (hhg_smooth.cuh)
static GSDesc gs_grid_desc(const hhg_grid *g, int variant, const double *coef, double omega,
                           double *u, const double *f) {
  GSDesc G{};
  G.n = g->n;
  G.ntets = g->ntets;
  G.L = g->lat_size;
  G.S = g->shell_size;
  G.nvol = g->nvol;
  G.vol_start = reinterpret_cast<const long long *>(g->vol_start);
  G.srow = g->srow;
  G.ghost = g->ghost;
  G.kc = g->kc;
  G.u = u;
  G.f = f;
  G.coef = coef;
  G.coef_stride = variant == HHG_VAR_NODAL ? 72 : 14;
  G.omega = omega;
  G.lattice = 0;
  return G;
}

int hhg_skew_coefficient(const hhg_grid *g, double *ks, void *stream) {
  if (g->n > HHG_MAX_N) return HHG_ERR_ARG;
  if (g->n < 4 || g->nvol == 0) return HHG_OK;
  GSDesc G = gs_grid_desc(g, HHG_VAR_SCALING, nullptr, 1.0, nullptr, nullptr);
  const int *xstart = nullptr, *xcode = nullptr;
  int rc = hyperplanes(g->n, &G.hp_ptr, &G.hp_code, &xstart, &xcode);
  if (rc) return rc;
  skew_move_kernel<2><<<dim3((int)((G.L + 255) / 256), g->ntets), 256, 0, S(stream)>>>(
      G, xcode, nullptr, ks);
  return check("skew_move_kernel");
}

int hhg_smooth_volume_skew(const hhg_grid *g, int variant, const double *coef, double omega,
                           double *u, const double *f, double *us, double *fs,
                           const double *ks, int flags, void *stream) {
  if (g->n > HHG_MAX_N) return HHG_ERR_ARG;
  if (g->n < 4 || g->nvol == 0) return HHG_OK;
  if (!us || !fs || !ks) return HHG_ERR_ARG;
  GSDesc G = gs_grid_desc(g, variant, coef, omega, u, f);
  const int *xstart = nullptr, *xcode = nullptr, *bcode = nullptr, *bpos = nullptr;
  const int *icode = nullptr;
  int nb = 0;
  int rc = hyperplanes(g->n, &G.hp_ptr, &G.hp_code, &xstart, &xcode, &bcode, &bpos, &nb, &icode);
  if (rc) return rc;
  const dim3 mx((int)((G.L + 255) / 256), g->ntets);
  if (flags & HHG_SKEW_U_CURRENT) {     // interior of us current: ghost values only
    skew_boundary_kernel<<<dim3((nb + 255) / 256, g->ntets), 256, 0, S(stream)>>>(
        G, bcode, bpos, nb, us);
    if ((rc = check("skew_boundary_kernel"))) return rc;
  } else {
    skew_move_kernel<0><<<mx, 256, 0, S(stream)>>>(G, xcode, u, us);
    if ((rc = check("skew_move_kernel"))) return rc;
  }
  if (!(flags & HHG_SKEW_F_CURRENT)) {
    skew_f_kernel<<<dim3((int)((g->nvol + 255) / 256), g->ntets), 256, 0, S(stream)>>>(G, f, fs);
    if ((rc = check("skew_f_kernel"))) return rc;
  }
  // CTAs per element: the most (<= 16) with which every element's cluster is
  // co-resident in one wave (the sweep is latency-bound: more threads per
  // hyperplane help, a second wave of elements does not); at least 4.
  // HHG_GS_CLUSTER_N fixes it.
  const bool nodal = variant == HHG_VAR_NODAL;
  const void *kfn = nodal ? (const void *)gs_volume_skew_kernel<1>
                          : (const void *)gs_volume_skew_kernel<0>;
  cudaLaunchConfig_t cfg = {};
  cfg.stream = S(stream);
  cfg.blockDim = dim3(nodal ? gs_cluster_threads<1>() : gs_cluster_threads<0>());
  cfg.dynamicSmemBytes = 8 * (G.n + 1) * sizeof(int);   // start-table ring
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int cl = gs_cluster();
  if (!getenv("HHG_GS_CLUSTER_N")) {
    static std::map<std::tuple<int, int, int>, int> pick;
    std::lock_guard<std::mutex> lock(g_cache_mu);
    const auto key = std::make_tuple(current_device(), (int)nodal, G.ntets);
    auto it = pick.find(key);
    if (it == pick.end()) {
      int best = 4;
      cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      for (int c = HHG_GS_CLUSTER_MAX; c > 4; --c) {
        cfg.gridDim = dim3(G.ntets * c);
        attr[0].val.clusterDim.x = c;
        int fit = 0;
        if (cudaOccupancyMaxActiveClusters(&fit, kfn, &cfg) == cudaSuccess && fit >= G.ntets) {
          best = c;
          break;
        }
        cudaGetLastError();
      }
      it = pick.emplace(key, best).first;
    }
    cl = it->second;
  }
  cfg.gridDim = dim3(G.ntets * cl);
  attr[0].val.clusterDim.x = cl;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e;
  if (nodal)
    e = cudaLaunchKernelEx(&cfg, gs_volume_skew_kernel<1>, G, us, (const double *)fs, ks, xstart);
  else
    e = cudaLaunchKernelEx(&cfg, gs_volume_skew_kernel<0>, G, us, (const double *)fs, ks, xstart);
  if (e != cudaSuccess) {
    fprintf(stderr, "hhg_b200: gs_volume_skew_kernel: %s\n", cudaGetErrorString(e));
    return HHG_ERR_CUDA;
  }
  if (HHG_SKEW_SCATTER_LAT)       // volume-block order: full-sector writes into u
    skew_scatter_kernel<<<dim3((int)((g->nvol + 255) / 256), g->ntets), 256, 0, S(stream)>>>(
        G, icode, xstart, us, u);
  else
    skew_move_kernel<1><<<mx, 256, 0, S(stream)>>>(G, xcode, us, u);
  return check("skew_move_kernel");
}

// ---------------------------------------------------------------------------
// tensor-coefficient operators (M = 6 components, hhg_tensor.cuh)
// ---------------------------------------------------------------------------
}  // extern "C"

template <bool NODAL, bool AOS>
static int ten_smem_ok() {
  const int smem = (int)ten_smem<NODAL>(ten_threads<NODAL>());
  if (smem_optin((const void *)tensor_volume_kernel<NODAL, false, AOS>, smem) ||
      smem_optin((const void *)tensor_volume_kernel<NODAL, true, AOS>, smem) ||
      smem_optin((const void *)tensor_gs_kernel<NODAL, AOS>, smem))
    return HHG_ERR_CUDA;
  return HHG_OK;
}

// tiles of the staged tensor kernel: (element, i0, j0, kmax), 32 x TR
// points per plane, ordered (group of 8 elements, band, element, i) like the
// scalar volume tiles so co-running CTAs share halo rows in L2
struct TenTiles {
  int count = 0;
  int4 *dev = nullptr;
};

static int tensor_tiles(int n, int ntets, int tr, TenTiles &out) {
  static std::map<std::tuple<int, int, int, int>, TenTiles> cache;
  std::lock_guard<std::mutex> lock(g_cache_mu);
  const auto key = std::make_tuple(current_device(), n, ntets, tr);
  auto it = cache.find(key);
  if (it == cache.end()) {
    std::vector<int4> tl;
    for (int g0 = 0; g0 < ntets; g0 += 8)
      for (int j0 = 1; j0 <= n - 3; j0 += tr)
        for (int t = g0; t < std::min(g0 + 8, ntets); ++t)
          for (int i0 = 1; i0 + j0 <= n - 2; i0 += 32)
            tl.push_back(make_int4(t, i0, j0, n - 1 - i0 - j0));
    TenTiles e;
    int rc = upload(tl, &e.dev);
    if (rc) return rc;
    e.count = (int)tl.size();
    it = cache.emplace(key, e).first;
  }
  out = it->second;
  return HHG_OK;
}

template <bool NODAL>
static int ten_tile_apply(const TenDesc &D, bool res, cudaStream_t st) {
  TenTiles cache;
  int rc = tensor_tiles(D.n, D.ntets, tt_rows<NODAL>(), cache);
  if (rc) return rc;
  const int smem = (int)tt_smem<NODAL>();
  if (smem_optin((const void *)tensor_tile_kernel<NODAL, false>, smem) ||
      smem_optin((const void *)tensor_tile_kernel<NODAL, true>, smem))
    return HHG_ERR_CUDA;
  if (cache.count == 0) return HHG_OK;
  if (res)
    tensor_tile_kernel<NODAL, true><<<cache.count, tt_threads<NODAL>(), smem, st>>>(D, cache.dev);
  else
    tensor_tile_kernel<NODAL, false><<<cache.count, tt_threads<NODAL>(), smem, st>>>(D, cache.dev);
  return check("tensor_tile_kernel");
}

template <bool NODAL, bool AOS>
static int ten_apply(const TenDesc &D, bool res, cudaStream_t st) {
  if (D.n < 4) return HHG_OK;
#ifndef HHG_TENSOR_TILED
#define HHG_TENSOR_TILED 1
#endif
  if (AOS && HHG_TENSOR_TILED) return ten_tile_apply<NODAL>(D, res, st);
  int rc = ten_smem_ok<NODAL, AOS>();
  if (rc) return rc;
  constexpr int R = ten_rows<NODAL>();
  const dim3 grid(D.n - 3, (D.n - 3 + R - 1) / R, D.ntets), block(32, R);
  const size_t smem = ten_smem<NODAL>(ten_threads<NODAL>());
  if (res) tensor_volume_kernel<NODAL, true, AOS><<<grid, block, smem, st>>>(D);
  else tensor_volume_kernel<NODAL, false, AOS><<<grid, block, smem, st>>>(D);
  return check("tensor_volume_kernel");
}

template <bool NODAL, bool AOS>
static int ten_gs(TenDesc D, cudaStream_t st) {
  if (D.n < 4) return HHG_OK;
  int rc = ten_smem_ok<NODAL, AOS>();
  if (rc) return rc;
  rc = hyperplanes(D.n, &D.hp_ptr, &D.hp_code);
  if (rc) return rc;
  tensor_gs_kernel<NODAL, AOS><<<D.ntets, ten_threads<NODAL>(),
                                 ten_smem<NODAL>(ten_threads<NODAL>()), st>>>(D);
  return check("tensor_gs_kernel");
}

static TenDesc ten_elem(int64_t n, const double *v, const double *km, const double *coef) {
  TenDesc D{};
  D.n = (int)n;
  D.ntets = 1;
  D.L = tetra(n);
  D.nvol = n >= 4 ? tetra(n - 4) : 0;
  D.km = km;
  D.u = v;
  D.coef = coef;
  D.out_split = 0;
  return D;
}

static TenDesc ten_grid(const hhg_grid *g, const double *km, const double *coef) {
  TenDesc D{};
  D.n = g->n;
  D.ntets = g->ntets;
  D.L = g->lat_size;
  D.S = g->shell_size;
  D.nvol = g->nvol;
  D.vol_start = reinterpret_cast<const long long *>(g->vol_start);
  D.ghost = g->ghost;
  D.km = km;
  D.coef = coef;
  D.out_split = 1;
  return D;
}

// u (split global layout + current ghost shells) -> element lattices
static int ten_gather(const TenDesc &G, const double *u, double *lat, cudaStream_t st) {
  TenDesc D = G;
  D.u = u;
  const dim3 grid(D.n + 1, (D.n + 1 + 3) / 4, D.ntets), block(32, 4);
  lattice_gather_kernel<<<grid, block, 0, st>>>(D, lat);
  return check("lattice_gather_kernel");
}

extern "C" {

int hhg_apply_scaling_tensor_3d(int64_t n, const int64_t *, const double *v,
                                const double *km, int64_t M, const double *shm,
                                double *out, void *stream) {
  if (n > HHG_MAX_N) return HHG_ERR_ARG;   // 32-bit lattice forms, 10-bit point codes
  if (M != kTenM) return HHG_ERR_ARG;
  TenDesc D = ten_elem(n, v, km, shm);
  D.out = out;
  return ten_apply<false, false>(D, false, S(stream));
}

int hhg_apply_nodal_tensor_3d(int64_t n, const int64_t *, const double *v, const double *km,
                              int64_t M, const int64_t *sched, int64_t nsched,
                              const int64_t *sums, const double *fac, const int64_t *tptr,
                              const int64_t *telem, double *out, void *stream) {
  if (n > HHG_MAX_N) return HHG_ERR_ARG;   // 32-bit lattice forms, 10-bit point codes
  if (M != kTenM) return HHG_ERR_ARG;
  if (!tables_match(sched, nsched, sums, tptr, telem)) return HHG_ERR_TABLE;
  TenDesc D = ten_elem(n, v, km, fac);
  D.out = out;
  return ten_apply<true, false>(D, false, S(stream));
}

int hhg_gs_scaling_tensor_3d(int64_t n, const int64_t *, double *u, const double *fv,
                             const double *km, int64_t M, const double *shm, double omega,
                             void *stream) {
  if (n > HHG_MAX_N) return HHG_ERR_ARG;   // 32-bit lattice forms, 10-bit point codes
  if (M != kTenM) return HHG_ERR_ARG;
  TenDesc D = ten_elem(n, u, km, shm);
  D.f = fv;
  D.omega = omega;
  return ten_gs<false, false>(D, S(stream));
}

int hhg_gs_nodal_tensor_3d(int64_t n, const int64_t *, double *u, const double *fv,
                           const double *km, int64_t M, const int64_t *sched, int64_t nsched,
                           const int64_t *sums, const double *fac, const int64_t *tptr,
                           const int64_t *telem, double omega, void *stream) {
  if (n > HHG_MAX_N) return HHG_ERR_ARG;   // 32-bit lattice forms, 10-bit point codes
  if (M != kTenM) return HHG_ERR_ARG;
  if (!tables_match(sched, nsched, sums, tptr, telem)) return HHG_ERR_TABLE;
  TenDesc D = ten_elem(n, u, km, fac);
  D.f = fv;
  D.omega = omega;
  return ten_gs<true, false>(D, S(stream));
}

int hhg_tensor_volume_apply(const hhg_grid *g, int variant, int flags, int M,
                            const double *km, const double *coef, const double *u,
                            const double *f, double *out, double *work, void *stream) {
  if (g->n > HHG_MAX_N) return HHG_ERR_ARG;   // 32-bit lattice forms, 10-bit point codes
  if (M != kTenM || !work) return HHG_ERR_ARG;
  if (variant != HHG_VAR_SCALING && variant != HHG_VAR_NODAL) return HHG_ERR_ARG;
  const bool res = (flags & HHG_FLAG_RESIDUAL) != 0;
  if (res && !f) return HHG_ERR_ARG;
  if (g->n < 4) return HHG_OK;
  TenDesc D = ten_grid(g, km, coef);
  int rc = ten_gather(D, u, work, S(stream));
  if (rc) return rc;
  D.u = work;
  D.f = f;
  D.out = out;
  return variant == HHG_VAR_NODAL ? ten_apply<true, true>(D, res, S(stream))
                                  : ten_apply<false, true>(D, res, S(stream));
}

int hhg_tensor_smooth_volume(const hhg_grid *g, int variant, int M, const double *km,
                             const double *coef, double omega, double *u, const double *f,
                             double *work, void *stream) {
  if (g->n > HHG_MAX_N) return HHG_ERR_ARG;   // 32-bit lattice forms, 10-bit point codes
  if (M != kTenM || !work) return HHG_ERR_ARG;
  if (variant != HHG_VAR_SCALING && variant != HHG_VAR_NODAL) return HHG_ERR_ARG;
  if (g->n < 4) return HHG_OK;
  TenDesc D = ten_grid(g, km, coef);
  int rc = ten_gather(D, u, work, S(stream));
  if (rc) return rc;
  D.u = work;
  D.f = f;
  D.omega = omega;
  rc = variant == HHG_VAR_NODAL ? ten_gs<true, true>(D, S(stream))
                                : ten_gs<false, true>(D, S(stream));
  if (rc) return rc;
  const dim3 grid(D.n - 3, (D.n - 3 + 3) / 4, D.ntets), block(32, 4);
  lattice_scatter_kernel<<<grid, block, 0, S(stream)>>>(D, work, u);
  return check("lattice_scatter_kernel");
}

int hhg_tensor_surface_prepare(const hhg_grid *g, const hhg_surface *s,
                               const hhg_surface_gs *gs, int M, const double *km,
                               void *stream) {
  if (g->n > HHG_MAX_N) return HHG_ERR_ARG;   // 32-bit lattice forms, 10-bit point codes
  if (M != kTenM) return HHG_ERR_ARG;
  if (s->nrows <= 0) return HHG_OK;
  SurfGSDesc G{};
  G.s = surf_desc(g, s);
  G.shell_gid = reinterpret_cast<const long long *>(g->shell_gid);
  G.ent_ptr = reinterpret_cast<const long long *>(gs->ent_ptr);
  G.ent_col = gs->ent_col;
  G.ent_val = gs->ent_val;
  G.row_diag = gs->row_diag;
  tensor_surface_fill_kernel<<<(int)((s->nrows + 127) / 128), 128, 0, S(stream)>>>(G, km);
  return check("tensor_surface_fill_kernel");
}

long long hhg_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int hhg_status(void) {
  int v = 0;
  cudaMemcpyFromSymbol(&v, g_status, sizeof(int));
  return v ? HHG_ERR_ZERO_DIAG : HHG_OK;
}

int hhg_status_reset(void) {
  int z = 0;
  cudaMemcpyToSymbol(g_status, &z, sizeof(int));
  return HHG_OK;
}

int hhg_volume_tile_rows(void) { return kW * kB; }
int hhg_face_tile(void) { return FACE_TA << 16 | FACE_TB; }   // W*B rows (W/4 warp rows of 4B)
int hhg_volume_tile_cols_mirror(void) { return 8 * HHG_MIRROR_NW; }

// host-side level schedule of the surface Gauss-Seidel: rows are in
// ascending global id, dep_idx[dep_ptr[r]..dep_ptr[r+1]) lists the row
// indices q < r row r reads updated values from.  level[r] = 1 + max level[q]
// in one ascending pass (O(nnz)).  Returns the number of levels.
int hhg_host_gs_levels(int64_t nrows, const int64_t *dep_ptr, const int64_t *dep_idx,
                       int64_t *level) {
  return hhg_host_gs_levels_seeded(nrows, dep_ptr, dep_idx, nullptr, level);
}

// the same with lower bounds seed[r] (sharded sweeps: the levels the
// neighbour rank computed for the shared interface rows)
int hhg_host_gs_levels_seeded(int64_t nrows, const int64_t *dep_ptr, const int64_t *dep_idx,
                              const int64_t *seed, int64_t *level) {
  int64_t nlev = 0;
  for (int64_t r = 0; r < nrows; ++r) {
    int64_t lv = seed ? seed[r] : 0;
    for (int64_t e = dep_ptr[r]; e < dep_ptr[r + 1]; ++e) {
      const int64_t q = dep_idx[e];
      if (q >= r) return HHG_ERR_ARG;
      if (level[q] + 1 > lv) lv = level[q] + 1;
    }
    level[r] = lv;
    if (lv + 1 > nlev) nlev = lv + 1;
  }
  return (int)nlev;
}

const char *hhg_build_info(void) {
  static char buf[128];
  snprintf(buf, sizeof buf, "sm_100a volume B=%d W=%d NS=%d MINB=%d mirror NW=%d", kB, kW, kNS,
           HHG_VOL_MINB, HHG_MIRROR_NW);
  return buf;
}

}  // extern "C"

#include "hhg_vector.cuh"
