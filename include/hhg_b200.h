/*
 * hhg_b200.h — C ABI of the B200 stencil-scaling operator library
 * (libhhg_b200.so, built from paper_1709_06793_b200/csrc/*.cu for sm_100a).
 *
 * Plain pointers and sizes only.  Unless stated otherwise every array
 * argument is a DEVICE pointer owned by the caller, `stream` is a
 * cudaStream_t (NULL = legacy default stream) and every call is
 * asynchronous on that stream.  No entry point allocates device memory.
 *
 * Return codes: HHG_OK, or a negative HHG_ERR_* code.  HHG_ERR_ZERO_DIAG is
 * the C form of the reference's ValueError("zero central stencil entry")
 * (pkg/src/hhgscale/kernels.py:547-548); it is reported by the *_status
 * query after the stream has been synchronised.
 *
 * Two layers:
 *  (1) per-macro-element kernels with exactly the arguments the reference
 *      passes to its numba kernels from Operator._run_volume / smooth
 *      (operators.py:391-462, 522-535) — lattice arrays of one element;
 *  (2) batched, fused entry points used by the drop-in Operator: all macro
 *      elements in one launch, reading the global vector directly plus a
 *      compact per-element ghost shell.
 */
#ifndef HHG_B200_H
#define HHG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HHG_OK 0
#define HHG_ERR_ARG (-1)
/* largest supported lattice size n = 2^level (level 9): lattice offsets are
 * 32-bit closed forms and point codes pack i, j, k in 10 bits each; every
 * entry point returns HHG_ERR_ARG for larger n */
#define HHG_MAX_N 512
#define HHG_ERR_CUDA (-2)
#define HHG_ERR_ZERO_DIAG (-3)
#define HHG_ERR_TABLE (-4)

/* operator variants of the volume kernels (operators.py:32) */
#define HHG_VAR_SCALING 0
#define HHG_VAR_NODAL 1
#define HHG_VAR_CONST 2
#define HHG_VAR_STORED 3

/* flags */
#define HHG_FLAG_RESIDUAL 1 /* write f - A u instead of A u               */
#define HHG_FLAG_FAST 2     /* FMA / mirror-pair reassociated arithmetic
                               (scaling and nodal rows; within 1e-12 of
                               the reference order)                        */
#define HHG_FLAG_MIRROR 4   /* caller guarantees sh[d] == sh[d+7] bitwise
                               for every element: edge terms shared by two
                               rows are evaluated once (result unchanged)  */

/* ---------------------------------------------------------------------
 * (1) per-macro-element kernels (lattice layout of one element)
 * n      : lattice size 2^level;  base: (n+1)*(n+1) int64 row table of
 *          SimplexLattice(3, n) (mesh.py:457-504) — the kernels use its
 *          closed form and accept only that canonical table (or NULL).
 * v, kc  : float64[(n+1)(n+2)(n+3)/6] lattice arrays
 * out    : float64[(n-1)(n-2)(n-3)/6] volume rows in (k, j, i) order
 * --------------------------------------------------------------------- */

/* replaces kernels.apply_scaling_3d(n, base, v, kc, sh, out), kernels.py:90-136 */
int hhg_apply_scaling_3d(int64_t n, const int64_t *base, const double *v,
                         const double *kc, const double *sh, double *out,
                         void *stream);

/* replaces kernels.apply_nodal_3d(n, base, v, kc, sched, sums, fac, tptr,
 * telem, out), kernels.py:139-189.  sched (40x3), sums (24), tptr (15) and
 * telem (72) are HOST int64 tables; they must equal the frozen patch tables
 * (reference_stencils.py:48-75) the kernel is compiled with, else
 * HHG_ERR_TABLE.  fac (72) is a device pointer. */
int hhg_apply_nodal_3d(int64_t n, const int64_t *base, const double *v,
                       const double *kc, const int64_t *sched, int64_t nsched,
                       const int64_t *sums, const double *fac,
                       const int64_t *tptr, const int64_t *telem, double *out,
                       void *stream);

/* replaces kernels.apply_const_3d(n, base, v, s, c0, out), kernels.py:22-53;
 * s is a device pointer to the 14 neighbour weights, c0 the diagonal weight */
int hhg_apply_const_3d(int64_t n, const int64_t *base, const double *v,
                       const double *s, double c0, double *out, void *stream);

/* replaces kernels.apply_stored_3d(n, base, v, w, out), kernels.py:56-87;
 * w is float64[nvol][15] */
int hhg_apply_stored_3d(int64_t n, const int64_t *base, const double *v,
                        const double *w, double *out, void *stream);

/* replaces kernels.csr_gs(rows, indptr, indices, data, diag, u, f, omega),
 * kernels.py:979-992: forward Gauss-Seidel over rows[0..nrows_list) of a
 * CSR matrix (int64 indptr / indices, float64 data; diag indexed by row id)
 * in list order, bitwise the sequential loop; a zero diagonal stops the
 * sweep at that row and is reported by hhg_status (HHG_ERR_ZERO_DIAG). */
int hhg_csr_gs(int64_t nrows_list, const int64_t *rows, const int64_t *indptr,
               const int64_t *indices, const double *data, const double *diag,
               double *u, const double *f, double omega, void *stream);

/* replaces kernels.gs_scaling_3d(n, base, u, fv, kc, sh, omega),
 * kernels.py:510-550: forward lexicographic Gauss-Seidel in place on the
 * lattice array u, executed as i+2j+3k hyperplane wavefronts (bitwise the
 * same update sequence). */
int hhg_gs_scaling_3d(int64_t n, const int64_t *base, double *u,
                      const double *fv, const double *kc, const double *sh,
                      double omega, void *stream);

/* replaces kernels.apply_scaling_2d(n, base, v, kc, kg, g, sh, out),
 * kernels.py:750-782: 2-D scaled stencil on a triangle lattice (row j at
 * base[j] = j (n+1) - j (j-1)/2), v, kc, kg float64[(n+1)(n+2)/2], sh (6)
 * and out ((n-1)(n-2)/2 rows) device pointers; g: 6 HOST flags, the
 * uniform-ellipticity (MA2) gray-edge selector - direction d averages the
 * safeguarded coefficient kg instead of kc where g[d] != 0 */
int hhg_apply_scaling_2d(int64_t n, const int64_t *base, const double *v,
                         const double *kc, const double *kg, const uint8_t *g,
                         const double *sh, double *out, void *stream);
/* replaces kernels.gs_scaling_2d(n, base, u, fv, kc, kg, g, sh, omega),
 * kernels.py:906-937 (wavefronts i + 2j, bitwise the sequential sweep) */
int hhg_gs_scaling_2d(int64_t n, const int64_t *base, double *u, const double *fv,
                      const double *kc, const double *kg, const uint8_t *g,
                      const double *sh, double omega, void *stream);

/* replaces kernels.gs_nodal_3d(...), kernels.py:553-600 (tables as above) */
int hhg_gs_nodal_3d(int64_t n, const int64_t *base, double *u,
                    const double *fv, const double *kc, const int64_t *sched,
                    int64_t nsched, const int64_t *sums, const double *fac,
                    const int64_t *tptr, const int64_t *telem, double omega,
                    void *stream);

/* ---------------------------------------------------------------------
 * (2) batched operator descriptor: all macro elements of one grid level
 * --------------------------------------------------------------------- */
typedef struct hhg_grid {
  int32_t n;               /* 2^level                                        */
  int32_t ntets;           /* macro elements on this device                  */
  int64_t lat_size;        /* (n+1)(n+2)(n+3)/6                              */
  int64_t nvol;            /* (n-1)(n-2)(n-3)/6                              */
  int64_t shell_size;      /* ghost points per element (compact shell)       */
  int64_t n_nodes;         /* length of global vectors                       */
  const int64_t *vol_start;/* [ntets] global id of the first volume node     */
  const int32_t *srow;     /* [(n+1)^2] offset of lattice row (k,j) in shell */
  const int64_t *shell_gid;/* [ntets*shell_size] global id of ghost points   */
  double *ghost;           /* [ntets*shell_size] ghost-layer values          */
  const double *kc;        /* [ntets*lat_size] coefficient, lattice layout   */
  const int32_t *tiles;    /* [ntiles*4] (tet, i0, j0, kmax) volume tiles    */
  int32_t ntiles;
  int32_t nmtiles;         /* tiles of the mirror (default scaling) kernel,  */
  const int32_t *mtiles;   /* hhg_volume_tile_cols_mirror() columns wide     */
} hhg_grid;

/* one free macro face whose interior points are surface rows (face-tiled
 * surface kernel): incident elements tet[0] < tet[1] (tet[1] = -1: the other
 * side is on another rank), the face's boundary class in each, and the
 * affine map from face-local (a, b), a, b >= 1, a + b <= n - 1, to element
 * lattice coordinates: (i, j, k) = c[e] + (A[e][0] a + A[e][1] b,
 * A[e][2] a + A[e][3] b, A[e][4] a + A[e][5] b).  The element's layer next
 * to the face is (i, j, k) = c[e] + nb[e] + A[e] (a, b); stencil direction d
 * of a face point (a, b) reaches layer dl[e][d] (0 face, 1 inner, -1 none)
 * at (a + da[e][d], b + db[e][d]). */
typedef struct hhg_face {
  int32_t tet[2];
  int32_t cls[2];
  int32_t A[2][6];
  int32_t c[2][3];
  int32_t nb[2][3];
  int8_t dl[2][14];
  int8_t da[2][14];
  int8_t db[2][14];
  int32_t nodal;           /* 1: nodal-integration rows (hybrid / nodal)     */
  int64_t fs;              /* global id of the face's first interior point   */
  int64_t rbase;           /* surface-row index of fs (rows are sorted)      */
} hhg_face;

typedef struct hhg_surface {
  int64_t nrows;           /* non-Dirichlet surface rows                     */
  const int64_t *rows;     /* [nrows] global ids                             */
  const uint8_t *row_nodal;/* [nrows] 1: nodal-integration row (hybrid/nodal)*/
  /* row-major incidences (macro element, boundary lattice point) per row,
   * ordered by element: used by the Gauss-Seidel sweep                     */
  const int32_t *inc_ptr;  /* [nrows+1]                                      */
  const int32_t *inc_tet;  /* [ninc]                                         */
  const int32_t *inc_code; /* [ninc] i | j << 10 | k << 20 (lattice coords)  */
  const uint8_t *inc_cls;  /* [ninc] boundary class 0..13                    */
  const double *psh;       /* [ntets*14*14] one-sided half stencils          */
  const double *pfac;      /* [ntets*14*72] one-sided nodal factors or NULL  */
  int64_t ndir;            /* Dirichlet rows                                 */
  const int64_t *dir_ids;  /* [ndir]                                         */
  /* element-major copy of the incidences (lattice order inside each
   * element) for the apply: partial rows are computed with coalesced
   * lattice reads, then summed per row in element order                    */
  int64_t ninc;
  const int32_t *p_tet;    /* [ninc]                                         */
  const int32_t *p_code;   /* [ninc]                                         */
  const uint8_t *p_cls;    /* [ninc]                                         */
  const uint8_t *p_nodal;  /* [ninc] row of this incidence is a nodal row    */
  const int32_t *row_inc;  /* [ninc] element-major index, row-major order    */
  double *partial;         /* [ninc] scratch                                 */
  /* face-tiled apply (hhg_surface_apply_csr): the rows of nfaces free macro
   * faces from face_tiles (face, a0, b0, 0) of 32 x 8 points, the remaining
   * (edge / vertex) rows nsub row indices in sub_rows; nfaces = 0: every
   * row through the precomputed rows                                     */
  int64_t nfaces;
  const hhg_face *faces;
  int64_t nface_tiles;
  const int32_t *face_tiles;
  int64_t nsub;
  const int32_t *sub_rows;
  /* static per-face layers of the face-tiled kernel: for face x, layer l
   * (0 = the face, 1 + e = element e's layer next to it) and face-local
   * (a, b), a, b in [-1, n+1]: the coefficient and the global id of that
   * lattice point at [(x * 3 + l) * sq * sq + (b + 1) * sq + (a + 1)],
   * sq = n + 3 (k = 0 / id = 0 outside the element)                      */
  const double *face_k;
  const int32_t *face_g;
  int32_t face_sq;
  int32_t pad_;
} hhg_surface;

/* stencil dumps of all macro elements (kernels.dump_scaling_3d /
 * dump_nodal_3d, kernels.py:293-376): w[t][c][15] = (centre, s_0..s_13)
 * of volume row c; variant HHG_VAR_SCALING (coef: sh[14] per element) or
 * HHG_VAR_NODAL (coef: fac[72]); the stored-stencil baseline's input */
int hhg_dump_stencils(const hhg_grid *g, int variant, const double *coef, double *w,
                      void *stream);

/* refresh the ghost layers: ghost[e] = u[shell_gid[e]] */
int hhg_ghost_update(const hhg_grid *g, const double *u, void *stream);

/* volume rows of all macro elements: out = A u (or f - A u with
 * HHG_FLAG_RESIDUAL).  coef: per element sh[14] (scaling), fac[72]
 * (nodal), s[14]+c0 (const, 15 doubles) or NULL (stored: w is
 * [ntets*nvol*15]).  Reads the ghost layer: call hhg_ghost_update first. */
int hhg_volume_apply(const hhg_grid *g, int variant, int flags,
                     const double *coef, const double *w, const double *u,
                     const double *f, double *out, void *stream);

/* surface rows (vertex/edge/face primitives) as sums of one-sided
 * partial stencils over the incident macro elements, plus Dirichlet
 * identity rows (0 for residuals). */
int hhg_surface_apply(const hhg_grid *g, const hhg_surface *s, int variant,
                      int flags, const double *u, const double *f,
                      double *out, void *stream);

/* ---------------------------------------------------------------------
 * vector kernels (CG / multigrid plumbing)
 * --------------------------------------------------------------------- */
/* result[0] = sum_i x[i]*y[i] (deterministic two-pass reduction);
 * work must hold >= 1024 doubles */
int hhg_dot(int64_t n, const double *x, const double *y, double *work,
            double *result, void *stream);
/* y = a*x + y with a read from device memory: a = sign * num[0]/den[0] */
int hhg_axpy_ratio(int64_t n, const double *num, const double *den,
                   double sign, const double *x, double *y, void *stream);
/* p = r + (num/den) p */
int hhg_xpay_ratio(int64_t n, const double *num, const double *den,
                   const double *r, double *p, void *stream);

/* fused CG / PCG updates (multigrid.py:169-194), scalars in device memory,
 * one pass each with the next dot's partials formed on the way (work: >= 1024
 * doubles; bitwise the separate axpy / dot sequence):
 *   cg_update : a = rs/pAp; x += a p; r -= a Ap; rs_new = r.r (over the
 *               entries with mask != 0 when mask is not NULL)
 *   pcg_update: a = rz/pAp; x += a p; r_new = r - a Ap; rr_new = r_new.r_new
 *   dot2      : result[0] = (a - b).c, result[1] = a.c (work >= 2048)
 *   dot_masked: result[0] = sum over mask != 0 of x y (sharded vectors)    */
int hhg_cg_update(int64_t n, const double *rs, const double *pAp, const double *p,
                  const double *Ap, double *x, double *r, const uint8_t *mask,
                  double *work, double *rs_new, void *stream);
int hhg_pcg_update(int64_t n, const double *rz, const double *pAp, const double *p,
                   const double *Ap, double *x, const double *r, double *r_new,
                   double *work, double *rr_new, void *stream);
int hhg_dot2(int64_t n, const double *a, const double *b, const double *c, double *work,
             double *result, void *stream);
int hhg_dot_masked(int64_t n, const double *x, const double *y, const uint8_t *mask,
                   double *work, double *result, void *stream);

/* y = A x for a CSR matrix (prolongation, restriction = P^T as a CSR of
 * the transpose); rows accumulate in stored column order (bitwise scipy) */
int hhg_csr_spmv(int64_t nrows, const int64_t *indptr, const int64_t *indices,
                 const double *data, const double *x, double *y, int accumulate,
                 void *stream);

/* grid transfers between levels l-1 (coarse) and l (fine) of one macro
 * mesh (multigrid.py:23-77, 130-138), lattice-native: volume rows in
 * closed form from the element lattices, the rows of surface nodes (macro
 * vertices / edges / faces) from small host-built CSRs with a row list */
typedef struct hhg_transfer {
  int32_t nf, nc;              /* fine / coarse 2^level                          */
  int32_t ntets, pad_;
  const int64_t *f_vol_start;  /* [ntets] fine volume blocks                     */
  const int64_t *c_vol_start;  /* [ntets] coarse volume blocks                   */
  const int64_t *c_shell_gid;  /* [ntets * c_shell_size] coarse ghost-shell ids  */
  int64_t c_shell_size;
  /* P rows of the fine surface nodes: y[p_rows[r]] = sum p_val x[p_col]     */
  int64_t p_nrows;
  const int64_t *p_rows, *p_ptr, *p_col;
  const double *p_val;
  /* P^T rows of the coarse surface nodes (children in ascending fine id)   */
  int64_t r_nrows;
  const int64_t *r_rows, *r_ptr, *r_col;
  const double *r_val;
  int64_t ndir;                /* coarse Dirichlet ids, zeroed by the restriction */
  const int64_t *c_dir_ids;
} hhg_transfer;

/* yf = P xc (accumulate != 0: yf += P xc), bitwise the reference's P @ x */
int hhg_prolongate(const hhg_transfer *T, const double *xc, double *yf, int accumulate,
                   void *stream);
/* yc = P^T xf with the coarse Dirichlet rows zeroed, bitwise the
 * reference's restrict (P.T @ r, then r[dirichlet] = 0) */
int hhg_restrict(const hhg_transfer *T, const double *xf, double *yc, void *stream);

/* y[ids[e]] = 0 (coarse Dirichlet rows after restriction) */
int hhg_scatter_zero(int64_t n, const int64_t *ids, double *y, void *stream);

/* interface exchange over NCCL (shard.exchange_partials; the reference has
 * no distributed path - its single-domain apply is operators.py:485-499):
 * y[e] = x[ids[e]] packs a rank's one-sided interface rows (mine) for the
 * send; out[ids[e]] = recv[e] + mine[e] (recv_first) or mine[e] + recv[e]
 * completes them in rank order, so both ranks hold bitwise equal rows */
int hhg_gather(int64_t n, const int64_t *ids, const double *x, double *y, void *stream);
int hhg_interface_add(int64_t n, const int64_t *ids, const double *mine, const double *recv,
                      int recv_first, double *out, void *stream);

/* smoother pieces (Operator.smooth): one level of the level-scheduled
 * surface Gauss-Seidel (rows given as indices into s->rows), and the volume
 * hyperplane wavefronts of all macro elements (reads the ghost layer, which
 * must be refreshed after the surface sweep) */
int hhg_smooth_surface_level(const hhg_grid *g, const hhg_surface *s,
                             const int64_t *level_rows, int64_t count,
                             double omega, double *u, const double *f,
                             void *stream);
/* precomputed surface rows of the smoother (level schedule + each row's
 * neighbour ids and weights in accumulation order); all DEVICE arrays */
typedef struct hhg_surface_gs {
  const int64_t *level_rows;  /* [nrows] rows ordered by level               */
  const int64_t *level_ptr;   /* [nlev+1]                                     */
  int64_t nlev;
  const int64_t *ent_ptr;     /* [nrows+1]                                    */
  int32_t *ent_col;           /* [nent] global ids (filled by _prepare)       */
  double *ent_val;            /* [nent] weights (filled by _prepare)          */
  double *row_diag;           /* [nrows] diagonals (filled by _prepare)       */
  /* optional level-ordered copy for the one-cluster sweep (filled by
   * hhg_smooth_surface_slots; NULL = not built): slot e is row
   * level_rows[e]; its first HHG_SURF_SLOT_PF entries are stored
   * slot-interleaved (entry m of slot e at m * nslots + e), so a thread
   * reads its next row with no dependent loads */
  int64_t nslots;             /* = nrows                                      */
  int64_t *slot_gid;          /* [nslots] global id of the row                */
  int32_t *slot_cnt;          /* [nslots] entries of the row                  */
  double *slot_diag;          /* [nslots]                                     */
  int32_t *slot_col;          /* [HHG_SURF_SLOT_PF * nslots]                  */
  double *slot_val;           /* [HHG_SURF_SLOT_PF * nslots]                  */
  int32_t *slot_dyn;          /* [nslots] bit m: entry m is a row of the
                                 previous level (read after the barrier; the
                                 others are prefetched across it)            */
  uint32_t *sweep_bar;        /* [1] scratch: arrival counter of the grid
                                 sweep's barrier (one per schedule, so
                                 sweeps on different streams never share) */
} hhg_surface_gs;
#define HHG_SURF_SLOT_PF 24

/* apply / residual of the surface rows (+ Dirichlet rows) from the rows
 * precomputed by hhg_smooth_surface_prepare; bitwise the matrix-free
 * surface kernels' result (the weights are the factors they recompute) */
int hhg_surface_apply_csr(const hhg_grid *g, const hhg_surface *s,
                          const hhg_surface_gs *gs, int flags, const double *u,
                          const double *f, double *out, void *stream);

/* ---------------------------------------------------------------------
 * multi-GPU interface exchange over peer memory (one process per GPU,
 * SURVEY.md §8e).  The interface rows' one-sided values are pushed into the
 * neighbour's receive buffer by the kernel that computes them, a signal
 * bumps the neighbour's arrival counter, and a pull kernel completes the
 * rows in rank order once the neighbour's values have arrived.
 * --------------------------------------------------------------------- */

/* apply (no residual) surface + Dirichlet rows as hhg_surface_apply_csr,
 * and for rows r with push_slot[r] >= 0 also store the row's value into
 * dst0[push_slot[r]] (slot < split) or dst1[push_slot[r] - split]: peer
 * device pointers (CUDA IPC) of the neighbours' receive buffers */
int hhg_surface_apply_csr_push(const hhg_grid *g, const hhg_surface *s,
                               const hhg_surface_gs *gs, const double *u, double *out,
                               const int32_t *push_slot, double *dst0, double *dst1,
                               int64_t split, void *stream);
/* system-scope fence, then atomically add 1 to the neighbour's counter */
int hhg_p2p_signal(unsigned long long *remote_flag, void *stream);
/* wait (bounded; *err = 1 on timeout) until *flag >= target, then
 * out[ids[i]] = recv_first ? recv[i] + out[ids[i]] : out[ids[i]] + recv[i] */
int hhg_p2p_pull(double *out, const int64_t *ids, int64_t count, const double *recv,
                 const unsigned long long *flag, unsigned long long target,
                 int recv_first, int *err, void *stream);
/* zero-initialised device allocation of its own (an IPC handle maps a whole
 * allocation, so exchange buffers are not sub-allocated) / release */
int hhg_device_alloc(int64_t bytes, void **ptr);
int hhg_device_free(void *ptr);
/* CUDA IPC plumbing: 64-byte handle of a hhg_device_alloc allocation; open /
 * close a peer's allocation in this process */
int hhg_ipc_get_handle(const void *ptr, void *handle);
int hhg_ipc_open_handle(const void *handle, void **ptr);
int hhg_ipc_close_handle(void *ptr);

int hhg_smooth_surface_prepare(const hhg_grid *g, const hhg_surface *s,
                               const hhg_surface_gs *gs, void *stream);
/* fill gs->slot_* (allocated by the caller) from the level schedule and
 * the prepared rows; call after _prepare and whenever they change.
 * gid_level[x] (device, nlv entries): level of the schedule row with global
 * id x, -1 for ids that are not rows of the sweep */
int hhg_smooth_surface_slots(const hhg_grid *g, const hhg_surface *s,
                             const hhg_surface_gs *gs, const int32_t *gid_level,
                             int64_t nlv, void *stream);
/* every level of the surface sweep in one launch: one thread-block cluster
 * with a cluster barrier between levels (narrow schedules, slots built), or
 * a cooperative grid with grid barriers */
int hhg_smooth_surface_all(const hhg_grid *g, const hhg_surface *s,
                           const hhg_surface_gs *gs, double omega, double *u,
                           const double *f, void *stream);
int hhg_smooth_volume(const hhg_grid *g, int variant, const double *coef,
                      double omega, double *u, const double *f, void *stream);
/* the same volume sweep in a hyperplane-major ("skewed") copy of each
 * element's whole lattice: u with its ghost (boundary) values is gathered
 * into us and ks holds the coefficient (ntets * L doubles each, L = lattice
 * points per element; ks filled once per operator by hhg_skew_coefficient),
 * f into fs (ntets * nvol doubles); the interior is swept with coalesced,
 * branch-free accesses and scattered back into u.  Bitwise
 * hhg_smooth_volume.  Caller-owned buffers.  flags (later sweeps of one
 * smoothing): HHG_SKEW_F_CURRENT - fs already holds this f;
 * HHG_SKEW_U_CURRENT - the interior of us equals u's (only the boundary
 * values are refreshed from the ghost shell). */
#define HHG_SKEW_F_CURRENT 1
#define HHG_SKEW_U_CURRENT 2
int hhg_skew_coefficient(const hhg_grid *g, double *ks, void *stream);
int hhg_smooth_volume_skew(const hhg_grid *g, int variant, const double *coef,
                           double omega, double *u, const double *f, double *us,
                           double *fs, const double *ks, int flags, void *stream);

/* ---------------------------------------------------------------------
 * (3) tensor-coefficient operators, M = 6 component fields
 *     (coefficients.py:120-200, TENSOR_DIRS_3D).  km is float64[M][L] per
 *     element (device), shm float64[M][14], fac float64[M][72]; any other
 *     M returns HHG_ERR_ARG.
 * --------------------------------------------------------------------- */

/* replaces kernels.apply_scaling_tensor_3d(n, base, v, km, shm, out),
 * kernels.py:192-232 (M = km.shape[0] passed explicitly) */
int hhg_apply_scaling_tensor_3d(int64_t n, const int64_t *base, const double *v,
                                const double *km, int64_t M, const double *shm,
                                double *out, void *stream);

/* replaces kernels.apply_nodal_tensor_3d(n, base, v, km, sched, sums, fac,
 * tptr, telem, out), kernels.py:235-286 (host tables as for
 * hhg_apply_nodal_3d) */
int hhg_apply_nodal_tensor_3d(int64_t n, const int64_t *base, const double *v,
                              const double *km, int64_t M, const int64_t *sched,
                              int64_t nsched, const int64_t *sums, const double *fac,
                              const int64_t *tptr, const int64_t *telem, double *out,
                              void *stream);

/* replaces kernels.gs_scaling_tensor_3d(n, base, u, fv, km, shm, omega),
 * kernels.py:603-640 (hyperplane wavefronts, bitwise the sequential sweep) */
int hhg_gs_scaling_tensor_3d(int64_t n, const int64_t *base, double *u,
                             const double *fv, const double *km, int64_t M,
                             const double *shm, double omega, void *stream);

/* replaces kernels.gs_nodal_tensor_3d(...), kernels.py:643-702 */
int hhg_gs_nodal_tensor_3d(int64_t n, const int64_t *base, double *u,
                           const double *fv, const double *km, int64_t M,
                           const int64_t *sched, int64_t nsched, const int64_t *sums,
                           const double *fac, const int64_t *tptr,
                           const int64_t *telem, double omega, void *stream);

/* batched volume rows of the tensor operators (Operator._run_volume tensor
 * branch, operators.py:406-426): variant HHG_VAR_SCALING or HHG_VAR_NODAL;
 * km [ntets][L][M] (all components of a point contiguous), coef
 * [ntets][M][14 | 72]; flags: HHG_FLAG_RESIDUAL.  work: caller-owned
 * float64[ntets * lat_size] scratch: u is gathered into element lattices
 * first (the reference's u[elem_gidx[t]], operators.py:383; ghost shells
 * must be current), the smoother scatters the interior back afterwards. */
int hhg_tensor_volume_apply(const hhg_grid *g, int variant, int flags, int M,
                            const double *km, const double *coef, const double *u,
                            const double *f, double *out, double *work, void *stream);
int hhg_tensor_smooth_volume(const hhg_grid *g, int variant, int M, const double *km,
                             const double *coef, double omega, double *u,
                             const double *f, double *work, void *stream);
/* surface rows of the tensor operators (operators.py:277-327 tensor branch):
 * s->psh is [ntets][M][14][14], s->pfac [ntets][M][14][72], km as above
 * ([ntets][L][M]); fills the same
 * precomputed rows hhg_smooth_surface_prepare fills for scalar k, so
 * hhg_surface_apply_csr / hhg_smooth_surface_all serve both */
int hhg_tensor_surface_prepare(const hhg_grid *g, const hhg_surface *s,
                               const hhg_surface_gs *gs, int M, const double *km,
                               void *stream);

/* HOST helper: level schedule of the surface Gauss-Seidel (see .cu);
 * _seeded: with lower bounds seed[r] (NULL = 0) */
int hhg_host_gs_levels(int64_t nrows, const int64_t *dep_ptr,
                       const int64_t *dep_idx, int64_t *level);
int hhg_host_gs_levels_seeded(int64_t nrows, const int64_t *dep_ptr,
                              const int64_t *dep_idx, const int64_t *seed, int64_t *level);

/* sharded surface sweep (one level of the global schedule, explicit row
 * index lists): rows updated directly; the partial row sums of shared
 * interface rows (acc over this rank's incidences, its part of the
 * diagonal) and the update from the rank-ordered sums of both sides */
int hhg_smooth_surface_rows(const hhg_grid *g, const hhg_surface *s,
                            const hhg_surface_gs *gs, const int64_t *rows, int64_t count,
                            double omega, double *u, const double *f, void *stream);
int hhg_smooth_surface_partial(const hhg_grid *g, const hhg_surface *s,
                               const hhg_surface_gs *gs, const int64_t *rows, int64_t count,
                               const double *u, double *acc, double *diag, void *stream);
int hhg_smooth_surface_finish(const hhg_grid *g, const hhg_surface *s,
                              const hhg_surface_gs *gs, const int64_t *rows, int64_t count,
                              const double *acc, const double *diag, double omega,
                              double *u, const double *f, void *stream);

/* rows of one volume tile (W*B) the kernels were compiled with */
int hhg_volume_tile_rows(void);
/* face tile of the face-tiled surface kernel: (a extent << 16) | b extent */
int hhg_face_tile(void);
/* columns of one tile of the mirror kernel (hhg_grid.mtiles) */
int hhg_volume_tile_cols_mirror(void);

/* status word of the last GS launch (HHG_OK / HHG_ERR_ZERO_DIAG) — call
 * after synchronising the stream */
int hhg_status(void);
int hhg_status_reset(void);

/* number of kernel launches this library has issued in the process
 * (host-side counter; every launch site counts one) */
long long hhg_launch_count(void);

/* compile-time kernel configuration, for reports */
const char *hhg_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* HHG_B200_H */
