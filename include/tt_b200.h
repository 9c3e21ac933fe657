/*
 * tt_b200.h -- C ABI of the B200-native Monte-Carlo conservative transfer library
 * (libtt_b200.so).  Plain pointers and sizes only; every pointer to array data is a
 * DEVICE pointer unless the comment says "host"; every call is stream-ordered on the
 * caller's cudaStream_t (passed as void*; NULL = legacy default stream) and returns a
 * TT_* status code (launch/parameter errors).  Data-dependent errors raised inside
 * kernels (non-finite source values, strict-outside samples) are OR-ed into a caller
 * supplied device int32 status word as TT_FLAG_* bits.
 *
 * Reference interfaces replaced (all in /root/reference/pkg/src/tritransfer):
 *   tt_locate_many        <- _kernels.locate_many            _kernels/_compiled.pyx:127-175
 *                            (the reference's only native FFI seam; same argument list)
 *   tt_locate             <- UniformGridLocator.locate_many   locate.py:76-88 (d = 2, 3)
 *   tt_nearest / tt_snap  <- UniformGridLocator.nearest_element locate.py:97-127 and the
 *                            snap branch of MeshBackedField    montecarlo.py:53-63
 *   tt_grid_count/_fill   <- UniformGridLocator.build          locate.py:33-74
 *   tt_plan_sobol         <- sobol.sobol_2d                    sobol.py:34-52 (d = 2, 3)
 *   tt_plan_pcg64         <- SamplePlan.build(mode="uniform")  montecarlo.py:100-102
 *   tt_bary_map           <- montecarlo.bary_map               montecarlo.py:68-77
 *   tt_plan_philox        <- (new) per-element counter-based streams
 *   tt_geometry           <- TriMesh areas/_bary_inv/centroids mesh.py:24-29,136-159
 *   tt_bbox               <- TriMesh.bbox                      mesh.py:110-111
 *   tt_mc_load            <- montecarlo._accumulate            montecarlo.py:110-141
 *                            (+ SourceField.__call__: AnalyticField :20-29,
 *                             MeshBackedField :49-65, NodalField.eval_in_elements fem.py:36-38)
 *   tt_mc_load_density    <- montecarlo.assemble_load_mc_weighted montecarlo.py:165-176
 *   tt_mc_cache_ids       <- MCTransferOperator.__init__ localisation transfer.py:74-87
 *   tt_mc_fold(_finish)   <- MCTransferOperator load matrix fold  transfer.py:88-110
 *   tt_spmv_rect          <- MCTransferOperator.apply R @ c      transfer.py:112-115
 *   tt_map_points         <- einsum("nj,ejd->end")             montecarlo.py:123-124
 *   tt_eval_points        <- SourceField.__call__ on given points
 *   tt_incidence_*        <- (support for np.add.at ordering)  montecarlo.py:144-147
 *   tt_reduce_nodes       <- montecarlo._reduce_to_nodes       montecarlo.py:144-147
 *   tt_mass_*             <- fem.assemble_mass_matrix          fem.py:78-110
 *   tt_pcg                <- fem.cg_solve                      fem.py:113-152
 *   tt_dpcg_*             <- fem.cg_solve, row-partitioned over GPUs (fem.py:113-152)
 *   tt_gather/scatter_rows <- (exchange plumbing of the partitioned load / solve)
 *   tt_integrate_p1       <- fem.integrate_field               fem.py:155-161
 *   tt_supermesh_integrals <- metrics.supermesh_l2/mass_error  metrics.py:35-74 (2-D, with
 *                            the intersect.py clip done on the device)
 */
#ifndef TT_B200_H
#define TT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mapped onto errors.py exceptions by the host layer) ---- */
#define TT_OK                   0
#define TT_ERR_INVALID_PARAMETER 1  /* errors.InvalidParameter   errors.py:29-30 */
#define TT_ERR_DIMENSION_MISMATCH 2 /* errors.DimensionMismatch  errors.py:37-38 */
#define TT_ERR_CUDA             3   /* launch / runtime failure (tt_last_error has text) */
#define TT_ERR_CAPACITY         4   /* a fixed per-row / per-cell capacity was exceeded */

/* ---- device status flags written by kernels ---- */
#define TT_FLAG_NONFINITE        1  /* SourceEvalFailed: non-finite f  montecarlo.py:126-127 */
#define TT_FLAG_OUTSIDE_STRICT   2  /* SourceEvalFailed: strict policy montecarlo.py:55-57 */
#define TT_FLAG_CAPACITY         4  /* row/list capacity exceeded in assembly            */
#define TT_FLAG_INVALID_DENSITY  8  /* InvalidDensity: p <= 0          montecarlo.py:129-130 */
#define TT_FLAG_NONMANIFOLD     16  /* a facet shared by > 2 elements (mesh.py:50-53)      */
#define TT_FLAG_WIDE_ROWS       32  /* an ELL column is > 32767 rows from its row: no slab  */
#define TT_FLAG_SNAPPED         64  /* tt_seed_elements: an anchor point was outside (snapped) */
#define TT_FLAG_PEER_TIMEOUT   128  /* a peer never reached a cross-GPU barrier (peer solve gave up) */

/* tt_source_t.hints */
#define TT_HINT_DEFER_SNAP       1  /* outside samples likely (the seeds saw TT_FLAG_SNAPPED):
                                       run their nearest-element searches warp-cooperatively at
                                       the end of each tile instead of on the diverged lane */

/* ---- enums ---- */
#define TT_PLAN_SHARED  0   /* one (N, k) barycentric table shared by all elements (reference) */
#define TT_PLAN_PHILOX  1   /* per-element Philox4x32-10 streams, mapped in-register          */

#define TT_SRC_EXPR     0   /* analytic field: postfix program evaluated in-kernel            */
#define TT_SRC_MESH     1   /* P1 nodal field on a source mesh + uniform-grid locator          */
#define TT_SRC_VALUES   2   /* precomputed values f[e - e_lo, j] (host black boxes)             */
#define TT_SRC_CACHED   3   /* P1 nodal field at cached source element ids (MCTransferOperator):
                               lambda_s recomputed, clipped >= 0 and renormalised, transfer.py:84-87 */

#define TT_OUTSIDE_SNAP   0
#define TT_OUTSIDE_STRICT 1

/* expression opcodes (postfix); operands: x, y, z coordinates and constants */
#define TT_OP_CONST 0
#define TT_OP_X     1
#define TT_OP_Y     2
#define TT_OP_Z     3
#define TT_OP_ADD   4
#define TT_OP_SUB   5
#define TT_OP_MUL   6
#define TT_OP_DIV   7
#define TT_OP_POW   8
#define TT_OP_NEG   9
#define TT_OP_SIN   10
#define TT_OP_COS   11
#define TT_OP_EXP   12
#define TT_OP_SQRT  13
#define TT_OP_LOG   14
#define TT_OP_TAN   15
#define TT_OP_ABS   16
#define TT_OP_SQUARE 17
#define TT_EXPR_MAX_OPS 64
#define TT_EXPR_MAX_STACK 16

/* ---- descriptors (host structs holding device pointers) ---- */
typedef struct tt_mesh {
    int32_t dim;              /* 2 = triangles, 3 = tetrahedra; k = dim + 1 vertices */
    int32_t reserved;
    int64_t n_nodes;
    int64_t n_elems;
    const double*  nodes;     /* (n_nodes, dim) row-major */
    const int32_t* elems;     /* (n_elems, k) row-major, positively oriented */
    const double*  measure;   /* (n_elems,) |area| / |volume| (may be NULL where unused) */
    const int32_t* gid;       /* optional (n_elems,) global element ids of a partition mesh:
                                 the Philox stream counter of element e is gid[e] (NULL = e) */
} tt_mesh_t;

/* Packed per-element locate record, stride TT_REC_STRIDE(dim) doubles (64 B in 2-D,
 * 128 B in 3-D: one aligned line per candidate test):
 *   [0, d*d)        binv, row-major          (mesh.py:148-159)
 *   [d*d, d*d+d)    origin = last vertex
 *   next 16 bytes   float tau (certification margin), int32 nbr[0..2]
 *   (3-D) next 4 B  int32 nbr[3]
 * nbr[i] = element across the facet opposite vertex i (-1 on the boundary); tau and
 * nbr are written by tt_grid_walk_prep (zero until then). */
#define TT_REC_STRIDE(dim) ((dim) == 2 ? 8 : 16)

typedef struct tt_grid {
    int32_t dim;
    int32_t n[3];             /* cells per axis; n[2] = 1 in 2-D; cell = (ix*n1 + iy)*n2 + iz */
    int32_t walk;             /* 1: certified facet walk before the reference scan (needs
                                 tt_grid_walk_prep on rec); 0: reference scan only */
    int32_t reserved;
    double  lo[3];            /* mesh bbox (min corner) */
    double  hi[3];            /* mesh bbox (max corner) */
    int64_t n_elems;
    const int64_t* cell_start;  /* (n0*n1*n2 + 1) CSR offsets */
    const int32_t* cell_elems;  /* ascending element ids per cell */
    const double*  rec;         /* (n_elems, TT_REC_STRIDE(dim)) packed binv/origin */
    const double*  centroids;   /* (n_elems, dim) */
    const double*  wrec;        /* optional compact walk records (n_elems, TT_WREC_STRIDE(dim)):
                                   origin (dim doubles), binv as float (dim*dim), float tau_f,
                                   int32 nbr[dim+1]; written by tt_grid_walk_prep */
} tt_grid_t;

/* compact walk record stride in doubles: 48 B (2-D), 80 B (3-D) */
#define TT_WREC_STRIDE(dim) ((dim) == 2 ? 6 : 10)

typedef struct tt_plan {
    int32_t  kind;            /* TT_PLAN_SHARED | TT_PLAN_PHILOX */
    int32_t  dim;
    int64_t  n_samples;       /* N samples per element */
    const double* lam;        /* SHARED: (N, dim+1) barycentric table */
    uint64_t seed;            /* PHILOX: key */
    const int32_t* order;     /* SHARED, optional (NULL: plan order): the order in which the fused
                                 mesh kernel takes an element's samples, with lam_walk = lam in
                                 that order (tt_plan_walk_order); ids are reported in plan order,
                                 loads differ only in the summation order */
    const double* lam_walk;
} tt_plan_t;

typedef struct tt_expr {
    int32_t n_ops;
    int32_t ops[TT_EXPR_MAX_OPS];
    double  consts[TT_EXPR_MAX_OPS];
} tt_expr_t;

typedef struct tt_source {
    int32_t kind;             /* TT_SRC_* */
    int32_t outside;          /* TT_OUTSIDE_SNAP | TT_OUTSIDE_STRICT (mesh sources) */
    int32_t dim;              /* point dimension the source is queried in (2 or 3) */
    int32_t hints;            /* TT_HINT_* bits (performance only, never results) */
    tt_expr_t expr;           /* TT_SRC_EXPR program (passed by value into the kernel) */
    tt_grid_t grid;           /* TT_SRC_MESH locator over the source mesh */
    const int32_t* src_elems; /* TT_SRC_MESH (E_s, k) */
    const double*  coeffs;    /* TT_SRC_MESH (n_s,) nodal coefficients */
    const double*  values;    /* TT_SRC_VALUES (e_hi - e_lo, N) */
    const int32_t* cached_ids;/* TT_SRC_CACHED (e_hi - e_lo, N) source element per sample */
    const int32_t* seeds;     /* TT_SRC_MESH optional (E_target, TT_SEED_ANCHORS) walk start
                                 elements per target element (tt_seed_elements), or NULL */
    const double*  elem_coeffs;/* TT_SRC_MESH/CACHED optional (E_s, 4) per-element vertex
                                 coefficients (tt_pack_coeffs); replaces src_elems+coeffs */
    const double*  elem_grad;  /* TT_SRC_MESH (E_s, 4): gradient g (dim) and the value at the
                                 origin vertex (tt_pack_grad): f = c_last + g.(x - o); required
                                 when seeds and grid.wrec are set (TT_ERR_INVALID_PARAMETER) */
} tt_source_t;

typedef struct tt_pcg_result {
    int64_t iterations;       /* iterations performed */
    double  residual;         /* final relative recurrence residual */
    double  best_residual;    /* best relative residual seen */
    int32_t converged;        /* 1 if residual <= tol */
    int32_t zero_rhs;         /* 1 if ||b|| == 0 (x = 0 returned) */
} tt_pcg_result_t;

/* ---- library ---- */
const char* tt_last_error(void);
int tt_version(void);
int tt_device_sm_count(int* out);   /* host int */

/* ---- plans ---- */
int tt_plan_sobol(int dim, int64_t count, int64_t skip, double* param /* (count, dim) */,
                  void* stream);
int tt_plan_pcg64(int dim, int64_t count, uint64_t state_hi, uint64_t state_lo,
                  uint64_t inc_hi, uint64_t inc_lo, double* param, void* stream);
int tt_bary_map(int dim, int64_t count, const double* param, double* lam /* (count, dim+1) */,
                void* stream);
int tt_plan_philox(int dim, int64_t e_lo, int64_t e_hi, int64_t n_samples, uint64_t seed,
                   double* param /* (e_hi-e_lo, N, dim) */, void* stream);

/* ---- geometry ---- */
int tt_geometry(const tt_mesh_t* mesh, double* signed_measure /* (E,) or NULL */,
                double* rec /* (E, TT_REC_STRIDE) or NULL */, double* centroids /* or NULL */,
                void* stream);
int tt_bbox(int dim, int64_t n_nodes, const double* nodes, double* out /* (2, dim): lo, hi */,
            void* stream);

/* ---- uniform-grid locator ---- */
int tt_grid_count(const tt_mesh_t* mesh, const tt_grid_t* grid /* dims + bbox used */,
                  int64_t* cell_start /* (ncells + 1): exclusive scan of counts */,
                  void* stream);
int tt_grid_fill(const tt_mesh_t* mesh, const tt_grid_t* grid /* dims, bbox, cell_start */,
                 int32_t* cell_elems, int64_t* cursor_scratch /* (ncells) */, void* stream);
int tt_locate(const tt_grid_t* grid, const double* points, int64_t count, double eps,
              int32_t* elem /* (count,) -1 = outside */, double* lam /* (count, dim+1) */,
              void* stream);
int tt_locate_many(const double* points, int64_t count, int nx, int ny,
                   const double* bbox_host /* host (xmin, ymin, xmax, ymax) */,
                   const int64_t* cell_start, const int32_t* cell_elems,
                   const double* binv /* (E,2,2) */, const double* origin /* (E,2) */,
                   double eps, int32_t* elem, double* lam /* (count,3) */, void* stream);
/* Certified facet walk: fills tau and nbr of every record from
 * the node incidence; sets TT_FLAG_NONMANIFOLD in *status for a non-manifold mesh. */
int tt_grid_walk_prep(const tt_mesh_t* mesh, const int64_t* inc_start, const int32_t* inc,
                      double eps, double* rec, double* wrec /* or NULL */, int32_t* status,
                      void* stream);
/* seeds[(e - e_lo)*TT_SEED_ANCHORS + s] = source element containing anchor point s of the
 * target element (reference scan, snapped when outside): s = 0 the centroid c, s = 1 + i the
 * point (v_i + c)/2, then 16 - (dim+2) k-means anchors (scripts/seed_anchors.py).  Walk
 * starts: a sample starts at its nearest anchor's element. */
#define TT_SEED_ANCHORS 48
int tt_seed_elements(const tt_grid_t* grid, const tt_mesh_t* target, int64_t e_lo,
                     int64_t e_hi, int32_t* seeds, int32_t* status /* TT_FLAG_SNAPPED, or NULL */,
                     void* stream);
int tt_nearest(const tt_grid_t* grid, const double* points, int64_t count,
               int32_t* elem /* out */, void* stream);
int tt_snap(const tt_grid_t* grid, const double* points, int64_t count,
            int32_t* elem /* in/out: -1 entries replaced */, double* lam /* in/out */,
            void* stream);

/* ---- Monte-Carlo load ---- */
int tt_map_points(const tt_mesh_t* target, int64_t e_lo, int64_t e_hi, const tt_plan_t* plan,
                  double* points /* (e_hi-e_lo, N, dim) */, void* stream);
int tt_eval_points(const tt_source_t* src, const double* points, int64_t count,
                   double* values, int32_t* status, void* stream);
/* order[N] = the shared plan's sample indices grouped by nearest walk anchor (stable) and
 * lam_walk (N, dim+1) = lam in that order, so a lane group of the fused kernel starts its walks
 * from the same seed element (1 <= N <= 4096) */
int tt_plan_walk_order(int dim, int64_t n_samples, const double* lam, int32_t* order, double* lam_walk,
                       void* stream);
int tt_mc_load(const tt_mesh_t* target, int64_t e_lo, int64_t e_hi, const tt_plan_t* plan,
               const tt_source_t* src,
               double* contrib /* (e_hi-e_lo, k) or NULL */,
               double* b /* (n_nodes) atomically accumulated when contrib == NULL */,
               int32_t* status, void* stream);
/* tt_mc_load with the contribution buffer transposed when contrib_ld > 0:
 * contrib[a*contrib_ld + (e - e_lo)] (contrib_ld >= e_hi - e_lo; the node gather's layout,
 * tt_reduce_nodes_ld); contrib_ld = 0 is tt_mc_load's (e_hi - e_lo, k) row-major buffer. */
int tt_mc_load_ld(const tt_mesh_t* target, int64_t e_lo, int64_t e_hi, const tt_plan_t* plan,
                  const tt_source_t* src, double* contrib, int64_t contrib_ld, double* b,
                  int32_t* status, void* stream);

/* importance-weighted load (montecarlo.py:165-176): contrib[e, a] = sum_j f_j / (N p_ej) lambda_ja
 * with the caller's densities p (e_hi-e_lo, N) for a shared plan; p <= 0 sets
 * TT_FLAG_INVALID_DENSITY, non-finite f TT_FLAG_NONFINITE */
int tt_mc_load_density(const tt_mesh_t* target, int64_t e_lo, int64_t e_hi, const tt_plan_t* plan,
                       const tt_source_t* src, const double* density, double* contrib,
                       int32_t* status, void* stream);

int tt_mc_cache_ids(const tt_mesh_t* target, int64_t e_lo, int64_t e_hi, const tt_plan_t* plan,
                    const tt_grid_t* grid, const int32_t* seeds /* (E_target, TT_SEED_ANCHORS) or NULL */,
                    int32_t* ids /* (e_hi-e_lo, N): located or snapped */, void* stream);

/* out[e*4 + i] = coeffs[elems[e*k + i]] (i < k, zero padded): one aligned 32-byte record
 * per source element, gathered once per coefficient update. */
int tt_pack_coeffs(const tt_mesh_t* src, const double* coeffs, double* out, void* stream);

/* out[e*4 ..] = (g, c_last): the P1 field's gradient on element e and its value at the
 * last vertex (the walk record's origin): g solves E g = d, rows e_i = v_i - v_last,
 * d_i = c_i - c_last, from the vertex coordinates (src->nodes, src->elems). */
int tt_pack_grad(const tt_mesh_t* src, const double* coeffs, double* out, void* stream);

/* MCTransferOperator's sparse load matrix R (n_t x n_s, transfer.py:56-110) folded on
 * the device from the cached sample ids (shared plans): tt_mc_fold computes it into an
 * opaque handle and returns nnz; tt_mc_fold_finish writes the CSR (row_ptr n_t+1, cols,
 * vals) and frees the handle.  Deterministic (stable sorts, fixed reductions). */
int tt_mc_fold(const tt_mesh_t* target, const tt_plan_t* plan, const tt_mesh_t* src,
               const double* src_rec, const int32_t* ids /* (E_t, N) */, int64_t* nnz_out /* host */,
               void** handle_out /* host */, void* stream);
int tt_mc_fold_finish(void* handle, int64_t* row_ptr, int32_t* cols, double* vals, void* stream);
/* y = A x for a rectangular CSR (one warp per row) */
int tt_spmv_rect(int64_t n_rows, const int64_t* row_ptr, const int32_t* cols, const double* vals,
                 const double* x, double* y, void* stream);

/* ---- node reduction / incidence (deterministic np.add.at order) ---- */
int tt_incidence_count(const tt_mesh_t* mesh, int64_t* inc_start /* (n_nodes+1) */,
                       void* stream);
int tt_incidence_fill(const tt_mesh_t* mesh, const int64_t* inc_start,
                      int32_t* inc /* (E*k) entries e*k+a, ascending per node */,
                      int64_t* cursor_scratch /* (n_nodes) */, void* stream);
/* b[n] = sum of contrib[(e - e_lo)*k + a] over node n's incidences e*k + a with
 * e_lo <= e < e_hi, in ascending order from 0.0 (np.add.at's order); k = 1, 3 or 4.  inc is
 * read in aligned 16-byte chunks: it must be 16-byte aligned and readable to a multiple of 4
 * entries. */
int tt_reduce_nodes(int64_t n_nodes, int k, const int64_t* inc_start, const int32_t* inc,
                    int64_t e_lo, int64_t e_hi, const double* contrib, double* b,
                    void* stream);
/* The same sum over a transposed contribution buffer (contrib_ld > 0, k = 3 or 4):
 * contrib[a*contrib_ld + (e - e_lo)], the layout tt_mc_load_ld writes for it; contrib_ld = 0
 * is tt_reduce_nodes. */
int tt_reduce_nodes_ld(int64_t n_nodes, int k, const int64_t* inc_start, const int32_t* inc,
                       int64_t e_lo, int64_t e_hi, const double* contrib, int64_t contrib_ld,
                       double* b, void* stream);

/* ---- P1 mass matrix (CSR, exactly symmetric) ---- */
int tt_mass_pattern(const tt_mesh_t* mesh, const int64_t* inc_start, const int32_t* inc,
                    int64_t* row_ptr /* (n_nodes+1) exclusive scan of row lengths */,
                    int32_t* status, void* stream);
int tt_mass_fill(const tt_mesh_t* mesh, const int64_t* inc_start, const int32_t* inc,
                 const double* local_host /* host (k, k) reference-element mass */,
                 const int64_t* row_ptr, int32_t* cols, double* vals, void* stream);

/* ---- Jacobi-preconditioned CG (single cooperative launch) ---- */
int64_t tt_pcg_workspace_doubles(int64_t n);
int tt_pcg(int64_t n, const int64_t* row_ptr, const int32_t* cols, const double* vals,
           const double* b, double tol, int64_t maxiter, double* x, double* best_x,
           double* work /* tt_pcg_workspace_doubles(n) */, tt_pcg_result_t* result /* device */,
           void* stream);
/* ELL form of the mass matrix (width 16, or 8 when every row has <= 8 entries -- the 2-D
 * meshes; padding (row, 0.0)) and the PCG over it; the same recurrence as tt_pcg with the
 * row-pointer round trip removed from every SpMV row.  TT_FLAG_CAPACITY in *status when a
 * row has more than `width` entries (use tt_pcg then); TT_FLAG_WIDE_ROWS when a column is
 * more than 32767 rows from its row (no slab). */
int tt_csr_to_ell(int64_t n, const int64_t* row_ptr, const int32_t* cols, const double* vals,
                  int width, int32_t* ell_cols /* (n, width) */, double* ell_vals /* (n, width) */,
                  double* diag /* (n,) */, int32_t* status, void* stream);
int tt_pcg_ell(int64_t n, int width, const int32_t* ell_cols, const double* ell_vals, const double* diag,
               const double* b, double tol, int64_t maxiter, double* x, double* best_x,
               double* work /* tt_pcg_workspace_doubles(n) */, tt_pcg_result_t* result,
               void* stream);
/* The same PCG with each block's rows of the ELL matrix held in shared memory for the whole
 * solve (80 B per row per 8 columns): all of them when they fit (n up to ~207k rows at width
 * 16, ~415k at width 8), else the first part of every block's range (at least 1/2 of it;
 * TT_PCG_SLAB_MIN_FRAC) with the rest streamed from L2/HBM.  Precondition: tt_csr_to_ell did
 * not set TT_FLAG_WIDE_ROWS.  Returns TT_ERR_CAPACITY, launching nothing, when too few rows
 * fit (the caller then uses tt_pcg_ell). */
int tt_pcg_ell_slab(int64_t n, int width, const int32_t* ell_cols, const double* ell_vals,
                    const double* diag, const double* b, double tol, int64_t maxiter, double* x,
                    double* best_x, double* work /* tt_pcg_workspace_doubles(n) */,
                    tt_pcg_result_t* result, void* stream);
/* The same solve with the pipelined (Ghysels-Vanroose) form of the recurrence: the same Krylov
 * iterates, stopping rule and best-iterate tracking in exact arithmetic, ONE grid barrier per
 * iteration.  For matrices whose Jacobi-preconditioned condition number is small (P1 mass
 * matrices: <= 4 in 2-D, <= 5 in 3-D), where its rounding matches the textbook recurrence's.
 * Workspace tt_pcg_workspace_doubles(n); TT_ERR_CAPACITY as tt_pcg_ell_slab. */
int tt_pcg_ell_slab_pipelined(int64_t n, int width, const int32_t* ell_cols, const double* ell_vals,
                              const double* diag, const double* b, double tol, int64_t maxiter, double* x,
                              double* best_x, double* work, tt_pcg_result_t* result, void* stream);
int tt_spmv(int64_t n, const int64_t* row_ptr, const int32_t* cols, const double* vals,
            const double* x, double* y, void* stream);

/* ---- multi-GPU: row-partitioned PCG and exchange helpers (tt_dist.cu) ---- */
/* One rank's part of the distributed Jacobi PCG (fem.py:113-152 in its Chronopoulos-Gear
 * form: one all-reduce of 3 scalars per iteration).  Rows = the rank's own target nodes; the
 * local vector u is (n_ext = own + halo) long, halo entries received from their owners each
 * iteration.  Host sequence:
 *   tt_dpcg_start -> halo exchange of send_buf into u[n_own:] -> tt_dpcg_spmv(parity 0) ->
 *   all-reduce(sum) of sums[0..3);  then per iteration k (q = k & 1):
 *   tt_dpcg_update(q) -> halo exchange -> tt_dpcg_spmv(q ^ 1) -> all-reduce of sums;
 *   tt_dpcg_finish.  The scalars stay on the device (state); every call is a no-op once the
 *   solve is done, so iterations can be issued in fixed chunks (e.g. one CUDA graph). */
#define TT_DPCG_STATE_BYTES 256
typedef struct tt_dpcg {
    int64_t n_own;            /* owned rows */
    int64_t n_ext;            /* local vector length: owned + halo */
    int32_t width;            /* ELL width 8 | 16 */
    int32_t reserved;
    const int32_t* ell_cols;  /* (n_own, width) local column ids into u (padding: own row, 0.0) */
    const double*  ell_vals;  /* (n_own, width) */
    const double*  diag;      /* (n_own,) */
    const double*  b;         /* (n_own,) */
    double* x; double* best_x; double* r; double* w; double* p; double* s; double* dinv; /* (n_own,) */
    double* u;                /* (n_ext,) */
    const int64_t* send_start;/* (n_own + 1,) CSR: row i's u goes to send_buf[send_pos[k]], */
    const int64_t* send_pos;  /*   k in [send_start[i], send_start[i+1]) (one slot per peer) */
    int64_t n_send;
    double* send_buf;         /* (n_send,) grouped by peer */
    double* part;             /* tt_dpcg_part_doubles() scratch */
    double* sums;             /* (3,) local sums (r.u, w.u, r.r): all-reduce them in place */
    double* state;            /* TT_DPCG_STATE_BYTES of device scalar state */
    double  tol;
    int64_t maxiter;
} tt_dpcg_t;
int64_t tt_dpcg_part_doubles(void);
int tt_dpcg_start(const tt_dpcg_t* a, void* stream);
int tt_dpcg_update(const tt_dpcg_t* a, int parity, void* stream);
int tt_dpcg_spmv(const tt_dpcg_t* a, int parity, void* stream);
/* the result record (device): iterations, residual, best residual, converged, zero_rhs */
int tt_dpcg_finish(const tt_dpcg_t* a, tt_pcg_result_t* result, void* stream);
/* Peer-memory forms (NVLink symmetric memory, no NCCL on the data path):
 * tt_reduce_nodes_ranked -- the owner-side node reduction reading each incidence's
 *   contribution straight from the rank that computed it: b[n] = sum over q in
 *   [inc_start[n], inc_start[n+1]) of ptrs[inc_rank[q]][inc_entry[q]], in that order.
 * tt_dpcg_peer_solve -- the whole distributed PCG as ONE cooperative launch per rank: u of the
 *   owned rows lives in the rank's symmetric buffer sym[rank] (u_len doubles, then 2 x 3
 *   partial-sum slots); halo column h is read from sym[halo_owner[h]][halo_row[h]]; two
 *   cross-GPU barriers per iteration over the signal pads (release/acquire at system scope;
 *   *epoch persists across solves); every rank sums the world's partials in rank order.
 *   A barrier that waits > ~20 s sets TT_FLAG_PEER_TIMEOUT in *status and returns unconverged. */
int tt_reduce_nodes_ranked(int64_t n_nodes, const int64_t* inc_start, const int32_t* inc_rank,
                           const int32_t* inc_entry, const double* const* ptrs, double* b, void* stream);
int tt_dpcg_peer_solve(const tt_dpcg_t* a, const int32_t* halo_owner, const int32_t* halo_row,
                       double* const* sym, uint32_t* const* pads, int64_t u_len, int rank, int world,
                       uint32_t* epoch, int32_t* status, tt_pcg_result_t* result, void* stream);
/* dst[t, :] = src[idx[t], :] and dst[idx[t], :] = src[t, :] for rows of k doubles */
int tt_gather_rows(int64_t n, int k, const int64_t* idx, const double* src, double* dst, void* stream);
int tt_scatter_rows(int64_t n, int k, const int64_t* idx, const double* src, double* dst, void* stream);

/* ---- reporting ---- */
int tt_integrate_p1(const tt_mesh_t* mesh, const double* coeffs, double* out /* device scalar */,
                    void* stream);

/* Supermesh integrals of two P1 fields on triangle meshes (metrics.py:35-74 over the
 * intersection polygons of intersect.py:60-80, clipped on the device): per target element
 * (E_t, 6) = [int (fs-ft)^2, int fs^2, int fs, int ft, covered area, covered / |t|] and the
 * totals (6,) = column sums (fixed order), last = min covered fraction.  Polygons of area
 * <= sliver_rel |t| are dropped (intersect.py:21). */
int tt_supermesh_integrals(const tt_mesh_t* target, const double* t_coeffs, const tt_mesh_t* source,
                           const double* s_coeffs, const tt_grid_t* src_grid, double sliver_rel,
                           double* per_elem, double* totals, void* stream);

/* ---- measurement helpers ---- */
int tt_fp64_peak_probe(int64_t iters, double* sink /* (blocks*threads) */, int* blocks_out,
                       int* threads_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TT_B200_H */
