/*
 * agipc.h -- C ABI of the B200-native AGIPC coarsening path (arXiv 2605.04773).
 *
 * One Newton iteration of AGIPC (main Alg 1 lines 8-10):
 *   1. agipc_tag_edges        edge tags tau_e from the Green-strain increment (Eq 3)
 *   2. agipc_build_map        fine->coarse map by group bit-hashing, prefix sum and
 *                             level-wise recursion (supp Alg S1/S2)
 *   3. agipc_assemble_coarse  DoF classification + reorder (supp Alg S3) and the
 *                             Galerkin coarse Hessian / gradient H_c = U H U^T, g_c = U g
 *                             with affine 12-DoF nodes (supp Alg S4, Eq S2/S3, P:258-319;
 *                             main Eq 4)
 *   4. agipc_pcg_solve        block-Jacobi PCG on the coarse system
 *   5. agipc_prolongate       d_f = U^T d_c back to the fine nodes (NEXT#1)
 * and the rows SURVEY 8(f) ranks next:
 *   agipc_bsr_upper / agipc_bsr_expand_upper / agipc_pcg_solve_sym
 *                             symmetric (diagonal + upper) storage (NEXT#2)
 *   agipc_triplet_plan / agipc_triplet_reduce
 *                             fine-level hash reduction of element triplets (NEXT#3)
 *   agipc_tag_shells / agipc_tag_rods
 *                             step 1 for triangles and edges (NEXT#4)
 * plus the partitioned multi-GPU pieces (agipc_gather_rows, agipc_coarse_halo,
 * agipc_assemble_halo, agipc_dpcg_*) and agipc_set_values_event (upload overlap).
 *
 * Conventions (all entry points):
 *  - Array arguments are DEVICE pointers owned by the caller (e.g. PyTorch CUDA tensors,
 *    C-contiguous) unless marked [host].  Inputs are never written.  The library keeps no
 *    caller pointer between calls.
 *  - Every kernel is enqueued on the handle's stream (agipc_set_stream; default: the
 *    legacy default stream).  Calls that return a data-dependent size in a [host] argument
 *    synchronise that stream before returning; the others are asynchronous.  build_map,
 *    assemble_coarse and the PCG status polls wait by spinning on a CUDA event (the calling
 *    thread stays busy; no blocking-sync wake-up latency while the GPU idles).
 *    assemble_coarse returns once the sizes are known; its numeric pass is still running on
 *    the stream (and on an internal second stream joined back into it).
 *  - Errors are returned as agipc_status, never thrown or aborted; agipc_last_error()
 *    returns a human-readable message for the last failing call on that handle.
 *  - Index types: node, slot and column ids are int32 (sizes >= 2^31-1 return
 *    AGIPC_ERANGE); row pointers are int64.
 *  - Thread safety: one handle per host thread / stream.  Handles on different devices
 *    are independent.
 *  - Precision: all floating point is IEEE fp64 ("double-precision").
 */
#ifndef AGIPC_H_
#define AGIPC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define AGIPC_API __attribute__((visibility("default")))
#else
#define AGIPC_API
#endif

#define AGIPC_VERSION_MAJOR 0
#define AGIPC_VERSION_MINOR 1

typedef struct agipc_handle_s *agipc_handle;

typedef enum {
  AGIPC_OK = 0,
  AGIPC_EINVAL = 1,       /* null pointer, group_size outside [1,32], negative size, bad map  */
  AGIPC_ERANGE = 2,       /* an index does not fit in int32                                   */
  AGIPC_ENOSPACE = 3,     /* output capacity too small; required sizes were written back     */
  AGIPC_ECUDA = 4,        /* a CUDA runtime call failed (message in agipc_last_error)         */
  AGIPC_ENCCL = 5,        /* NCCL missing or an NCCL call failed (multi-GPU path)             */
  AGIPC_EDEGENERATE = 6,  /* a tet with det(D_m) == 0 at rest                    */
  AGIPC_ESINGULAR = 7,    /* a block-Jacobi diagonal block is missing or singular     */
  AGIPC_EINDEFINITE = 8,  /* p^T A p <= 0 in PCG                                      */
  AGIPC_EBREAKDOWN = 9,   /* NaN/Inf in PCG                                           */
  AGIPC_NOT_CONVERGED = 10 /* max_iters reached; x holds the last iterate (not fatal)         */
} agipc_status;

/* ---- handle ------------------------------------------------------------------------- */
AGIPC_API agipc_status agipc_create(agipc_handle *h, int cuda_device);
AGIPC_API agipc_status agipc_destroy(agipc_handle h);
/* stream: a cudaStream_t passed as void* (e.g. torch.cuda.current_stream().cuda_stream). */
AGIPC_API agipc_status agipc_set_stream(agipc_handle h, void *stream);
/* One-shot: the next agipc_assemble_coarse makes its numeric phase (the only part that reads
 * H_fine values and g_fine) wait for this CUDA event (cudaEvent_t as void*; NULL clears), so an
 * upload of the values on another stream overlaps steps 1-2 AND the classification + symbolic
 * phases of step 3. */
AGIPC_API agipc_status agipc_set_values_event(agipc_handle h, void *event);
AGIPC_API const char *agipc_last_error(agipc_handle h);
AGIPC_API const char *agipc_status_string(agipc_status s);
AGIPC_API void agipc_version(int *major /*[host]*/, int *minor /*[host]*/);
/* Options (agipc_set_option):
 *  AGIPC_OPT_CHECK_SYMMETRY (0/1, default 0): agipc_assemble_coarse first checks the precondition
 *    it relies on (R22: H_fine bitwise symmetric, B_ji == B_ij^T for every stored block,
 *    the transposed block present) in one extra pass + host sync, and returns AGIPC_EINVAL with the
 *    number of violations if it fails.
 *  AGIPC_OPT_L2_PERSIST (bytes, default 0): sets the device's persisting-L2 limit ONCE, now (the
 *    only device-wide setting the library ever changes, and only on this request), and lets the
 *    PCG solves place their vector arena in a persisting access-policy window of that size;
 *    the persisting lines are released after every solve.  0 = plain caching (no window).
 *  AGIPC_OPT_COMM_ALWAYS (0/1, default 0): issue the NCCL all-reduces of agipc_dpcg_solve even on
 *    a one-rank communicator (where the sum is the identity and they are skipped) -- lets a
 *    single-GPU test run the captured NCCL path.
 *  AGIPC_OPT_DETERMINISTIC (0/1, default 0): the 12-DoF (large) coarse rows are assembled without
 *    fp64 atomics -- every 32-children chunk writes its partial diagonal block, g_c part and one
 *    record per interface block, and a fixed-order reduction sums them -- so H_c and g_c (and with
 *    them the PCG iterates and iteration counts) are bitwise reproducible run to run.  Default: the
 *    faster atomic accumulation, reproducible to rounding (inside the 1e-12 |.|-bound contract).
 *    The coarse PCG is bitwise reproducible either way (per-slice p.q partials, fixed-order sums). */
#define AGIPC_OPT_CHECK_SYMMETRY 1
#define AGIPC_OPT_L2_PERSIST 2
#define AGIPC_OPT_COMM_ALWAYS 3
#define AGIPC_OPT_DETERMINISTIC 4
AGIPC_API agipc_status agipc_set_option(agipc_handle h, int option, int64_t value);

/* Workspace.  By default the handle cudaMallocs grow-only named scratch buffers on first use.
 * agipc_set_workspace hands it a caller-owned device arena instead (e.g. a torch uint8 tensor;
 * 256-byte aligned base): every scratch buffer is then carved from it by a bump pointer and the
 * library never allocates device memory; a call whose scratch does not fit returns
 * AGIPC_ENOSPACE (nothing is freed or moved while a call runs) -- register a larger arena and
 * retry.  set_workspace synchronises the stream, releases the internal buffers and re-places all
 * scratch on next use; ws = NULL returns to internal allocation.  The arena must stay valid
 * until the next set_workspace / destroy.  EINVAL during a split-phase distributed solve.
 * agipc_workspace_size: bytes to register -- the largest of (the sum of the largest size every
 * scratch buffer of this handle has needed so far) and an a-priori estimate for one Newton step
 * (tag, map, assemble, coarse PCG) on a mesh of these sizes. */
AGIPC_API agipc_status agipc_workspace_size(agipc_handle h, int64_t n_nodes, int64_t n_tets, int64_t nnz_adj,
                                            int64_t nnzb_fine, size_t *bytes /*[host]*/);
AGIPC_API agipc_status agipc_set_workspace(agipc_handle h, void *ws, size_t bytes);

/* Number of kernels this handle has enqueued since creation ([host] counter). */
AGIPC_API int64_t agipc_kernel_launches(agipc_handle h);

/* Profiling.  agipc_profile(h, 1) resets and enables CUDA-event timing on the streams the
 * kernels are launched on: one interval per entry-point call (tag_edges, build_map,
 * assemble_coarse, pcg_setup, pcg_solve) and, inside the PCG graph, one interval per kernel
 * launch of every 8th iteration (pcg_spmv = K1 with the fused p update, pcg_update = K2;
 * launches that exit early after convergence are not counted).  agipc_profile_read synchronises pending events and fills
 * up to cap entries; returns the number written (or the number available if out == NULL). */
typedef struct {
  char name[32];
  int64_t count;     /* timed intervals */
  double total_ms;   /* summed duration */
} agipc_profile_entry;
AGIPC_API agipc_status agipc_profile(agipc_handle h, int enable);
AGIPC_API int agipc_profile_read(agipc_handle h, agipc_profile_entry *out /*[host]*/, int cap);

/* ---- static fine mesh ("static underlying topology"; P:838 precomputed adjacency) -- */
typedef struct {
  int64_t n_nodes;          /* N                                                              */
  int64_t n_tets;           /* T                                                              */
  int64_t nnz_adj;          /* 2E: directed adjacency slots                                   */
  const int32_t *tets;      /* [T][4] node ids; D_m = [X_b-X_a | X_c-X_a | X_d-X_a]           */
  const int64_t *adj_ptr;   /* [N+1] symmetric adjacency, no self loops                       */
  const int32_t *adj_nbr;   /* [2E] neighbours, ascending within a row                        */
  const int32_t *tet_slots; /* [T][12] for local edge e in (01,02,03,12,13,23): the adjacency
                               slot of (u->v) at 2e and of (v->u) at 2e+1; -1 = no slot      */
  const double *x_rest;     /* [N(+ghosts)][3] rest positions X; also X_bar = (x,y,z,1), Eq 4 */
} agipc_mesh;
/* Partitioned meshes (multi-GPU): a rank passes its LOCAL mesh -- N = owned nodes
 * 0..N-1, ghost nodes N.. (non-owned vertices of the tets that touch an owned node).  tets may
 * reference ghosts, and x_rest / x_prev / x_cur then cover N + n_ghost rows; adjacency rows
 * and neighbours are owned nodes only; tet_slots is -1 for an edge with a ghost end.  Every
 * step below then works on the rank's own rows (rank-local recursion, reading R24). */

/* Block sparse row matrix with 3x3 blocks (full storage, ascending columns per row). */
typedef struct {
  int64_t n_rows;           /* block rows (nodes or slots)                                    */
  int64_t nnzb;             /* stored blocks                                                  */
  const int64_t *row_ptr;   /* [n_rows+1]                                                     */
  const int32_t *col;       /* [nnzb] ascending within a row                                  */
  const double *val;        /* [nnzb][3][3] row-major blocks                                  */
} agipc_bsr;

/* ---- step 1: edge tags ----------------------------------------------------------------
 * main Sec 4.2 Eq 3, supp Sec 1.1.  For every tet t:
 *   F = D_s D_m^-1 (D_m^-1 = adj(D_m) * (1/det D_m)), G = 1/2 (F^T F - I) at x_prev and x_cur,
 *   n_t = ||G(x_cur) - G(x_prev)||_F, flagged iff n_t > threshold (strict).
 * slot_tags[s] = 0 if the edge of adjacency slot s belongs to a flagged tet, else 1
 * (both directed slots of an edge agree).  Fixed fp64 operation order without FMA
 * contraction (R12), so tags are reproducible bit for bit.
 *   x_prev, x_cur : [N][3] iterates x_{i-1}, x_i (at the first Newton iteration pass x^t twice)
 *   slot_tags     : out [nnz_adj] uint8
 *   tet_norm      : out [T] n_t, nullable
 *   n_flagged     : [host] out number of flagged tets, nullable (non-null => synchronises)
 * Errors: EINVAL (null inputs); EDEGENERATE (a tet has det D_m == 0) is reported only when
 * n_flagged is non-null (the call then synchronises); an asynchronous call treats such a
 * tet as flagged (its edges are protected). */
AGIPC_API agipc_status agipc_tag_edges(agipc_handle h, const agipc_mesh *mesh, const double *x_prev,
                             const double *x_cur, double threshold, uint8_t *slot_tags,
                             double *tet_norm, int64_t *n_flagged);

/* ---- step 2: fine -> coarse map -------------------------------------------------------
 * supp Alg S1/S2 applied level-wise, readings R1-R8:
 * nodes are split into contiguous groups of group_size; inside a group the tagged edges
 * are OR-propagated into 32-bit connectivity hashes; a component's local index is the
 * rank of its first set bit among the group's elected lanes; an exclusive prefix sum of
 * per-group counts gives global ids.  The surviving tagged edges mapped through the level
 * map form the next level's graph; repeat until a level merges nothing or max_levels
 * levels ran.  Result: map[f] = rank of f's aggregate ordered by its minimum fine node.
 *   slot_tags  : [nnz_adj] 1 collapsible / 0 protected; must be symmetric
 *   group_size : 1..32 (32 = one warp per group)
 *   max_levels : 0 = until no merge
 *   map        : out [N] int32 coarse id in [0, n_coarse)
 *   agg_size   : out [N] capacity, first n_coarse entries = fine nodes per aggregate; nullable
 *   info       : [host] out; synchronises the stream. */
typedef struct {
  int64_t n_coarse;
  int32_t n_levels;          /* passes run, including the final no-merge pass               */
  int32_t reserved;
  int64_t level_n[64];       /* node count after each of the first 64 levels               */
  int64_t n_cross_edges;     /* tagged fine edges between level-0 groups                    */
} agipc_map_info;

AGIPC_API agipc_status agipc_build_map(agipc_handle h, const agipc_mesh *mesh, const uint8_t *slot_tags,
                             int group_size, int max_levels, int32_t *map, int32_t *agg_size,
                             agipc_map_info *info);

/* ---- step 3: classification + Galerkin assembly ----------------------------------------
 * supp Alg S3: a coarse node is 12-DoF iff it aggregates more than
 * affine_threshold fine nodes (32); stable reorder, 3-DoF nodes first.
 * Expanded slots (Eq S2/S3, reading R14): slot(c) = c for c < n3,
 * slot(c,p) = n3 + 4(c-n3) + p for a 12-DoF node, p = 0..3 (rows of X_bar (x) I3).
 * H_c[slot(a,p), slot(b,q)] = sum over stored fine blocks (i,j) with new_map(i)=a,
 * new_map(j)=b of w_i[p] w_j[q] B_ij, w = X_bar for 12-DoF parents, 1 otherwise
 * (Alg S4 + Eq 4; == U H_f U^T).  g_c[slot(a,p)] = sum w_f[p] g_f[f].
 * Output is canonical BSR over n_slots block rows with ascending columns and a
 * structural pattern (a block exists iff at least one fine block maps to it, R17).
 *   H_fine : fine BSR over N rows; must be symmetric (B_ji = B_ij^T, as the SPD proxy H of
 *            P:786 is): a mixed 3-DoF/12-DoF block pair is computed once and mirrored.
 *   g_fine : [N][3], nullable (then out->g_c is not written)
 *   out    : sizes are written back; if cap_slots < n_slots or cap_nnzb < nnzb the call
 *            returns AGIPC_ENOSPACE with n3/n12/n_slots/nnzb filled and nothing else
 *            written.  new_map is always written.  Synchronises the stream. */
typedef struct {
  int64_t n3, n12, n_slots, nnzb; /* [host] out                                             */
  int64_t cap_slots, cap_nnzb;    /* [host] in: capacities of row_ptr/g_c and col/val       */
  int32_t *new_map;               /* out [N] reordered coarse id of every fine node          */
  int64_t *row_ptr;               /* out [cap_slots+1]                                       */
  int32_t *col;                   /* out [cap_nnzb]                                          */
  double *val;                    /* out [cap_nnzb][3][3]                                    */
  double *g_c;                    /* out [cap_slots][3], nullable                            */
} agipc_coarse;

AGIPC_API agipc_status agipc_assemble_coarse(agipc_handle h, const agipc_mesh *mesh, const int32_t *map,
                                   int64_t n_coarse, int64_t affine_threshold,
                                   const agipc_bsr *H_fine, const double *g_fine,
                                   agipc_coarse *out);

/* ---- step 4: block-Jacobi PCG ----------------------------------------------------------
 * Preconditioned CG (textbook, reading R20) on A x = b with D^-1 = inverse of each row's
 * 3x3 diagonal block ("3x3 block Jacobi").  Stops when ||r_k||_2 <= rel_tol ||b||_2
 * on the recurrence residual or after max_iters iterations.  Convergence is
 * tested on the device every iteration; the host polls every check_every iterations
 * (the iterations in between are captured in one CUDA graph).
 *   A       : SPD BSR (n_rows slots)
 *   b       : [n_rows][3];  x : [n_rows][3] in: x0 (ignored if zero_x0), out: solution
 *   zero_x0 : nonzero = start from x0 = 0 (the coarse solve of each Newton step)
 *   stats   : [host] out; synchronises the stream.
 * The coarse Newton direction of P:752 is d_c = -x for b = g_c (CG is linear in b). */
typedef struct {
  int32_t iters;
  int32_t status;             /* agipc_status of the solve                                  */
  double rel_residual;        /* ||r||_2 / ||b||_2 at exit (recurrence residual)            */
  double b_norm;
} agipc_pcg_stats;

AGIPC_API agipc_status agipc_pcg_solve(agipc_handle h, const agipc_bsr *A, const double *b, double *x,
                                       int zero_x0, double rel_tol, int max_iters, int check_every,
                                       agipc_pcg_stats *stats);

/* agipc_pcg_set_static: register A's pattern (row_ptr, col, n_rows, nnzb) as STATIC -- the caller
 * promises that the contents behind these two pointers do not change while it is registered (the
 * fine mesh topology is static).  Solves on a matrix with exactly these pointers and sizes
 * keep the SELL layout of the first such solve (segments, sorted windows, slices) and only refill
 * the values: NEXT#1's post-coarsening fine solve every Newton step.  A = NULL clears.
 * Without a registration, solves of at most 32 iterations stream the BSR as it is (no re-layout). */
AGIPC_API agipc_status agipc_pcg_set_static(agipc_handle h, const agipc_bsr *A);

/* ---- NEXT#2: symmetric (diagonal + upper-triangular) storage -----------------------------
 * "both FEM elasticity and IPC contact/friction Hessians are symmetric, so we store and
 * accumulate only the diagonal and upper-triangular entries ... This reduces memory traffic ...
 * for both the fine-mesh Hessian and the subsequent coarse system" (main Sec 6).
 *
 * agipc_bsr_upper: U = the blocks of a full-storage BSR A (columns ascending per row) with
 *   col >= row, same order.  row_ptr : out [n_rows+1]; col : out [cap_nnzb]; val : out
 *   [cap_nnzb][3][3].  *nnzb_upper [host] = the block count; ENOSPACE (row_ptr written) if it
 *   exceeds cap_nnzb -- call again with a larger capacity.  Synchronises the stream.
 *
 * agipc_pcg_solve_sym: agipc_pcg_solve (same stopping rule, preconditioner, stats and errors)
 *   whose SpMV streams only the diagonal + upper blocks once per iteration and applies each
 *   block twice: q_i += A_ij p_j and, for j > i, q_j += A_ij^T p_i.  A must be symmetric
 *   (A_ji = A_ij^T; not checked).  storage:
 *     AGIPC_STORAGE_FULL  : A in full storage, every block streamed (= agipc_pcg_solve);
 *     AGIPC_STORAGE_SYM   : A in full storage; the per-solve re-layout keeps col >= row only;
 *     AGIPC_STORAGE_UPPER : A holds only col >= row (e.g. from agipc_bsr_upper); a block
 *                           below the diagonal returns EINVAL.
 *   The scatter sums in shared memory and L2 in no fixed order, so q (and the iterate) is
 *   reproducible only up to rounding; the SPD/tolerance contract is that of agipc_pcg_solve. */
#define AGIPC_STORAGE_FULL 0
#define AGIPC_STORAGE_SYM 1
#define AGIPC_STORAGE_UPPER 2
AGIPC_API agipc_status agipc_bsr_upper(agipc_handle h, const agipc_bsr *A, int64_t cap_nnzb, int64_t *row_ptr,
                                       int32_t *col, double *val, int64_t *nnzb_upper /*[host]*/);
/* agipc_bsr_expand_upper: the fine Hessian arrives in symmetric storage and the
 *   assembly reads full rows: val (out, [full->nnzb][3][3]) on the full pattern (full->row_ptr,
 *   full->col; full->val unused) gets U_ij for col >= row and U_ji^T below the diagonal.  The
 *   full pattern must be the symmetric closure of U's (same column order, every diagonal
 *   block stored first in its U row).  check != 0: the kernel counts pattern mismatches and
 *   the call synchronises the stream and returns EINVAL if any (val is then unreliable);
 *   check == 0: no host round trip (for a pattern pair validated once -- the topology is
 *   static), mismatching blocks are skipped silently. */
AGIPC_API agipc_status agipc_bsr_expand_upper(agipc_handle h, const agipc_bsr *full, const agipc_bsr *U, double *val,
                                              int check);
AGIPC_API agipc_status agipc_pcg_solve_sym(agipc_handle h, const agipc_bsr *A, int storage, const double *b,
                                           double *x, int zero_x0, double rel_tol, int max_iters,
                                           int check_every, agipc_pcg_stats *stats);

/* ---- NEXT#4: step 1 for shells and rods ------------------------------------------------
 * "applicable to various element types (shells, volumes, rods)" (main Sec 4.2).
 *   shells (triangles a,b,c): rest tangent basis t1 = e1/|e1|, n = e1 x e2 / |e1 x e2|,
 *     t2 = n x t1 (e1 = X_b - X_a, e2 = X_c - X_a); D_m = [t_r . e_c] (2x2);
 *     F = D_s D_m^-1 (3x2), D_s = [x_b - x_a | x_c - x_a]; G = 1/2 (F^T F - I_2)
 *   rods (edges a,b): F = |x_b - x_a| / |X_b - X_a|, G = 1/2 (F^2 - 1)
 *   n_el = ||G(x_cur) - G(x_prev)||_F, flagged iff n_el > threshold (strict); every slot listed
 *   for a flagged element gets tag 0.  Flags ACCUMULATE into slot_tags: reset_tags = 1 first
 *   sets all nnz_adj slots to 1; a mixed mesh calls agipc_tag_edges (which resets) and then
 *   these with reset_tags = 0, so an edge is protected iff ANY adjacent element is flagged.
 *   tris [T][3] / segs [S][2]: node ids; tri_slots [T][6] = slots of (01,10,02,20,12,21),
 *   seg_slots [S][2] = slots of (ab, ba); -1 = no slot.  Fixed fp64 operation order (R12).
 *   Errors / n_flagged / EDEGENERATE as agipc_tag_edges. */
AGIPC_API agipc_status agipc_tag_shells(agipc_handle h, int64_t n_tris, const int32_t *tris, const int32_t *tri_slots,
                                        const double *x_rest, const double *x_prev, const double *x_cur,
                                        double threshold, int64_t nnz_adj, int reset_tags, uint8_t *slot_tags,
                                        double *tri_norm, int64_t *n_flagged /*[host]*/);
AGIPC_API agipc_status agipc_tag_rods(agipc_handle h, int64_t n_segs, const int32_t *segs, const int32_t *seg_slots,
                                      const double *x_rest, const double *x_prev, const double *x_cur,
                                      double threshold, int64_t nnz_adj, int reset_tags, uint8_t *slot_tags,
                                      double *seg_norm, int64_t *n_flagged /*[host]*/);

/* ---- NEXT#3: fine-level hash reduction -------------------------------------------------
 * supp Sec 2: unreduced Hessian triplets (i, j, B_ij) get the key (i << 32) | j,
 * are sorted by key (equal keys keep their input order) and each run of equal keys is summed
 * in that order; the unique triplets form the fine BSR (rows ascending, columns ascending).
 * The topology is static: agipc_triplet_plan does the key sort once per mesh (caller
 * buffers, capacity retry on col/seg_ptr: ENOSPACE with nnzb set; synchronises), and
 * agipc_triplet_reduce streams the values of every Newton step (thread per unique block,
 * in-order sums, bit-identical to the sequential definition).
 *   ti, tj : [n_trip] row / column ids (0 <= ti < n_rows, tj >= 0; EINVAL otherwise, checked before
 *            any use; the columns need not be square: the unique blocks carry them as given)
 *   tval   : [n_trip][3][3];  val : out [nnzb][3][3] */
typedef struct {
  int64_t n_rows, n_trip;  /* [host] set by plan */
  int64_t nnzb;            /* [host] out: unique blocks */
  int64_t cap_nnzb;        /* [host] in: capacity of col and seg_ptr (seg_ptr holds cap_nnzb+1) */
  int64_t *row_ptr;        /* out [n_rows+1] */
  int32_t *col;            /* out [cap_nnzb] */
  int64_t *seg_ptr;        /* out [cap_nnzb+1]: triplets of block u are seg_idx[seg_ptr[u]..seg_ptr[u+1]) */
  int32_t *seg_idx;        /* out [n_trip]: triplet ids sorted by (key, id) */
} agipc_triplet_plan_t;

AGIPC_API agipc_status agipc_triplet_plan(agipc_handle h, int64_t n_rows, int64_t n_trip, const int32_t *ti,
                                          const int32_t *tj, agipc_triplet_plan_t *plan);
AGIPC_API agipc_status agipc_triplet_reduce(agipc_handle h, const agipc_triplet_plan_t *plan, const double *tval,
                                            double *val);

/* ---- NEXT#1: prolongation d_f = U^T d_c ------------------------------------------------
 * "we mathematically prolongate the displacement to the fine mesh using the transpose of
 * the restriction operator" (main Sec 4.3).  For every fine node f with parent
 * c = new_map[f]:
 *   c <  n3 : d_f[f] = alpha * x_c[c]
 *   c >= n3 : d_f[f] = alpha * sum_{p<4} w_f[p] x_c[n3 + 4(c-n3) + p],  w_f = (X_bar_f, 1)
 * (A_f^T applied to the 12 coarse DoFs, A_f = [X_bar^T 1] (x) I3).  alpha = -1 turns
 * the coarse solution y of H_c y = g_c into the fine direction of P:752 in the same pass.
 * The post-coarsening fine PCG (<= 10 iterations) is agipc_pcg_solve on H_f with
 * this d_f as x0 (zero_x0 = 0).
 *   mesh    : n_nodes, x_rest [N][3] (the X_bar of assemble) -- the other fields are unused
 *   new_map : [N] as written by agipc_assemble_coarse; n3 = out->n3, n_slots = out->n_slots
 *             (entries outside [0, n3 + (n_slots-n3)/4) give AGIPC_EINVAL, d_f unspecified)
 *   x_c     : [n_slots][3] coarse vector;  d_f : [N][3] out.
 * Asynchronous on the handle's stream except for the error check (one 4-byte D2H). */
AGIPC_API agipc_status agipc_prolongate(agipc_handle h, const agipc_mesh *mesh, const int32_t *new_map,
                                        int64_t n3, int64_t n_slots, const double *x_c, double alpha,
                                        double *d_f);

/* ==== Multi-GPU partitioned path (north star) ==========
 * One process per GPU; rank r owns a contiguous range of fine nodes and passes its LOCAL mesh
 * (see agipc_mesh above).  Steps 1-3 run unchanged on the local mesh (H_fine = the rank's rows
 * x owned columns); the caller moves the buffers below between ranks (torch.distributed /
 * NCCL: send/recv for halos, all-gather of per-rank counts, all-reduce of the PCG sums).
 * Global coarse numbering is rank-major: rank r's slots are [S_r, S_r + n_slots_r) with
 * S_r = exclusive prefix sum of n_slots over ranks (the north star's all-gather exclusive scan),
 * each rank's own slots ordered 3-DoF then 12-DoF as on one GPU.
 *
 * agipc_gather_rows: dst[k] = src[idx[k]] for rows of row_bytes bytes (multiple of 4) -- halo
 *   send buffers (exchange 1: x_prev/x_cur rows of the send lists; exchange 3: column codes).
 *
 * agipc_coarse_halo (owner side of exchange 3): for the fine nodes send_idx[0..n_send) sent to
 *   one peer, the coarse slots that peer needs -- aggregates in order of first appearance in
 *   the send list, 1 or 4 consecutive slots each -- into send_slots[0..*n_slots) (this rank's
 *   local slot ids; pack z at these slots every PCG iteration), and for every sent fine node
 *   its column code ghost_code[k] = (offset of its aggregate's first slot in that list) |
 *   (1<<30 if the aggregate is 12-DoF).  Capacity retry: *n_slots > cap_slots => ENOSPACE
 *   with *n_slots set.  Synchronises.
 *
 * agipc_assemble_halo: the Galerkin blocks of this rank's coarse rows x ghost coarse columns
 *   (Alg S4 + Eq 4 for fine blocks (i owned, j ghost); the off-rank part of U H U^T).
 *   H_halo: rows = owned fine nodes, col = ghost index g (local node n_nodes + g), ascending.
 *   ghost_code[g]: the owner's column code (above), received for every ghost.  Peer q's ghosts
 *   are g in [peer_ghost_ptr[q], peer_ghost_ptr[q+1]) ([host], n_peers+1) and its slots start
 *   at local column peer_slot_base[q] ([host]; >= n_slots of this rank: ghost slots follow the
 *   owned slots in the PCG vectors).  Output: BSR over this rank's n_slots rows, columns = local
 *   ghost-slot columns, ascending; capacity retry on col/val like agipc_assemble_coarse.
 *   Synchronises.
 *
 * Distributed PCG: the 1-GPU iteration split at its reductions.  red is a device double[4]
 * that the CALLER sums over all ranks (all-reduce) after every setup / spmv / update call:
 *   setup(A, A_halo, n_ghost_slots, b)    -> red = [r.z, r.r, b.b] partials     (x0 = 0)
 *   pack(send_slots) -> sendbuf; exchange; spmv(recvbuf = ghost z, red) -> red = [p.q]
 *   update(red) -> red = [r.z, r.r];  pack + exchange; spmv; ...     status() polls (syncs);
 *   finish(red, x) consumes the last reduced sums and copies the rank's rows of x.
 * Every rank applies the same scalar logic to the same reduced sums, so all ranks stop at the
 * same iteration.  Vectors: owned slots 0..n_rows-1, ghost slots n_rows..n_rows+n_ghost_slots-1
 * (the recv buffer holds them in that order; A_halo's columns index them). */
/* ---- library-owned communicator (NCCL, resolved at run time) ---------------------------
 * The north star's exchanges run inside libagipc: one NCCL communicator per handle (agipc_comm_init),
 * collectives on the handle's stream.  The caller only moves the 128-byte unique id (rank 0 calls
 * agipc_comm_unique_id and broadcasts it, e.g. over a torch.distributed process group).
 * AGIPC_ENCCL: libnccl.so.2 could not be loaded (or $AGIPC_NCCL_LIB) or an NCCL call failed.
 *
 * agipc_comm_allgather_scan (exchange 2): local [k] int64 device values of this rank ->
 *   all [nranks][k] (every rank's values), scan [2k]: scan[j] = sum over ranks r' < rank of
 *   all[r'][j] (the exclusive prefix = this rank's global offset), scan[k + j] = the total.
 *   Asynchronous.
 * agipc_comm_alltoall_i64: send[q] goes to rank q, recv[q] comes from rank q (device, [nranks]).
 * agipc_halo_exchange (exchanges 1 and 3): rows of row_bytes bytes (multiple of 4).  For every peer
 *   q: the rows src[send_idx[send_ptr[q] .. send_ptr[q+1])] are sent to peer_rank[q], and the rows
 *   received from it land at dst rows [recv_ptr[q], recv_ptr[q+1]) (dst = the ghost region, e.g.
 *   x + 3 n_owned).  Grouped send/recv, asynchronous. */
#define AGIPC_UNIQUE_ID_BYTES 128
typedef struct {
  int n_peers;
  const int *peer_rank;      /* [host] [n_peers] */
  const int64_t *send_ptr;   /* [host] [n_peers+1] */
  const int32_t *send_idx;   /* device [send_ptr[n_peers]] rows of src to send */
  const int64_t *recv_ptr;   /* [host] [n_peers+1] rows of dst to receive */
} agipc_halo;

AGIPC_API agipc_status agipc_comm_unique_id(void *unique_id /*[host] out, 128 B*/);
AGIPC_API agipc_status agipc_comm_init(agipc_handle h, const void *unique_id /*[host] 128 B*/, int nranks, int rank);
AGIPC_API agipc_status agipc_comm_info(agipc_handle h, int *nranks, int *rank, int *nccl_version /*[host]*/);
AGIPC_API agipc_status agipc_comm_allgather_scan(agipc_handle h, const int64_t *local, int k, int64_t *all,
                                                 int64_t *scan);
AGIPC_API agipc_status agipc_comm_alltoall_i64(agipc_handle h, const int64_t *send, int64_t *recv);
AGIPC_API agipc_status agipc_halo_exchange(agipc_handle h, const agipc_halo *halo, const void *src, int row_bytes,
                                           void *dst);

/* agipc_dpcg_solve: the whole distributed block-Jacobi PCG (the split-phase iteration below with
 * its reductions and halo inside the library): per iteration the z values of the send slots go to
 * the peers by NCCL send/recv (exchange 4), the p.q and [r.z, r.r] partials are summed by
 * ncclAllReduce, and check_every iterations are captured -- NCCL calls included -- in one CUDA
 * graph; the host polls the device done flag between graph launches, as agipc_pcg_solve.
 *   A, A_halo, n_ghost_slots, b : as agipc_dpcg_setup (x0 = 0);  x : out [A->n_rows][3]
 *   slots : the PCG halo -- send_idx = this rank's slots to send (coarse_halo send lists),
 *           recv_ptr = the ghost-slot ranges (rows of the ghost region, [0, n_ghost_slots))
 * Every rank must call it with the same rel_tol / max_iters / check_every; all stop together.
 * Singular diagonal blocks on any rank stop every rank (ESINGULAR everywhere). */
AGIPC_API agipc_status agipc_dpcg_solve(agipc_handle h, const agipc_bsr *A, const agipc_bsr *A_halo,
                                        int64_t n_ghost_slots, const agipc_halo *slots, const double *b, double *x,
                                        double rel_tol, int max_iters, int check_every, agipc_pcg_stats *stats);

typedef struct {
  int64_t n_rows, nnzb;  /* [host] out */
  int64_t cap_nnzb;      /* [host] in  */
  int64_t *row_ptr;      /* out [n_rows+1] (n_rows = n3 + 4 n12 of this rank) */
  int32_t *col;          /* out [cap_nnzb] */
  double *val;           /* out [cap_nnzb][3][3] */
} agipc_halo_matrix;

AGIPC_API agipc_status agipc_gather_rows(agipc_handle h, const void *src, const int32_t *idx, int64_t n,
                                         int row_bytes, void *dst);
AGIPC_API agipc_status agipc_coarse_halo(agipc_handle h, const int32_t *new_map, int64_t n3, int64_t n_coarse,
                                         const int32_t *send_idx, int64_t n_send, int32_t *ghost_code,
                                         int32_t *send_slots, int64_t cap_slots, int64_t *n_slots /*[host]*/);
AGIPC_API agipc_status agipc_assemble_halo(agipc_handle h, const agipc_mesh *mesh, const int32_t *new_map,
                                           int64_t n3, int64_t n_coarse, const agipc_bsr *H_halo, int64_t n_ghost,
                                           const int32_t *ghost_code, int n_peers,
                                           const int64_t *peer_ghost_ptr /*[host]*/,
                                           const int64_t *peer_slot_base /*[host]*/, agipc_halo_matrix *out);
AGIPC_API agipc_status agipc_dpcg_setup(agipc_handle h, const agipc_bsr *A, const agipc_bsr *A_halo /*nullable*/,
                                        int64_t n_ghost_slots, const double *b, double rel_tol, int max_iters,
                                        double *red);
AGIPC_API agipc_status agipc_dpcg_pack(agipc_handle h, const int32_t *send_slots, int64_t n_send, double *sendbuf);
AGIPC_API agipc_status agipc_dpcg_spmv(agipc_handle h, const double *recvbuf, double *red);
AGIPC_API agipc_status agipc_dpcg_update(agipc_handle h, double *red);
AGIPC_API agipc_status agipc_dpcg_status(agipc_handle h, int *done /*[host]*/, agipc_pcg_stats *stats /*[host]*/);
AGIPC_API agipc_status agipc_dpcg_finish(agipc_handle h, const double *red, double *x, agipc_pcg_stats *stats);

#ifdef __cplusplus
}
#endif
#endif /* AGIPC_H_ */
