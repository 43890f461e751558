/* libhks -- C ABI of the B200-native hierarchical kernel factorize / solve.
 *
 * This is the drop-in boundary for the north-star path of the reference
 * package `hikersolve` (arXiv 1701.02324).  The reference has no FFI: its
 * boundary is the Python API re-exported in pkg/src/hikersolve/__init__.py:12-75.
 * Every entry point below replaces the numerical core of one of those
 * functions (cited per function); the Python package
 * `paper_1701_02324_b200` keeps the reference's names, argument meaning and
 * exceptions on top of this ABI, and INTEGRATION.md shows the ctypes binding
 * a maintainer of the reference would add.
 *
 * Conventions
 *  - all pointers are DEVICE pointers unless a parameter says "host";
 *  - matrices are column-major with an explicit leading dimension;
 *  - points are row-major (n x d) float64 in tree order;
 *  - every call is stream-ordered on `stream` (a cudaStream_t, NULL = legacy
 *    default stream) and returns HKS_OK or an error code; the thread-local
 *    message of the last failure is hks_last_error();
 *  - no call allocates persistent device memory except hks_plan_create,
 *    which owns its descriptor tables and level workspaces until
 *    hks_plan_destroy.
 */
#ifndef HKS_H_
#define HKS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HKS_ABI_VERSION 1

enum hks_status {
  HKS_OK = 0,
  HKS_ERR_INVALID = 1,          /* ValueError in the reference */
  HKS_ERR_CUDA = 2,             /* CUDA runtime failure */
  HKS_ERR_SINGULAR = 3,         /* SingularMatrixError, linalg.py:163-168 */
  HKS_ERR_REDUCED_SINGULAR = 4, /* FactorizationError, solver.py:99-105 */
  HKS_ERR_SKELETON = 5,         /* RuntimeError, skeleton.py:166-169 */
  HKS_ERR_NOT_SUPPORTED = 6
};

enum hks_family { HKS_GAUSSIAN = 0, HKS_LAPLACE3D = 1, HKS_POLYNOMIAL = 2 };

/* KernelSpec, kernels.py:23-48 */
typedef struct hks_kernel {
  int32_t family;
  int32_t degree;
  double h;
  double shift;
  double regularization;
} hks_kernel;

/* Flat per-node buffers of a factorization layout (see hks_layout). */
enum hks_buffer {
  HKS_BUF_INTERP = 0,   /* double: r x c interpolation matrix P (Skeleton.interp), ld r */
  HKS_BUF_SKEL = 1,     /* int64:  r skeleton indices (Skeleton.indices) */
  HKS_BUF_THETA = 2,    /* double: r x r theta (NodeFactor.theta), ld r */
  HKS_BUF_LEAF_LU = 3,  /* double: m x m LU of K_aa + lam I (NodeFactor.diag_lu.lu), ld m */
  HKS_BUF_LEAF_PIV = 4, /* int32:  m pivots, 0-based (NodeFactor.diag_lu.piv) */
  HKS_BUF_PHI = 5,      /* double: m x r phi, ld m */
  HKS_BUF_Z_LU = 6,     /* double: R x R LU of Z, ld R */
  HKS_BUF_Z_PIV = 7,    /* int32:  R pivots, 0-based */
  HKS_BUF_PUSH = 8,     /* double: R x r child_push, ld R */
  HKS_BUF_COUP = 9,     /* double: r_left x r_right coupling K(q_l, q_r), ld r_left */
  HKS_BUF_STATS = 10,   /* per node: double anorm[nnodes], double rcond[nnodes] (dgecon),
                           int32 info[nnodes] (first zero pivot) -- 3 * nnodes doubles */
  HKS_NBUF = 11
};

typedef struct hks_plan hks_plan;

const char* hks_last_error(void);
int hks_abi_version(void);

/* Storage layout of a complete tree with n points, `depth` levels below the
 * root and rank cap `max_rank` (leaf ranks <= min(max_rank, leaf size),
 * internal ranks <= min(max_rank, r_left + r_right)).  Host outputs:
 * sizes[HKS_NBUF] element counts; offsets[b * nnodes + i] element offset of
 * node i in buffer b (-1 if node i has no such array).  `offsets` may be NULL.
 * Node ranges follow tree.py:100-121 (left child takes ceil(size / 2)). */
int hks_layout(int64_t n, int64_t depth, int64_t max_rank, int64_t* sizes, int64_t* offsets);

/* eval_block, kernels.py:64-105: out = K(X[rows], X[cols]) + diag * [i == j].
 * rows/cols: device int64 index lists, or NULL for the ranges
 * [row0, row0 + nrows) / [col0, col0 + ncols).  row_major selects out[i*ldo + j]
 * instead of out[i + j*ldo]. */
int hks_eval_block(const double* X, int64_t d, const hks_kernel* kern, const int64_t* rows,
                   int64_t row0, int64_t nrows, const int64_t* cols, int64_t col0, int64_t ncols,
                   double* out, int64_t ldo, int32_t row_major, double diag, void* stream);

/* Fused kernel summation U = beta U + K(X[rows], X[cols]) W (+ diag * W when
 * rows and cols are the same range) without forming K -- the "never
 * materialise K" path of treecode.py:99-101, krylov.py:176-185 (dense_oracle)
 * and the sampled residual checks.  W: ncols x k (ldw), U: nrows x k (ldu). */
int hks_kernel_sum(const double* X, int64_t d, const hks_kernel* kern, const int64_t* rows,
                   int64_t row0, int64_t nrows, const int64_t* cols, int64_t col0, int64_t ncols,
                   const double* W, int64_t ldw, int64_t k, double* U, int64_t ldu, double beta,
                   double diag, void* stream);

/* Cross kernel summation U = beta U + K(Xq[rows], Xs) W for nq query points
 * (rows: device int64 indices into Xq, or NULL for Xq[0..nq)) against ns
 * source points, both row-major n x d, W ns x k (ldw), U nq x k (ldu).  The
 * sources are split into column chunks so few queries still fill the GPU;
 * the chunks' partial sums are added in a fixed order (deterministic).
 * KRR prediction (cli.py:415-422 _cross_predict) and the sampled-row error
 * metrics.  Synchronous (returns when U is written). */
int hks_cross_sum(const double* Xq, int64_t nq, const double* Xs, int64_t ns, int64_t d, const hks_kernel* kern,
                  const int64_t* rows, const double* W, int64_t ldw, int64_t k, double* U, int64_t ldu,
                  double beta, void* stream);

/* factor_dense, linalg.py:151-169: in-place LU with partial pivoting of an
 * n x n matrix; piv 0-based (scipy lu_factor); *info_host = 0 or the 1-based
 * step of the first exactly-zero pivot. */
int hks_lu_factor(double* A, int64_t n, int64_t lda, int32_t* piv, int32_t* info_host, void* stream);

/* solve_dense, linalg.py:172-179: B := A^-1 B in place (nrhs columns). */
int hks_lu_solve(const double* LU, const int32_t* piv, int64_t n, int64_t lda, double* B,
                 int64_t ldb, int64_t nrhs, void* stream);

/* pivoted_qr + interpolative_decomposition, linalg.py:43-136, for one
 * m x n matrix A (column-major, lda; overwritten).  Outputs (device):
 * pivots[n] int64, interp[max_rank x n] (ld = rank), host *rank_host. */
int hks_interp_decomp(double* A, int64_t m, int64_t n, int64_t lda, double tol, int64_t max_rank,
                      int64_t* pivots, double* interp, int64_t* rank_host, void* stream);

/* ----- plan: the level program of one compressed operator ----------------
 * A plan holds the tree layout, the skeleton ranks and the uploaded
 * descriptor programs of build_operator / factorize / solve / hmatvec /
 * upward_pass.  It owns no factor storage: every call receives
 * `buffers[HKS_NBUF]`, the device base pointers of the flat per-node arrays
 * of hks_layout (entries a call does not touch may be NULL), so one plan
 * serves any number of factorizations (e.g. different lambda) of the same
 * operator.  X: n x d tree-ordered points (device, must outlive the plan);
 * ranks_host[nnodes] the skeleton ranks (root ignored).  Calls on one plan
 * must be ordered on one stream (plan-owned workspaces). */
int hks_plan_create(hks_plan** plan, const double* X, int64_t n, int64_t d, int64_t depth,
                    int64_t max_rank, const int64_t* ranks_host, const hks_kernel* kern);
int hks_plan_destroy(hks_plan* plan);

/* ----- subtree sharding (solver.py:111-259 split at level p) --
 * A tree sharded over P = 2^p ranks is one subtree plan per rank plus one top
 * plan, replicated on every rank.
 *  HKS_PLAN_SUBTREE: the rank's shard, a complete subtree rooted at a level-p
 *    node of the global tree (X = the shard's first point, n = shard size,
 *    skeleton indices local to the shard).  Its root keeps a skeleton
 *    (ranks_host[0] = r_0): factorize also forms the root's Theta and push;
 *    solve / hmatvec run in two halves around the exchange (hks_solve_part).
 *  HKS_PLAN_TOP: levels 0..p of the global tree (X = all points, skeleton
 *    indices global).  Its 2^p leaves are the shard roots: their Theta and
 *    skeleton indices are written by the caller (the layout puts leaf j's
 *    s x s Theta at j * s * s and its s indices at j * s, so an all-gather of
 *    the ranks' blocks lands in place), and factorize starts at level p - 1.
 * Layout / plan creation take the mode; HKS_PLAN_FULL is the unsharded tree. */
enum hks_plan_mode { HKS_PLAN_FULL = 0, HKS_PLAN_SUBTREE = 1, HKS_PLAN_TOP = 2 };
int hks_layout_ex(int64_t n, int64_t depth, int64_t max_rank, int32_t mode, int64_t* sizes, int64_t* offsets);
int hks_plan_create_ex(hks_plan** plan, const double* X, int64_t n, int64_t d, int64_t depth,
                       int64_t max_rank, const int64_t* ranks_host, const hks_kernel* kern, int32_t mode);

/* Split solve / hmatvec.  Subtree plans: part 1 = leaf solves and the upward
 * sweep, leaving the root's psi (solve) or skeleton weights (hmatvec) in
 * xchg (r_0 x k, ld r_0); part 2 = the downward sweep from the root's
 * incoming correction / accumulator read from xchg.  x (u) must be the same
 * buffer in both halves.  Top plans and full plans: part 0.  For top plans
 * b (w) holds the shard roots' psi and x (u) receives their corrections,
 * shard j's r_j x k block at j * max_rank * k (ld r_j). */
int hks_solve_part(hks_plan* plan, void* const* buffers, const double* b, double* x, int64_t k, int32_t part,
                   double* xchg, void* stream);
int hks_hmatvec_part(hks_plan* plan, void* const* buffers, const double* w, double* u, int64_t k, double lam,
                     int32_t part, double* xchg, void* stream);

/* build_operator, treecode.py:41-62: the sibling couplings K(q_l, q_r) from
 * HKS_BUF_SKEL into HKS_BUF_COUP.  Leaf blocks: by default re-evaluated
 * inside factorize and the fused hmatvec; hks_plan_cache_leaves evaluates
 * them once into plan-owned device memory (N x m doubles, as the
 * reference's build_operator caches HierarchicalOperator.leaf_blocks,
 * treecode.py:48-51), after which factorize copies K_aa + lam I and the
 * hmatvec leaf level is a batched GEMM -- call it before the plan's first
 * factorize / solve / hmatvec (HKS_ERR_INVALID otherwise; a no-op for top
 * plans).  hks_leaf_block gives the leaf_blocks diagnostic view (the cached
 * values when cached). */
int hks_build_operator(hks_plan* plan, void* const* buffers, void* stream);
int hks_plan_cache_leaves(hks_plan* plan, void* stream);
int hks_leaf_block(hks_plan* plan, int64_t leaf, double* out, void* stream);

/* factorize, solver.py:111-186.  Reads INTERP, COUP; writes THETA, LEAF_LU,
 * LEAF_PIV, PHI, Z_LU, Z_PIV, PUSH, STATS.  with_cond: also run the dgecon
 * estimate of every Z (NodeFactor.z_cond) -- asynchronously, on the
 * condition stream (hks_set_cond_stream), each level as soon as its LU is
 * done; Z_LU and STATS must stay allocated until it finishes (hks_cond_wait
 * / hks_factor_stats).  Returns once the factorization itself is complete.
 * On an exactly-zero pivot returns
 * HKS_ERR_SINGULAR (leaf, linalg.py:163-168) or HKS_ERR_REDUCED_SINGULAR
 * (Z, solver.py:99-105) with the failing heap index in *bad_node_host. */
int hks_factorize(hks_plan* plan, void* const* buffers, double lam, int32_t with_cond,
                  int64_t* bad_node_host, void* stream);

/* Device milliseconds per level of the last hks_factorize (ms_host[level],
 * level 0..depth; Factorization.level_seconds, solver.py:164-176). */
int hks_factor_level_ms(hks_plan* plan, double* ms_host);

/* z_cond (1 / dgecon rcond; 0 for leaves) and info per node, host outputs;
 * waits for the plan's pending dgecon estimates first. */
int hks_factor_stats(hks_plan* plan, void* const* buffers, double* z_cond_host, int32_t* info_host,
                     void* stream);

/* The stream the dgecon estimates run on (NULL: the plan's own lowest-
 * priority stream), and a device-side wait of `stream` for the last
 * factorization's estimates. */
int hks_set_cond_stream(hks_plan* plan, void* stream);
int hks_cond_wait(hks_plan* plan, void* stream);

/* solve / solve_multi, solver.py:189-270: x = (Ktilde + lam I)^-1 b for k
 * right-hand sides in tree order; b, x: n x k column-major (ld n); x may
 * alias b. */
int hks_solve(hks_plan* plan, void* const* buffers, const double* b, double* x, int64_t k,
              void* stream);

/* hmatvec, treecode.py:92-128: u = (Ktilde + lam I) w, n x k (ld n), u != w. */
int hks_hmatvec(hks_plan* plan, void* const* buffers, const double* w, double* u, int64_t k,
                double lam, void* stream);

/* upward_pass, treecode.py:65-89 (k columns): skeleton weights of every
 * non-root node written into `out`; node i's r_i x k block starts at
 * out + offsets[i] with leading dimension lds[i] (hks_upward_offsets). */
int hks_upward_offsets(hks_plan* plan, int64_t k, int64_t* offsets_host, int64_t* lds_host,
                       int64_t* total_host);
int hks_upward(hks_plan* plan, void* const* buffers, const double* w, int64_t k, double* out,
               void* stream);

/* ----- vector kernels of the GMRES driver (krylov.py:82-130) ----------------
 * hks_vdots: out[v] = scale * <X[v], y> (+ out[v] when accumulate) for m
 * vectors at stride ldv; deterministic fixed-grid reduction; part = caller
 * scratch of m * 296 doubles.  hks_vaxpys: y += scale * sum_v coef[v] X[v]
 * (coef on the device). */
int hks_vdots(const double* X, int64_t ldv, int64_t m, const double* y, int64_t n, double* out,
              double scale, int32_t accumulate, double* part, void* stream);
int hks_vaxpys(const double* X, int64_t ldv, int64_t m, const double* coef, double scale, double* y,
               int64_t n, void* stream);

/* ----- setup stages ------------------------------------------------------------
 * build_tree, tree.py:87-144: X_in n x d input-order points; starts[(2^depth - 1)
 * x d] the normalised power-method start vectors default_rng([seed, level,
 * begin]).standard_normal(d) / norm (heap order); outputs X_out (tree order),
 * perm_out, split_dirs, split_vals. */
int hks_build_tree(const double* X_in, int64_t n, int64_t d, int64_t depth, int64_t steps,
                   const double* starts, double* X_out, int64_t* perm_out, double* split_dirs,
                   double* split_vals, void* stream);

/* knn_bruteforce, tree.py:163-188: out[n x k] int64, (d^2, index) order, k <= 32. */
int hks_knn(const double* X, int64_t n, int64_t d, int64_t k, int64_t* out, void* stream);
/* The same lists for the query rows [q0, q0 + nq) only (a shard's points
 * against all n): out[nq x k]. */
int hks_knn_rows(const double* X, int64_t n, int64_t d, int64_t k, int64_t q0, int64_t nq, int64_t* out,
                 void* stream);

/* Approximate kNN building blocks (no reference
 * counterpart): every point of segment [seg_off_host[i], seg_off_host[i+1])
 * of X against the points of its own segment (a random-projection-tree
 * leaf), rows by position, ids = perm[position], d^2 beside them
 * (out_idx / out_d2 n x k); and the per-row union of two (d^2, id)-sorted
 * lists with duplicates dropped. */
int hks_knn_segments(const double* X, int64_t n, int64_t d, int64_t k, const int64_t* seg_off_host, int64_t nseg,
                     const int64_t* perm, int64_t* out_idx, double* out_d2, void* stream);
int hks_knn_merge(const int64_t* a_idx, const double* a_d2, const int64_t* b_idx, const double* b_d2, int64_t n,
                  int64_t k, int64_t* out_idx, double* out_d2, void* stream);

/* sample_rows(knn_augmented), skeleton.py:111-121, for every node of one
 * level: mark = per-node bitmap of neighbours outside the node (counts to
 * the host); fill = map the host's top-up draws (ranks into the sorted rest
 * set) and compact each node's rows in ascending order. */
int hks_knn_rows_mark(const int64_t* knn, int64_t n, int64_t kappa, int64_t level, int64_t depth,
                      int32_t* bitmap, int64_t* counts_host, void* stream);
int hks_knn_rows_fill(int64_t n, int64_t level, int64_t depth, int32_t* bitmap, const int64_t* extra,
                      const int64_t* extra_off_host, int64_t* rows, const int64_t* row_off_host,
                      void* stream);
/* Sharded variants: the nodes [node0, node0 + count) of `level` only, and
 * kNN lists of the points [row0, row0 + nrows) only (a shard's rows; global
 * indices).  A node spanning several shards gets the OR of the ranks'
 * bitmaps (the caller's all-gather) and its counts from hks_bitmap_count. */
int hks_knn_rows_mark_ex(const int64_t* knn, int64_t row0, int64_t nrows, int64_t n, int64_t kappa, int64_t level,
                         int64_t node0, int64_t count, int32_t* bitmap, int64_t* counts_host, void* stream);
int hks_bitmap_count(const int32_t* bitmap, int64_t n, int64_t count, int64_t* counts_host, void* stream);
int hks_knn_rows_fill_ex(int64_t n, int64_t level, int64_t node0, int64_t count, int32_t* bitmap,
                         const int64_t* extra, const int64_t* extra_off_host, int64_t* rows,
                         const int64_t* row_off_host, void* stream);

/* build_skeletons for one level, skeleton.py:125-182: sampled block eval +
 * truncated column-pivoted QR + ID for `count` nodes (first heap index
 * first_node); rows / cands device flat lists with host offsets[count+1];
 * skeleton indices / interp written into the SKEL / INTERP layouts at the
 * given element offsets; ranks_host[count]. */
int hks_skeletonize_level(const double* X, int64_t d, const hks_kernel* kern, int64_t count,
                          int64_t first_node, const int64_t* rows, const int64_t* row_off,
                          const int64_t* cands, const int64_t* cand_off, double tau,
                          int64_t max_rank, int64_t* skel_buf, const int64_t* skel_off,
                          double* interp_buf, const int64_t* interp_off, int64_t* ranks_host,
                          void* stream);

/* hks_skeletonize_level keeps its stream-ordered workspace in the device's
 * default memory pool from level to level; this returns it (after the last
 * level; skeleton.py's build_skeletons calls it once). */
int hks_skeleton_workspace_release(void* stream);

/* ----- instrumentation ----------------------------------------------------------
 * hks_profile(1, ...) resets and starts per-kind CUDA-event timing of every
 * plan step; hks_profile(0, out) stops; out[kind * 4 + {launches, ms, flops,
 * bytes}] for kinds GEMM, COPY, GETRF, GETRS, GECON, EVAL_CM, EVAL_RM, KSUM
 * (flops / bytes are the algorithmic counts of the executed descriptors).
 * hks_launch_count: plan-step launches since load. */
int hks_profile(int32_t enable, double* out_host);
long long hks_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* HKS_H_ */
