/*
 * libinvaskit — B200 (sm_100a) Inv-ASKIT factorization and solve, C ABI.
 *
 * This is the drop-in boundary for the reference's factor/solve entry points
 * (kernelsolve 0.1.0, /root/reference/pkg/src/kernelsolve):
 *
 *   ks_create + ks_factorize   replace  factorize(ck, lam, threads)   solver.py:92-189
 *   ks_solve                   replaces solve(hf, b)                  solver.py:192-197
 *                                       solve_many(hf, B)             solver.py:200-213
 *   ks_get_diag / ks_get_z_cond / ks_get_fallback_nodes
 *                              expose   HierFactor.diagnostics       solver.py:111-116,175-188
 *   ks_get_node_h / ks_get_leaf_factor
 *                              expose   NodeFactor.H / LeafFactor.factor (parity debugging)
 *
 * The problem is passed exactly as the reference's CompressedKernel holds it
 * (compress.py:93-142, tree.py:53-81): points in ORIGINAL order, the tree
 * permutation, BFS node table, skeleton ids (global point ids, pivot order)
 * and interpolation matrices P (rank x |cand|, row-major). Plain pointers and
 * sizes only; the library copies what it needs to the device at create time.
 *
 * Right-hand sides and solutions are n x q row-major in TREE (perm) order, as
 * solve_many takes them (solver.py:193). They may be host or
 * device pointers; the library detects which.
 *
 * Return codes (the Python layer maps them to kernelsolve.errors types):
 */
#ifndef INVASKIT_H
#define INVASKIT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KS_OK 0
#define KS_ERR_INVALID 1      /* InvalidArgumentError            (errors.py:13) */
#define KS_ERR_NOT_SPD 2      /* NotSPDError (not returned: non-SPD leaves take the LU fallback, solver.py:127-130) */
#define KS_ERR_SINGULAR 3     /* SingularMatrixError             (errors.py:25, linalg.py:205-206) */
#define KS_ERR_ILL_COND 4     /* IllConditionedError(node, cond) (errors.py:29-39, solver.py:150-152) */
#define KS_ERR_CUDA 5         /* device / runtime failure */
#define KS_ERR_UNSUPPORTED 6  /* shape outside what the kernels handle */
#define KS_ERR_IO 7           /* file missing, truncated or not in the KSINVASK container format */

typedef struct ks_problem {
  int64_t n;                  /* points */
  int64_t d;                  /* dimension */
  const double* coords;       /* n x d row-major, ORIGINAL order (PointSet.coords) */
  const int64_t* perm;        /* n, tree permutation (PartitionTree.perm) */
  int64_t n_nodes;            /* BFS node count, node 0 = root */
  const int64_t* node_begin;  /* n_nodes, TreeNode.begin */
  const int64_t* node_end;    /* n_nodes, TreeNode.end */
  const int64_t* node_left;   /* n_nodes, children[0] or -1 at leaves */
  const int64_t* node_right;  /* n_nodes, children[1] or -1 at leaves */
  const int64_t* rank;        /* n_nodes, Skeleton.rank (0: no skeleton, e.g. root) */
  const int64_t* skel_off;    /* n_nodes + 1 offsets into skel */
  const int64_t* skel;        /* Skeleton.skel, global point ids, pivot order */
  const int64_t* coeff_off;   /* n_nodes + 1 offsets into coeff */
  const double* coeff;        /* Skeleton.coeff, rank x |cand| row-major */
  double bandwidth;           /* Gaussian h (KernelSpec.bandwidth) */
} ks_problem;

typedef struct ks_diag {
  int64_t cholesky_fallbacks; /* diagnostics["cholesky_fallbacks"] */
  int64_t n_z_cond;           /* number of internal nodes with a Z condition estimate */
  int64_t n_warnings;         /* z_cond > 1e10 (solver.py:183-188) */
  int64_t error_node;         /* node id for KS_ERR_ILL_COND / KS_ERR_SINGULAR, else -1 */
  double error_cond;          /* condition estimate for KS_ERR_ILL_COND */
  double max_z_cond;
} ks_diag;

typedef struct ks_factor ks_factor;

/* Validate the problem, upload it (tree order) and allocate factor storage on
 * `device`. No factorization yet. */
int ks_create(const ks_problem* prob, int device, ks_factor** out);

/* Factor K~ + lam I (solver.py:92-189). `threads` of the reference is accepted
 * by the Python layer and ignored: the result does not depend on it. May be
 * called again on the same handle (e.g. a new lam); `stream` may be NULL. */
int ks_factorize(ks_factor* f, double lam, void* stream);

/* X = (K~ + lam I)^-1 B, B and X n x q row-major, tree order; q >= 0.
 * Reentrant on one handle: every call runs in a workspace of its own, so
 * concurrent calls from several threads / on several streams are safe (the
 * reference's HierFactor is immutable and shared, solver.py:77-89). With
 * device pointers the call is asynchronous on `stream`. */
int ks_solve(ks_factor* f, const double* B, double* X, int64_t q, void* stream);

/* ---- subtree sharding (one process per GPU) ----
 * ks_create_shard: the handle factors the subtree of `shard_root` (a node at
 * level k = log2 p) with ks_factorize, and the levels above k with
 * ks_factorize_top once the H of every level-k node has been imported with
 * ks_node_exchange (the caller all-gathers them, e.g. NCCL). The solve runs as
 * ks_solve_up (local rows) -> exchange c of the level-k nodes ->
 * ks_solve_top -> ks_solve_down (local rows). B_local / X_local are device
 * pointers to the shard's rows [begin, end) of the tree-order RHS. */
int ks_create_shard(const ks_problem* prob, int device, int64_t shard_root, ks_factor** out);
int ks_factorize_top(ks_factor* f, void* stream);
int ks_solve_up(ks_factor* f, const double* B_local, int64_t q, void* stream);
int ks_solve_top(ks_factor* f, int64_t q, void* stream);
int ks_solve_down(ks_factor* f, double* X_local, int64_t q, void* stream);
/* which: 0 = H (s_pad x s_pad), 1 = c (s_pad x q), 2 = t (s_pad x q); dir 0 out, 1 in. */
int ks_node_exchange(ks_factor* f, int which, int64_t node, double* dev, int64_t q, int dir, void* stream);
/* [shard_root, level, begin, end, s_pad, n_peers, peer node ids...]; returns length. */
int ks_shard_info(const ks_factor* f, int64_t* out, int64_t cap);

/* Y = K~ W, the compressed operator itself (hss_matvec, compress.py:352-411),
 * n x q row-major tree order, host or device; for residual checks
 * ||(K~ + lam I) X - B|| at any size. Needs a factorized (unsharded) handle. */
int ks_matvec(ks_factor* f, const double* W, double* Y, int64_t q, void* stream);

/* out[j] = sum_i exp(-|x_test_j - x_train_i|^2 / (2 h^2)) w_i: the dense, exact
 * cross-kernel matvec of krr_predict (solver.py:273-301). Coordinates row-major
 * (n x d), any order; host or device pointers. No handle needed. */
int ks_kernel_matvec(const double* x_test, int64_t n_test, const double* x_train, int64_t n_train, int64_t d,
                     double bandwidth, const double* w, double* out, int device, void* stream);

/* ---- persistence (operator inputs and factors; container layout in
 * paper_1602_01376_b200/csrc/container.h). The reference persists
 * only points (points.py:65-129, restated in paper_1602_01376_b200/persist.py);
 * these cache the compression output and the factorization across runs. ---- */
/* Write the operator inputs (coords, tree, skeletons, P, h) with a fingerprint. */
int ks_save_problem(const ks_problem* prob, const char* path);
/* Read them back; the arrays live in host memory owned by *owner until
 * ks_free_problem(*owner). A fingerprint mismatch (corruption) is KS_ERR_IO. */
int ks_load_problem(const char* path, ks_problem* out, void** owner);
int ks_free_problem(void* owner);
/* Save a factorized (unsharded) handle: factor buffers, lam, diagnostics and
 * the fingerprint of `prob`, the operator it was created from. */
int ks_save_factor(const ks_factor* f, const ks_problem* prob, const char* path);
/* Recreate a factorized handle on `device` from `prob` and a factor file;
 * KS_ERR_INVALID if the file was saved for a different operator. */
int ks_load_factor(const char* path, const ks_problem* prob, int device, ks_factor** out);

int ks_get_diag(const ks_factor* f, ks_diag* out);
/* lam of the last factorization (HierFactor.lam, solver.py:77-89). */
int ks_get_lam(const ks_factor* f, double* lam);
/* Fill up to cap (node id, Z condition estimate) pairs, ascending node id. */
int64_t ks_get_z_cond(const ks_factor* f, int64_t* nodes, double* conds, int64_t cap);
/* Fill up to cap leaf node ids that fell back from Cholesky to LU. */
int64_t ks_get_fallback_nodes(const ks_factor* f, int64_t* nodes, int64_t cap);
/* Copy the symmetrized reduced matrix H of a non-root node (rank x rank). */
int ks_get_node_h(const ks_factor* f, int64_t node, double* out);
/* Copy the m x m lower Cholesky factor of a leaf (LeafFactor.factor.lower). */
int ks_get_leaf_factor(const ks_factor* f, int64_t node, double* out);

/* Device bytes held by the handle. */
int64_t ks_device_bytes(const ks_factor* f);
/* Host -> device bytes ks_create / ks_create_shard copied: the operator inputs
 * the handle reads (a shard skips the P blocks of the other shards' subtrees). */
int64_t ks_upload_bytes(const ks_factor* f);
/* Per-phase device times (ms) of the last ks_factorize / ks_solve, measured with
 * CUDA events on the launching stream when profiling is on:
 * [0] leaf assembly, [1] leaf Cholesky + L21, [2] leaf SYRK (H), [3] internal
 * levels, [4] whole factorization, [5] whole solve. Returns count written. */
int ks_set_profiling(ks_factor* f, int on);
int ks_get_phase_ms(const ks_factor* f, double* ms, int cap);
/* Per internal level (deepest first) main-stream time of the last factorization. */
int ks_get_level_ms(const ks_factor* f, double* ms, int cap);
/* Levels the schedule runs per subtree on the subtree's own stream (subtree
 * pipelining): out2[0] as planned, out2[1] as enabled for this handle (0 when
 * KS_PIPE=0 or the group count disables it). */
int ks_pipelined_levels(const ks_factor* f, int* out2);
/* With KS_TRACE=1 in the environment: per-kernel device time table of the last
 * factorization (events after every launch on the launching stream). */
int ks_trace_report(const ks_factor* f, char* buf, int64_t len);
/* Kernel launches issued by the last factorize / solve. */
int64_t ks_last_launches(const ks_factor* f, int which /* 0 factor, 1 solve */);

/* Parity debugging: copy `count` doubles of an internal buffer (0 z per leaf,
 * 1 c per node, 2 t per node, 3 y per internal index, 4 augmented LU per
 * internal index, 5 leaf trapezoid per leaf index) and the padded layout
 * (m_pad, s_pad, t_pad, T, R, q_cap, n_internal, n_leaves). */
int ks_debug_copy(const ks_factor* f, int which, int64_t index, double* out, int64_t count);
int ks_debug_layout(const ks_factor* f, int64_t* out8);
/* Raw device address of an internal buffer (ids as ks_debug_copy; 6 = H), probes only. */
int64_t ks_debug_ptr(const ks_factor* f, int which);

/* Test hook: the library's batched DMMA GEMM on strided device batches. */
int ks_test_gemm(int M, int N, int K, int batch, int tri, const double* A, const double* B, double* C,
                 int64_t lda, int64_t sa, int64_t ldb, int64_t sb, int64_t ldc, int64_t sc, double alpha, double beta,
                 int ta, int tb, void* stream);

int ks_test_gemm_cidx(int M, int N, int K, int batch, const double* A, const double* B, double* C, const int* cidx,
                      int64_t lda, int64_t sa, int64_t ldb, int64_t sb, int64_t ldc, int64_t sc, int ta, int tb,
                      void* stream);

/* Release the handle and its device memory (to the library's device pool). */
void ks_destroy(ks_factor* f);

/* Return the memory the library's private device pool caches for reuse by the
 * next handle (up to KS_POOL_GB, default 32 GB) to the driver. */
int ks_trim_pool(int device);

/* Last error message of this thread (NUL-terminated, truncated to len). */
int ks_last_error(char* buf, int64_t len);

/* Library build fingerprint ("sm_100a ..."). */
const char* ks_version(void);

#ifdef __cplusplus
}
#endif

#endif /* INVASKIT_H */
