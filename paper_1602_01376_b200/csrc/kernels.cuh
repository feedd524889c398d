// Kernel argument blocks and launchers shared by the factor/solve runtime.
#pragma once

#include "common.cuh"

namespace ks {

// Device-resident problem tables (tree order everywhere).
struct DevTree {
  int64_t n, d;
  const double* coords;      // n x d, tree order (coords[perm])
  const int* rank;           // per node
  const int64_t* skel_off;   // per node, into skel_pos
  const int* skel_pos;       // skeleton point positions in tree order
  const int64_t* coeff_off;  // per node, into coeff
  const double* coeff;       // P per node, rank x |cand| row-major
  double h;                  // Gaussian bandwidth
};

// Leaf batch: leaves are processed together regardless of tree level.
struct LeafBatch {
  int count;
  const int* node;    // node id per leaf
  const int* begin;   // first point (tree order)
  const int* size;    // points in the leaf
  int m_pad, s_pad;   // padded leaf size / rank
  double* A;          // count x (m_pad + s_pad) x m_pad workspace, ld = m_pad
  int64_t a_stride;
};

// Internal nodes of one level (contiguous internal indices).
//
// Block formulation of the node step: Z = I + W G =
// [[I, X], [Y, I]] with X = B H_r, Y = B^T H_l (padded s_pad x s_pad each)
// is eliminated with its identity (1,1) block as pivot, leaving
// S = I - Y X, whose LU with partial pivoting is the only pivoted step; the
// augmented matrix the LU kernels see is
//     Aug = [[S, E], [F, C]]   (T = 2 s_pad, pivots among the first t_pad = s_pad rows)
//     E = P_r^T - Y P_l^T,  F = P_l H_l X - P_r H_r,  C = P_l H_l P_l^T,
// so after the LU its trailing block is C - F S^-1 E = P G Z^-1 P^T = H.
struct NodeBatch {
  int count;
  int first;         // internal index of the batch's first node (per-node solve buffers)
  const int* node;   // node ids
  const int* left;   // child node ids
  const int* right;
  int s_pad, t_pad, T;  // LU view: t_pad = s_pad pivot rows, T = t_pad + s_pad = 2 s_pad
  int zt;               // order of the padded Z (2 s_pad): P's row length, the solve's per-node vector
  double* Aug;          // count x T x T (row-major) [[S, E], [F, C]] -> LU, already offset to the level
  double* XY;           // count x 2 x s_pad x s_pad: X = B H_r, then Y = B^T H_l
  double* PHl;          // count x s_pad x s_pad: P_l H_l
  double* Bc;           // count x s_pad x s_pad coupling blocks
  double* BcT;          // count x s_pad x s_pad, B^T
  double* PT;           // count x zt x s_pad, P^T (rows [0, s_pad): P_l^T, then P_r^T)
  double* XS;           // count x zt x dk: gathered skeleton coordinates [left; right] (GEMM-form coupling), or null
  double* XN;           // count x zt: their squared norms
  int dk;               // padded dimension of XS (even)
  double* Pn;           // count x s_pad x zt padded P
  int* piv;             // count x t_pad
  double* norm1;        // count
  double* cond;         // count
  int* info;            // count (LU: first zero pivot column + 1)
  int* moves;           // count x (1 + 2*64): rows moved by the last LU panel
  int* pm;              // count x t_pad: composed row interchanges, (Pi v)[i] = v[pm[i]]
  double* scratch;      // count x 32 x 64: U12 of the last fused LU merge
};

// --- factor launchers (factor_kernels.cu) ---
void launch_gather_rows(const double* src, const int64_t* perm, int64_t n, int64_t d, double* dst, cudaStream_t st);
void launch_row_sqnorms(const double* X, int64_t n, int64_t d, double* out, cudaStream_t st);
// out[r] = sum_{t < tiles} partial[t * n + r], t ascending (deterministic)
void launch_sum_partials(const double* partial, int tiles, int n, double* out, cudaStream_t st);
void launch_leaf_copy_p(const DevTree& t, const LeafBatch& lb, cudaStream_t st);
void launch_leaf_assemble(const DevTree& t, const LeafBatch& lb, const double* lam, cudaStream_t st);
void launch_potrf64(const LeafBatch& lb, int j0, double* inv, int* info, cudaStream_t st);
void launch_sym_h(double* H, int64_t h_stride, const int* node_idx, int count, int s_pad, cudaStream_t st);
void launch_coupling(const DevTree& t, const NodeBatch& nb, cudaStream_t st);
// block formulation (node_kernels.cu): S = I and E = P_r^T blocks of Aug, the padded P copy
void launch_p_layout(const DevTree& t, const NodeBatch& nb, cudaStream_t st);
// ||Z||_1 from X and Y (linalg.py:176): max column abs sum of [[I, X], [Y, I]]
void launch_znorm1(const NodeBatch& nb, cudaStream_t st);
// pend (may be null): {row0, col0, rows, cols} of a U12 block waiting in nb.scratch
void launch_lu_panel(const NodeBatch& nb, int c0, int w, cudaStream_t st, const int* pend = nullptr);
void launch_trsm_unit_lower(const NodeBatch& nb, int r0, int w, int c0, int ncols, cudaStream_t st);
// dinv: scratch for the diagonal-block inverses, 2 x t_pad x 16 doubles per internal node
// max_ctas bounds the estimator's grid (it loops over the batch's nodes)
// lut (may be null): t_pad x t_pad per internal node, the column-major copy of
// Z's factors the estimator's non-transposed solves read (t_pad <= 512)
void launch_hager(const DevTree& t, const NodeBatch& nb, double* dinv, double* lut, int max_ctas, cudaStream_t st);
int hager_launches(const NodeBatch& nb);
// diagonal-block inverses of the LU factors (Hager solves), 2 x t_pad x 8 per node
void launch_diag_inv(const NodeBatch& nb, double* dinv, cudaStream_t st);
void launch_extract_h(const NodeBatch& nb, double* H, int64_t h_stride, cudaStream_t st);
void launch_compose_perm(const NodeBatch& nb, cudaStream_t st);
void launch_lu_merge(const NodeBatch& nb, int c0, int h, int w, cudaStream_t st);
// persistent per-node LU of a level (lu_slab.cu): slab width (0 = unsupported
// shape) and the cooperative launch (0 ok). sync: 4 zeroed words per node;
// err: the watchdog word. write_h: sym(H) -> H[node] (not at the root).
int slab_width(const NodeBatch& nb);
// 32-column panel as two 16-column halves in shared memory (lu_slab.cu)
bool lu_panel32_ok(const NodeBatch& nb);
void launch_lu_panel32(const NodeBatch& nb, int c0, cudaStream_t st);
int launch_lu_slab(const NodeBatch& nb, double* H, int64_t h_stride, bool write_h, unsigned* sync, unsigned* err,
                   cudaStream_t st);
void launch_fb_assemble(const DevTree& t, const NodeBatch& fb, const int* begin, const int* size, const double* lam,
                        cudaStream_t st);
void launch_fb_up(const NodeBatch& fb, const int* begin, const int* size, const double* B, int64_t ldb, double* Y,
                  double* c, int q, cudaStream_t st);
void launch_fb_down(const NodeBatch& fb, const int* begin, const int* size, const double* Y, const double* tin,
                    double* X, int64_t ldx, int q, bool has_tin, cudaStream_t st);
// leaf LU fallback (NotSPD leaves): augmented [[A, P^T], [-P, 0]]
void launch_leaf_aug_init(const DevTree& t, const LeafBatch& lb, const NodeBatch& fb, double lam,
                          cudaStream_t st);

// --- solve launchers (solve_kernels.cu) ---
struct SolveBufs {
  int q;                 // RHS columns (row-major [row][q])
  double* z;             // leaves x m_pad x q
  double* c;             // nodes x s_pad x q (skeleton weights, up pass)
  double* tin;           // nodes x s_pad x q (incoming, down pass)
  double* y;             // internal x t_pad x q
};
void launch_leaf_fwd(const LeafBatch& lb, const double* B, int64_t ldb, const SolveBufs& sb, cudaStream_t st);
void launch_leaf_bwd(const LeafBatch& lb, double* X, int64_t ldx, const SolveBufs& sb, bool has_tin,
                     cudaStream_t st);
void launch_node_up(const NodeBatch& nb, const SolveBufs& sb, bool root, cudaStream_t st);
void launch_node_down(const NodeBatch& nb, const SolveBufs& sb, bool root, cudaStream_t st);
void launch_node_up_cluster(const NodeBatch& nb, const SolveBufs& sb, bool root, int q0, int qc, cudaStream_t st);
void launch_node_down_cluster(const NodeBatch& nb, const SolveBufs& sb, bool root, int q0, int qc, cudaStream_t st);
// leaf LU fallback solves
void launch_leaf_lu_fwd(const LeafBatch& lb, const NodeBatch& fb, const int* leaf_idx, const double* B,
                        int64_t ldb, const SolveBufs& sb, cudaStream_t st);
void launch_leaf_lu_bwd(const LeafBatch& lb, const NodeBatch& fb, const int* leaf_idx, double* X,
                        int64_t ldx, const SolveBufs& sb, bool has_tin, cudaStream_t st);

// --- multi-RHS solve building blocks (solve_gemm.cu) ---
void launch_trsm_rhs(int w, bool upper, bool unit, const double* A, int64_t lda, int64_t sa, double* B, int64_t ldb,
                     int64_t sb, int ncols, int batch, cudaStream_t st);
void launch_leaf_gather(const LeafBatch& lb, const double* B, int64_t ldb, double* Z, int q, cudaStream_t st);
void launch_leaf_scatter(const LeafBatch& lb, const double* Z, double* X, int64_t ldx, int q, cudaStream_t st);
void launch_permute_rows(const NodeBatch& nb, const double* W, double* Y, int q, cudaStream_t st);
void launch_split_u(const NodeBatch& nb, const double* U, double* tin, int q, cudaStream_t st);

// --- compressed matvec (matvec_kernels.cu), hss_matvec compress.py:352-411 ---
void launch_mv_up_leaf(const DevTree& t, const LeafBatch& lb, const double* W, int64_t ldw, double* c, int S, int q,
                       cudaStream_t st);
void launch_mv_up_node(const DevTree& t, const NodeBatch& nb, double* c, int S, int q, cudaStream_t st);
void launch_mv_couple(const DevTree& t, const NodeBatch& nb, const double* c, double* inc, int S, int q,
                      cudaStream_t st);
void launch_mv_down(const DevTree& t, const NodeBatch& nb, const double* inc, double* tot, int S, int q, bool has_tot,
                    cudaStream_t st);
void launch_mv_leaf(const DevTree& t, const LeafBatch& lb, const double* W, int64_t ldw, const double* tot, double* Y,
                    int S, int q, bool has_tot, cudaStream_t st);

}  // namespace ks
