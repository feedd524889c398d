// Telescoping solve on the stored factors (replaces the reference's recursive
// _solve_node, solver.py:216-237, which visits a level-l node 2^l times; the
// up/down form below visits every node once).
//
//   up   leaf  z = L^-1 b ;  c = L21 z                     (= P A^-1 b)
//        node  r1 = B c_r ; y2 = L^-1 Pi (B^T c_l - Y r1) ; c = P cc - P_l H_l r1 + L21 y2
//   down node  w2 = U^-1 (y2 + U12 t) ; w1 = r1 + P_l^T t - X w2 ; t_l, t_r = w1, w2
//        leaf  x = L^-T (z - L21^T t)
// (node factors in the block formulation of kernels.cuh NodeBatch: Z^-1 through
// Z = [[I, 0], [Y, I]] [[I, X], [0, S]] and the LU of S)
//
// Every kernel streams its node's factor rows once, coalesced along rows, with
// warp-shuffle reductions; right-hand sides are processed QC columns at a time.
#include <utility>
#include <vector>

#include "kernels.cuh"
#include "trsv.cuh"

namespace ks {

// ---------------------------------------------------------------------------
// leaf up: z = L^-1 b, c = L21 z
// ---------------------------------------------------------------------------
template <int QC>
__global__ void __launch_bounds__(STHREADS, 8) k_leaf_fwd(LeafBatch lb, const double* B, int64_t ldb, SolveBufs sb,
                                                        int q0) {
  extern __shared__ double x[];  // m_pad x QC
  __shared__ double D[SB][SB + 1];
  const int leaf = blockIdx.x;
  const int node = lb.node[leaf], begin = lb.begin[leaf], m = lb.size[leaf];
  const int M = lb.m_pad;
  const double* A = lb.A + (int64_t)leaf * lb.a_stride;
  for (int e = threadIdx.x; e < M * QC; e += STHREADS) {
    const int r = e / QC, q = e % QC;
    x[e] = (r < m) ? B[(int64_t)(begin + r) * ldb + q0 + q] : 0.0;
  }
  __syncthreads();
  cta_trsv_rows<QC, false, false>(A, M, M, x, D);
  double* z = sb.z + (int64_t)leaf * M * sb.q;
  for (int e = threadIdx.x; e < M * QC; e += STHREADS) z[(e / QC) * sb.q + q0 + e % QC] = x[e];
  if (lb.s_pad > 0) {
    double* c = sb.c + (int64_t)node * lb.s_pad * sb.q + q0;
    cta_gemv_rows<QC>(A + (int64_t)M * M, M, lb.s_pad, M, x, c, sb.q, false);
  }
}

// ---------------------------------------------------------------------------
// leaf down: x = L^-T (z - L21^T t)
// ---------------------------------------------------------------------------
template <int QC>
__global__ void __launch_bounds__(STHREADS, 8) k_leaf_bwd(LeafBatch lb, double* X, int64_t ldx, SolveBufs sb, int q0,
                                                        int has_tin) {
  extern __shared__ double sm[];
  double* x = sm;                       // m_pad x QC
  double* tv = sm + lb.m_pad * QC;      // s_pad x QC
  double* red = tv + lb.s_pad * QC;     // SWARPS x 32 x QC
  __shared__ double D[SB][SB + 1];
  const int leaf = blockIdx.x;
  const int node = lb.node[leaf], begin = lb.begin[leaf], m = lb.size[leaf];
  const int M = lb.m_pad, S = lb.s_pad;
  const double* A = lb.A + (int64_t)leaf * lb.a_stride;
  const double* z = sb.z + (int64_t)leaf * M * sb.q;
  for (int e = threadIdx.x; e < M * QC; e += STHREADS) x[e] = z[(e / QC) * sb.q + q0 + e % QC];
  if (has_tin) {
    const double* ti = sb.tin + (int64_t)node * S * sb.q;
    for (int e = threadIdx.x; e < S * QC; e += STHREADS) tv[e] = ti[(e / QC) * sb.q + q0 + e % QC];
  }
  __syncthreads();
  if (has_tin) cta_gemv_cols<QC>(A + (int64_t)M * M, M, S, M, tv, x, -1.0, red);
  cta_trsv_trans<QC, false, false>(A, M, M, x, D, red);  // L^T x = r
  for (int e = threadIdx.x; e < m * QC; e += STHREADS) X[(int64_t)(begin + e / QC) * ldx + q0 + e % QC] = x[e];
}

// ---------------------------------------------------------------------------
// internal node up (block formulation, kernels.cuh NodeBatch):
//   r1 = B c_r ;  r2 = B^T c_l - Y r1 ;  y2 = L^-1 Pi r2
//   y[node] = [r1; y2] ;  c = P cc - (P_l H_l) r1 + L21 y2
// ---------------------------------------------------------------------------
template <int QC>
__global__ void __launch_bounds__(STHREADS) k_node_up(NodeBatch nb, SolveBufs sb, int q0, int root) {
  extern __shared__ double sm[];
  const int S = nb.s_pad, T = nb.T, ZT = nb.zt;
  double* cc = sm;               // 2S x QC: [c_l; c_r]
  double* r = cc + ZT * QC;      // 2S x QC: [r1; r2 -> y2]
  double* tq = r + ZT * QC;      // S x QC: Y r1, then -r1
  double* red = tq + S * QC;     // SWARPS x 32 x QC
  __shared__ double D[SB][SB + 1];
  const int k = blockIdx.x;
  const int v = nb.node[k], l = nb.left[k], rr = nb.right[k];
  const double* cl = sb.c + (int64_t)l * S * sb.q;
  const double* cr = sb.c + (int64_t)rr * S * sb.q;
  for (int e = threadIdx.x; e < S * QC; e += STHREADS) {
    const int i = e / QC, q = e % QC;
    cc[e] = cl[(int64_t)i * sb.q + q0 + q];
    cc[S * QC + e] = cr[(int64_t)i * sb.q + q0 + q];
    r[S * QC + e] = 0.0;
  }
  __syncthreads();
  const double* Bc = nb.Bc + (int64_t)k * S * S;
  double* r1 = r;
  double* r2 = r + S * QC;
  cta_gemv_rows<QC>(Bc, S, S, S, cc + S * QC, r1, QC, false);   // B c_r
  cta_gemv_cols<QC>(Bc, S, S, S, cc, r2, 1.0, red);              // B^T c_l
  __syncthreads();
  const double* X = nb.XY + (int64_t)k * 2 * S * S;
  const double* Y = X + (int64_t)S * S;
  cta_gemv_rows<QC>(Y, S, S, S, r1, tq, QC, false);              // Y r1
  __syncthreads();
  for (int e = threadIdx.x; e < S * QC; e += STHREADS) r2[e] -= tq[e];
  __syncthreads();
  {  // Pi r2 through S's composed row interchanges (tq as scratch)
    const int* pm = nb.pm + (int64_t)k * S;
    for (int e = threadIdx.x; e < S * QC; e += STHREADS) tq[e] = r2[pm[e / QC] * QC + e % QC];
    __syncthreads();
    for (int e = threadIdx.x; e < S * QC; e += STHREADS) r2[e] = tq[e];
  }
  __syncthreads();
  const double* A = nb.Aug + (int64_t)k * T * T;
  cta_trsv_rows<QC, false, true>(A, T, S, r2, D);                // y2 = L^-1 Pi r2
  double* y = sb.y + (int64_t)(nb.first + k) * ZT * sb.q;
  for (int e = threadIdx.x; e < ZT * QC; e += STHREADS) y[(e / QC) * sb.q + q0 + e % QC] = r[e];
  if (!root) {
    for (int e = threadIdx.x; e < S * QC; e += STHREADS) tq[e] = -r1[e];
    double* c = sb.c + (int64_t)v * S * sb.q + q0;
    cta_gemv_rows<QC>(nb.Pn + (int64_t)k * S * ZT, ZT, S, ZT, cc, c, sb.q, false);
    __syncthreads();
    cta_gemv_rows<QC>(nb.PHl + (int64_t)k * S * S, S, S, S, tq, c, sb.q, true);
    __syncthreads();
    cta_gemv_rows<QC>(A + (int64_t)S * T, T, S, S, r2, c, sb.q, true);
  }
}

// ---------------------------------------------------------------------------
// internal node down: y2 += U12 t, r1 += P_l^T t (not at the root);
//   w2 = U^-1 y2 ;  w1 = r1 - X w2 ;  the children receive w1 (left), w2 (right)
// ---------------------------------------------------------------------------
template <int QC>
__global__ void __launch_bounds__(STHREADS) k_node_down(NodeBatch nb, SolveBufs sb, int q0, int root) {
  extern __shared__ double sm[];
  const int S = nb.s_pad, T = nb.T, ZT = nb.zt;
  double* u = sm;                 // 2S x QC: [r1; y2]
  double* tv = u + ZT * QC;       // S x QC: incoming t, then X w2
  double* red = tv + S * QC;      // SWARPS x 32 x QC
  __shared__ double D[SB][SB + 1];
  const int k = blockIdx.x;
  const int v = nb.node[k], l = nb.left[k], r = nb.right[k];
  const double* y = sb.y + (int64_t)(nb.first + k) * ZT * sb.q;
  for (int e = threadIdx.x; e < ZT * QC; e += STHREADS) u[e] = y[(e / QC) * sb.q + q0 + e % QC];
  if (!root) {
    const double* ti = sb.tin + (int64_t)v * S * sb.q;
    for (int e = threadIdx.x; e < S * QC; e += STHREADS) tv[e] = ti[(e / QC) * sb.q + q0 + e % QC];
  }
  __syncthreads();
  const double* A = nb.Aug + (int64_t)k * T * T;
  double* u1 = u;
  double* u2 = u + S * QC;
  if (!root) {
    cta_gemv_rows<QC>(A + S, T, S, S, tv, u2, QC, true);                      // y2 += U12 t
    cta_gemv_cols<QC>(nb.Pn + (int64_t)k * S * ZT, ZT, S, S, tv, u1, 1.0, red);  // r1 += P_l^T t
    __syncthreads();
  }
  cta_trsv_rows<QC, true, false>(A, T, S, u2, D);                             // w2 = U^-1 y2
  const double* X = nb.XY + (int64_t)k * 2 * S * S;
  cta_gemv_rows<QC>(X, S, S, S, u2, tv, QC, false);                           // X w2
  __syncthreads();
  double* tl = sb.tin + (int64_t)l * S * sb.q;
  double* tr = sb.tin + (int64_t)r * S * sb.q;
  for (int e = threadIdx.x; e < S * QC; e += STHREADS) {
    const int i = e / QC, q = e % QC;
    tl[(int64_t)i * sb.q + q0 + q] = u1[e] - tv[e];
    tr[(int64_t)i * sb.q + q0 + q] = u2[e];
  }
}

// ---------------------------------------------------------------------------
// launchers: RHS columns in chunks of QC (largest of 4, 2, 1 dividing q)
// ---------------------------------------------------------------------------
template <typename F>
static void for_chunks(int q, F f) {
  int q0 = 0;
  while (q0 < q) {
    const int rem = q - q0;
    const int qc = rem >= 4 ? 4 : (rem >= 2 ? 2 : 1);
    f(q0, qc);
    q0 += qc;
  }
}

template <typename K>
static void set_smem(K kern, size_t bytes) {
  ensure_smem(kern, bytes, 100);
}

void launch_leaf_fwd(const LeafBatch& lb, const double* B, int64_t ldb, const SolveBufs& sb, cudaStream_t st) {
  for_chunks(sb.q, [&](int q0, int qc) {
    const size_t smem = (size_t)lb.m_pad * qc * sizeof(double);
#define KS_CASE(QC)                                                  \
  if (qc == QC) {                                                    \
    set_smem(k_leaf_fwd<QC>, smem);                                  \
    k_leaf_fwd<QC><<<lb.count, STHREADS, smem, st>>>(lb, B, ldb, sb, q0); \
  }
    KS_CASE(1) KS_CASE(2) KS_CASE(4)
#undef KS_CASE
  });
}

void launch_leaf_bwd(const LeafBatch& lb, double* X, int64_t ldx, const SolveBufs& sb, bool has_tin,
                     cudaStream_t st) {
  for_chunks(sb.q, [&](int q0, int qc) {
    const size_t smem = ((size_t)lb.m_pad + lb.s_pad + SWARPS * 32) * qc * sizeof(double);
#define KS_CASE(QC)                                                                  \
  if (qc == QC) {                                                                    \
    set_smem(k_leaf_bwd<QC>, smem);                                                  \
    k_leaf_bwd<QC><<<lb.count, STHREADS, smem, st>>>(lb, X, ldx, sb, q0, has_tin ? 1 : 0); \
  }
    KS_CASE(1) KS_CASE(2) KS_CASE(4)
#undef KS_CASE
  });
}

// ---------------------------------------------------------------------------
// LU-fallback leaves (augmented [[A, -P^T], [P, 0]] factors, see k_fb_assemble):
//   up   y = L^-1 Pi b_leaf,  c = L21aug y           (= P A^-1 b)
//   down x = U^-1 (y + U12aug t)                     (= A^-1 (b - P^T t))
// ---------------------------------------------------------------------------
template <int QC>
__global__ void __launch_bounds__(STHREADS) k_fb_up(NodeBatch fb, const int* begin, const int* size, const double* B,
                                                     int64_t ldb, double* Y, double* c, int q, int q0) {
  extern __shared__ double sm[];
  const int TP = fb.t_pad, T = fb.T, S = T - TP;
  double* w = sm;            // TP x QC
  double* x = sm + TP * QC;  // TP x QC
  __shared__ double D[SB][SB + 1];
  const int k = blockIdx.x;
  const int b0 = begin[k], m = size[k], v = fb.node[k];
  for (int e = threadIdx.x; e < TP * QC; e += STHREADS) {
    const int r = e / QC;
    w[e] = (r < m) ? B[(int64_t)(b0 + r) * ldb + q0 + e % QC] : 0.0;
  }
  __syncthreads();
  const int* pm = fb.pm + (int64_t)k * TP;
  for (int e = threadIdx.x; e < TP * QC; e += STHREADS) x[e] = w[pm[e / QC] * QC + e % QC];
  __syncthreads();
  const double* A = fb.Aug + (int64_t)k * T * T;
  cta_trsv_rows<QC, false, true>(A, T, TP, x, D);
  double* y = Y + (int64_t)k * TP * q;
  for (int e = threadIdx.x; e < TP * QC; e += STHREADS) y[(e / QC) * q + q0 + e % QC] = x[e];
  if (S > 0) cta_gemv_rows<QC>(A + (int64_t)TP * T, T, S, TP, x, c + (int64_t)v * S * q + q0, q, false);
}

template <int QC>
__global__ void __launch_bounds__(STHREADS) k_fb_down(NodeBatch fb, const int* begin, const int* size, const double* Y,
                                                       const double* tin, double* X, int64_t ldx, int q, int q0,
                                                       int has_tin) {
  extern __shared__ double sm[];
  const int TP = fb.t_pad, T = fb.T, S = T - TP;
  double* u = sm;            // TP x QC
  double* tv = sm + TP * QC;  // S x QC
  __shared__ double D[SB][SB + 1];
  const int k = blockIdx.x;
  const int b0 = begin[k], m = size[k], v = fb.node[k];
  const double* y = Y + (int64_t)k * TP * q;
  for (int e = threadIdx.x; e < TP * QC; e += STHREADS) u[e] = y[(e / QC) * q + q0 + e % QC];
  if (has_tin)
    for (int e = threadIdx.x; e < S * QC; e += STHREADS) tv[e] = tin[((int64_t)v * S + e / QC) * q + q0 + e % QC];
  __syncthreads();
  const double* A = fb.Aug + (int64_t)k * T * T;
  if (has_tin && S > 0) {
    cta_gemv_rows<QC>(A + TP, T, TP, S, tv, u, QC, true);
    __syncthreads();
  }
  cta_trsv_rows<QC, true, false>(A, T, TP, u, D);
  for (int e = threadIdx.x; e < m * QC; e += STHREADS) X[(int64_t)(b0 + e / QC) * ldx + q0 + e % QC] = u[e];
}

void launch_fb_up(const NodeBatch& fb, const int* begin, const int* size, const double* B, int64_t ldb, double* Y,
                  double* c, int q, cudaStream_t st) {
  for_chunks(q, [&](int q0, int qc) {
    const size_t smem = (size_t)2 * fb.t_pad * qc * sizeof(double);
#define KS_CASE(QC)                                                                             \
  if (qc == QC) {                                                                               \
    set_smem(k_fb_up<QC>, smem);                                                                \
    k_fb_up<QC><<<fb.count, STHREADS, smem, st>>>(fb, begin, size, B, ldb, Y, c, q, q0);        \
  }
    KS_CASE(1) KS_CASE(2) KS_CASE(4)
#undef KS_CASE
  });
}

void launch_fb_down(const NodeBatch& fb, const int* begin, const int* size, const double* Y, const double* tin,
                    double* X, int64_t ldx, int q, bool has_tin, cudaStream_t st) {
  for_chunks(q, [&](int q0, int qc) {
    const size_t smem = ((size_t)fb.t_pad + (fb.T - fb.t_pad)) * qc * sizeof(double);
#define KS_CASE(QC)                                                                                          \
  if (qc == QC) {                                                                                            \
    set_smem(k_fb_down<QC>, smem);                                                                           \
    k_fb_down<QC><<<fb.count, STHREADS, smem, st>>>(fb, begin, size, Y, tin, X, ldx, q, q0, has_tin ? 1 : 0); \
  }
    KS_CASE(1) KS_CASE(2) KS_CASE(4)
#undef KS_CASE
  });
}

// Levels with many nodes keep one CTA per node (enough CTAs to saturate HBM);
// levels with few nodes use an 8-CTA cluster per node (solve_cluster.cu).
constexpr int kClusterMaxNodes = 128;

void launch_node_up(const NodeBatch& nb, const SolveBufs& sb, bool root, cudaStream_t st) {
  for_chunks(sb.q, [&](int q0, int qc) {
    if (nb.count <= kClusterMaxNodes) {
      launch_node_up_cluster(nb, sb, root, q0, qc, st);
      return;
    }
    const size_t smem = ((size_t)2 * nb.zt + nb.s_pad + SWARPS * 32) * qc * sizeof(double);
#define KS_CASE(QC)                                                                 \
  if (qc == QC) {                                                                   \
    set_smem(k_node_up<QC>, smem);                                                  \
    k_node_up<QC><<<nb.count, STHREADS, smem, st>>>(nb, sb, q0, root ? 1 : 0);      \
  }
    KS_CASE(1) KS_CASE(2) KS_CASE(4)
#undef KS_CASE
  });
}

void launch_node_down(const NodeBatch& nb, const SolveBufs& sb, bool root, cudaStream_t st) {
  for_chunks(sb.q, [&](int q0, int qc) {
    if (nb.count <= kClusterMaxNodes) {
      launch_node_down_cluster(nb, sb, root, q0, qc, st);
      return;
    }
    const size_t smem = ((size_t)nb.zt + nb.s_pad + SWARPS * 32) * qc * sizeof(double);
#define KS_CASE(QC)                                                                 \
  if (qc == QC) {                                                                   \
    set_smem(k_node_down<QC>, smem);                                                \
    k_node_down<QC><<<nb.count, STHREADS, smem, st>>>(nb, sb, q0, root ? 1 : 0);    \
  }
    KS_CASE(1) KS_CASE(2) KS_CASE(4)
#undef KS_CASE
  });
}

}  // namespace ks
