// Internal-node solve passes on 8-CTA thread-block clusters (sm_90+ clusters,
// DSMEM). One cluster per node: the skeleton-sized GEMVs are split across the
// cluster's CTAs, and the t x t triangular solves are blocked by 32 rows with
// the off-diagonal partial sums computed by all CTAs (column blocks dealt round
// robin), reduced into CTA 0 through distributed shared memory, and the solved
// block broadcast back to every CTA's copy of the vector. A single CTA per node
// was latency bound (one SM streaming a whole node's factors).
//
//   up   r1 = B c_r ; y2 = L^-1 Pi (B^T c_l - Y r1) ; c = P cc - P_l H_l r1 + L21 y2
//   down w2 = U^-1 (y2 + U12 t) ; w1 = r1 + P_l^T t - X w2 ; t_l, t_r = w1, w2
// (block formulation of the node factors, kernels.cuh NodeBatch)
// (reference: solver.py:216-237 in its O(N) telescoping form)
#include <cooperative_groups.h>

#include "kernels.cuh"
#include "trsv.cuh"

namespace cg = cooperative_groups;

namespace ks {

constexpr int CN = 8;  // CTAs per cluster (portable cluster size)

// The node's factor rows this pass reads, pulled into L2 at the start of the
// kernel (rows [r0, r1), columns [0, ncols) of the row-major matrix): the
// triangular solve below walks them block by block and would otherwise wait on
// an HBM round trip per block step. One prefetch per 128-byte line, spread over
// the cluster's threads.
// DESC: last rows first (the backward solve starts at the bottom).
__device__ __forceinline__ void l2_prefetch_rows(const double* A, int64_t lda, int r0, int r1, int ncols, int rank,
                                                 bool desc = false) {
  const int lines = (ncols + 15) / 16;
  const int total = (r1 - r0) * lines;
  for (int e = rank * STHREADS + threadIdx.x; e < total; e += CN * STHREADS) {
    const int r = desc ? r1 - 1 - e / lines : r0 + e / lines, c = (e % lines) * 16;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(A + (int64_t)r * lda + c));
  }
}

// Cluster-blocked triangular solve in place on every CTA's copy of x (n x QC):
// UPPER selects U (backward, non-unit) vs unit L (forward).
template <int QC, bool UPPER>
__device__ void cluster_trsv(cg::cluster_group& cl, const double* __restrict__ A, int64_t lda, int n, double* x,
                             double* part, double (*D)[SB + 1]) {
  const int rank = (int)cl.block_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = n / SB;
  double* part0 = cl.map_shared_rank(part, 0);
  for (int s = 0; s < nb; ++s) {
    const int bi = UPPER ? nb - 1 - s : s;
    const int r0 = bi * SB;
    double dreg[SB * SB / STHREADS];
    if (rank == 0) {
#pragma unroll
      for (int u = 0; u < SB * SB / STHREADS; ++u) {
        const int e = threadIdx.x + u * STHREADS;
        dreg[u] = A[(int64_t)(r0 + e / SB) * lda + r0 + e % SB];
      }
    }
    // partial sums over this CTA's column blocks: jb < bi (lower) or jb > bi (upper)
    double acc[4][QC];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int q = 0; q < QC; ++q) acc[i][q] = 0.0;
    const int rb = r0 + warp * 4;
    const int jb0 = UPPER ? bi + 1 : 0, jb1 = UPPER ? nb : bi;
    for (int jb = jb0 + ((rank - jb0) % CN + CN) % CN; jb < jb1; jb += CN) {
      const int c = jb * SB + lane;
      double a[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = __ldg(A + (int64_t)(rb + i) * lda + c);
#pragma unroll
      for (int q = 0; q < QC; ++q) {
        const double xv = x[c * QC + q];
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i][q] = fma(a[i], xv, acc[i][q]);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int q = 0; q < QC; ++q) {
        const double v = warp_sum(acc[i][q]);
        if (lane == 0) part0[(rank * SB + warp * 4 + i) * QC + q] = v;
      }
    if (rank == 0) {
#pragma unroll
      for (int u = 0; u < SB * SB / STHREADS; ++u) {
        const int e = threadIdx.x + u * STHREADS;
        D[e / SB][e % SB] = dreg[u];
      }
    }
    cl.sync();
    if (rank == 0 && warp == 0) {
      double v[QC];
#pragma unroll
      for (int q = 0; q < QC; ++q) {
        double sum = 0.0;
#pragma unroll
        for (int r = 0; r < CN; ++r) sum += part[(r * SB + lane) * QC + q];
        v[q] = x[(r0 + lane) * QC + q] - sum;
      }
      // 1 / pivot for this lane's row, started before the substitution chain
      // (a multiply in the chain instead of a division)
      const double rd = UPPER ? 1.0 / D[lane][lane] : 1.0;
#pragma unroll 4
      for (int s2 = 0; s2 < SB; ++s2) {
        const int c = UPPER ? SB - 1 - s2 : s2;
        if (UPPER && lane == c) {
#pragma unroll
          for (int q = 0; q < QC; ++q) v[q] *= rd;
        }
        const double dl = D[lane][c];
        const bool upd = UPPER ? (lane < c) : (lane > c);
#pragma unroll
        for (int q = 0; q < QC; ++q) {
          const double xc = __shfl_sync(0xffffffffu, v[q], c);
          if (upd) v[q] = fma(-dl, xc, v[q]);
        }
      }
#pragma unroll
      for (int r = 0; r < CN; ++r) {
        double* xr = cl.map_shared_rank(x, r);
#pragma unroll
        for (int q = 0; q < QC; ++q) xr[(r0 + lane) * QC + q] = v[q];
      }
    }
    cl.sync();
  }
}

// rows [r0, r1) of out = A x (+ out) for this CTA, then broadcast to every CTA's
// copy (dst_local + offset, ld QC) through DSMEM
template <int QC>
__device__ void cluster_rows_bcast(cg::cluster_group& cl, const double* __restrict__ A, int64_t lda, int r0, int r1,
                                   int ncols, const double* x, double* dst_local, bool accumulate) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int rb = r0 + warp * 4; rb < r1; rb += SWARPS * 4) {
    double acc[4][QC];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int q = 0; q < QC; ++q) acc[i][q] = 0.0;
    warp_rows4<QC>(A, lda, rb, r1, 0, ncols, x, acc);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int q = 0; q < QC; ++q) {
        const double v = warp_sum(acc[i][q]);
        if (lane < CN && rb + i < r1) {  // lane r writes CTA r's copy
          double* d = cl.map_shared_rank(dst_local, lane) + (rb + i) * QC + q;
          *d = accumulate ? *d + v : v;
        }
      }
  }
}

// rows [r0, r1) of -(A x) for this CTA, subtracted from every CTA's copy (DSMEM)
template <int QC>
__device__ void cluster_rows_sub(cg::cluster_group& cl, const double* __restrict__ A, int64_t lda, int r0, int r1,
                                 int ncols, const double* x, double* dst_local) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int rb = r0 + warp * 4; rb < r1; rb += SWARPS * 4) {
    double acc[4][QC];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int q = 0; q < QC; ++q) acc[i][q] = 0.0;
    warp_rows4<QC>(A, lda, rb, r1, 0, ncols, x, acc);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int q = 0; q < QC; ++q) {
        const double v = warp_sum(acc[i][q]);
        if (lane < CN && rb + i < r1) {
          double* d = cl.map_shared_rank(dst_local, lane) + (rb + i) * QC + q;
          *d -= v;
        }
      }
  }
}

// columns [rank*chunk, +chunk) of A^T x (A: nrows x ncols, ld lda) added to
// every CTA's copy of out (DSMEM); red: SWARPS x 32 x QC scratch
template <int QC>
__device__ void cluster_cols_add(cg::cluster_group& cl, const double* __restrict__ A, int64_t lda, int nrows,
                                 int chunk, const double* x, double* out, double* tmp, double* red) {
  const int rank = (int)cl.block_rank();
  for (int e = threadIdx.x; e < chunk * QC; e += STHREADS) tmp[e] = 0.0;
  __syncthreads();
  cta_gemv_cols<QC>(A + rank * chunk, lda, nrows, chunk, x, tmp, 1.0, red);
  for (int e = threadIdx.x; e < chunk * QC; e += STHREADS)
    for (int rr = 0; rr < CN; ++rr) cl.map_shared_rank(out, rr)[rank * chunk * QC + e] += tmp[e];
}

// up pass (block formulation): r1 = B c_r ; r2 = B^T c_l - Y r1 ; y2 = L^-1 Pi r2 ;
// y[node] = [r1; y2] ; c = P cc - (P_l H_l) r1 + L21 y2 (rows of c split over the cluster)
template <int QC>
__global__ void __cluster_dims__(CN, 1, 1) __launch_bounds__(STHREADS)
    k_node_up_cl(NodeBatch nb, SolveBufs sb, int q0, int root) {
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int k = blockIdx.x / CN;
  extern __shared__ double sm[];
  const int S = nb.s_pad, T = nb.T, ZT = nb.zt;
  double* cc = sm;                    // 2S x QC: [c_l; c_r]
  double* r = cc + ZT * QC;           // 2S x QC: [r1; r2 -> y2]
  double* nr = r + ZT * QC;           // S x QC: -r1, then scratch
  double* part = nr + S * QC;         // CN x SB x QC
  double* red = part + CN * SB * QC;  // SWARPS x 32 x QC
  __shared__ double D[SB][SB + 1];
  const int v = nb.node[k], l = nb.left[k], rch = nb.right[k];
  const double* A = nb.Aug + (int64_t)k * T * T;
  // L and L21 (columns [0, S) of every row)
  l2_prefetch_rows(A, T, 0, T, S, rank);
  const double* cl_ = sb.c + (int64_t)l * S * sb.q;
  const double* cr_ = sb.c + (int64_t)rch * S * sb.q;
  for (int e = threadIdx.x; e < S * QC; e += STHREADS) {
    const int i = e / QC, q = e % QC;
    cc[e] = cl_[(int64_t)i * sb.q + q0 + q];
    cc[S * QC + e] = cr_[(int64_t)i * sb.q + q0 + q];
  }
  cl.sync();  // every CTA of the cluster is running before any DSMEM write
  const double* Bc = nb.Bc + (int64_t)k * S * S;
  const double* X = nb.XY + (int64_t)k * 2 * S * S;
  const double* Y = X + (int64_t)S * S;
  const int chunk = S / CN;  // S is a multiple of 64
  double* r1 = r;
  double* r2 = r + S * QC;
  // r1 rows [rank*chunk, +chunk) = B c_r ; r2 columns [rank*chunk, +chunk) = B^T c_l
  cluster_rows_bcast<QC>(cl, Bc, S, rank * chunk, (rank + 1) * chunk, S, cc + S * QC, r1, false);
  {
    for (int e = threadIdx.x; e < chunk * QC; e += STHREADS) r2[(rank * chunk) * QC + e] = 0.0;
    __syncthreads();
    cta_gemv_cols<QC>(Bc + rank * chunk, S, S, chunk, cc, r2 + rank * chunk * QC, 1.0, red);
    for (int e = threadIdx.x; e < chunk * QC; e += STHREADS)
      for (int rr = 0; rr < CN; ++rr)
        if (rr != rank) cl.map_shared_rank(r2, rr)[rank * chunk * QC + e] = r2[rank * chunk * QC + e];
  }
  cl.sync();
  cluster_rows_sub<QC>(cl, Y, S, rank * chunk, (rank + 1) * chunk, S, r1, r2);  // r2 -= Y r1
  cl.sync();
  // y2 = Pi r2 (composed row interchanges of S), then L^-1
  const int* pm = nb.pm + (int64_t)k * S;
  for (int e = threadIdx.x; e < S * QC; e += STHREADS) nr[e] = r2[pm[e / QC] * QC + e % QC];
  __syncthreads();
  for (int e = threadIdx.x; e < S * QC; e += STHREADS) r2[e] = nr[e];
  __syncthreads();
  cluster_trsv<QC, false>(cl, A, T, S, r2, part, D);
  if (rank == 0) {
    double* yg = sb.y + (int64_t)(nb.first + k) * ZT * sb.q;
    for (int e = threadIdx.x; e < ZT * QC; e += STHREADS) yg[(e / QC) * sb.q + q0 + e % QC] = r[e];
  }
  if (!root) {  // c = P cc - (P_l H_l) r1 + L21 y2, rows of c split over the cluster
    for (int e = threadIdx.x; e < S * QC; e += STHREADS) nr[e] = -r1[e];
    __syncthreads();
    double* c = sb.c + (int64_t)v * S * sb.q + q0;
    const int c0 = rank * chunk;
    cta_gemv_rows<QC>(nb.Pn + (int64_t)k * S * ZT + (int64_t)c0 * ZT, ZT, chunk, ZT, cc, c + (int64_t)c0 * sb.q, sb.q,
                      false);
    __syncthreads();
    cta_gemv_rows<QC>(nb.PHl + (int64_t)k * S * S + (int64_t)c0 * S, S, chunk, S, nr, c + (int64_t)c0 * sb.q, sb.q,
                      true);
    __syncthreads();
    cta_gemv_rows<QC>(A + (int64_t)(S + c0) * T, T, chunk, S, r2, c + (int64_t)c0 * sb.q, sb.q, true);
  }
  cl.sync();  // keep every CTA's shared memory alive until remote writes are done
}

// down pass: y2 += U12 t, r1 += P_l^T t (not at the root); w2 = U^-1 y2 ;
// w1 = r1 - X w2 ; the children receive w1 (left) and w2 (right)
template <int QC>
__global__ void __cluster_dims__(CN, 1, 1) __launch_bounds__(STHREADS)
    k_node_down_cl(NodeBatch nb, SolveBufs sb, int q0, int root) {
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int k = blockIdx.x / CN;
  extern __shared__ double sm[];
  const int S = nb.s_pad, T = nb.T, ZT = nb.zt;
  double* u = sm;                     // 2S x QC: [r1; y2]
  double* tv = u + ZT * QC;           // S x QC
  double* tmp = tv + S * QC;          // S x QC
  double* part = tmp + S * QC;        // CN x SB x QC
  double* red = part + CN * SB * QC;  // SWARPS x 32 x QC
  __shared__ double D[SB][SB + 1];
  const int v = nb.node[k], l = nb.left[k], r = nb.right[k];
  const double* A = nb.Aug + (int64_t)k * T * T;
  // U and U12: the first S rows, all T columns
  l2_prefetch_rows(A, T, 0, S, T, rank, true);
  const double* yg = sb.y + (int64_t)(nb.first + k) * ZT * sb.q;
  for (int e = threadIdx.x; e < ZT * QC; e += STHREADS) u[e] = yg[(e / QC) * sb.q + q0 + e % QC];
  if (!root) {
    const double* ti = sb.tin + (int64_t)v * S * sb.q;
    for (int e = threadIdx.x; e < S * QC; e += STHREADS) tv[e] = ti[(e / QC) * sb.q + q0 + e % QC];
  }
  cl.sync();  // every CTA of the cluster is running before any DSMEM write
  double* u1 = u;
  double* u2 = u + S * QC;
  const int chunk = S / CN;
  if (!root) {
    cluster_rows_bcast<QC>(cl, A + S, T, rank * chunk, (rank + 1) * chunk, S, tv, u2, true);  // y2 += U12 t
    cluster_cols_add<QC>(cl, nb.Pn + (int64_t)k * S * ZT, ZT, S, chunk, tv, u1, tmp, red);    // r1 += P_l^T t
  }
  cl.sync();
  cluster_trsv<QC, true>(cl, A, T, S, u2, part, D);
  const double* X = nb.XY + (int64_t)k * 2 * S * S;
  cluster_rows_sub<QC>(cl, X, S, rank * chunk, (rank + 1) * chunk, S, u2, u1);  // w1 = r1 - X w2
  cl.sync();
  if (rank == 0) {
    double* tl = sb.tin + (int64_t)l * S * sb.q;
    double* tr = sb.tin + (int64_t)r * S * sb.q;
    for (int e = threadIdx.x; e < S * QC; e += STHREADS) {
      const int i = e / QC, q = e % QC;
      tl[(int64_t)i * sb.q + q0 + q] = u1[e];
      tr[(int64_t)i * sb.q + q0 + q] = u2[e];
    }
  }
  cl.sync();
}

template <typename K>
static void set_attr(K kern, size_t bytes) {
  ensure_smem(kern, bytes);
}

void launch_node_up_cluster(const NodeBatch& nb, const SolveBufs& sb, bool root, int q0, int qc, cudaStream_t st) {
  const size_t smem = ((size_t)2 * nb.zt + nb.s_pad + CN * SB + SWARPS * 32) * qc * sizeof(double);
#define KS_CASE(QC)                                                                          \
  if (qc == QC) {                                                                            \
    set_attr(k_node_up_cl<QC>, smem);                                                        \
    k_node_up_cl<QC><<<nb.count * CN, STHREADS, smem, st>>>(nb, sb, q0, root ? 1 : 0);       \
    return;                                                                                  \
  }
  KS_CASE(1) KS_CASE(2) KS_CASE(4)
#undef KS_CASE
}

void launch_node_down_cluster(const NodeBatch& nb, const SolveBufs& sb, bool root, int q0, int qc, cudaStream_t st) {
  const size_t smem = ((size_t)nb.zt + 2 * nb.s_pad + CN * SB + SWARPS * 32) * qc * sizeof(double);
#define KS_CASE(QC)                                                                          \
  if (qc == QC) {                                                                            \
    set_attr(k_node_down_cl<QC>, smem);                                                      \
    k_node_down_cl<QC><<<nb.count * CN, STHREADS, smem, st>>>(nb, sb, q0, root ? 1 : 0);     \
    return;                                                                                  \
  }
  KS_CASE(1) KS_CASE(2) KS_CASE(4)
#undef KS_CASE
}

}  // namespace ks
