// Internal-node solve passes on 8-CTA thread-block clusters (sm_90+ clusters,
// DSMEM). One cluster per node: the skeleton-sized GEMVs are split across the
// cluster's CTAs, and the t x t triangular solves are blocked by 32 rows with
// the off-diagonal partial sums computed by all CTAs (column blocks dealt round
// robin), reduced into CTA 0 through distributed shared memory, and the solved
// block broadcast back to every CTA's copy of the vector. A single CTA per node
// was latency bound (one SM streaming a whole node's factors).
//
//   up   w = [B c_r ; B^T c_l] ;  y = L^-1 Pi w ;  c = P cc + L21aug y
//   down u = U^-1 (y + U12aug t) ;  t_l, t_r = split(u)
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

template <int QC>
__global__ void __cluster_dims__(CN, 1, 1) __launch_bounds__(STHREADS)
    k_node_up_cl(NodeBatch nb, SolveBufs sb, int q0, int root) {
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int k = blockIdx.x / CN;
  extern __shared__ double sm[];
  const int S = nb.s_pad, TP = nb.t_pad, T = nb.T;
  double* cc = sm;                  // TP x QC
  double* w = cc + TP * QC;         // TP x QC
  double* y = w + TP * QC;          // TP x QC
  double* part = y + TP * QC;       // CN x SB x QC
  double* red = part + CN * SB * QC;  // SWARPS x 32 x QC
  __shared__ double D[SB][SB + 1];
  const int v = nb.node[k], l = nb.left[k], r = nb.right[k];
  // L (rows < TP, columns < TP) and L21aug (rows >= TP): columns [0, TP) of every row
  l2_prefetch_rows(nb.Aug + (int64_t)k * T * T, T, 0, T, TP, rank);
  const double* cl_ = sb.c + (int64_t)l * S * sb.q;
  const double* cr_ = sb.c + (int64_t)r * S * sb.q;
  for (int e = threadIdx.x; e < S * QC; e += STHREADS) {
    const int i = e / QC, q = e % QC;
    cc[e] = cl_[(int64_t)i * sb.q + q0 + q];
    cc[S * QC + e] = cr_[(int64_t)i * sb.q + q0 + q];
  }
  cl.sync();  // every CTA of the cluster is running before any DSMEM write
  const double* Bc = nb.Bc + (int64_t)k * S * S;
  const int chunk = S / CN;  // S is a multiple of 64
  // w_top rows [rank*chunk, +chunk) = B c_r ; w_bot cols [rank*chunk, +chunk) = B^T c_l
  cluster_rows_bcast<QC>(cl, Bc, S, rank * chunk, (rank + 1) * chunk, S, cc + S * QC, w, false);
  {
    double* wb = w + S * QC;
    for (int e = threadIdx.x; e < chunk * QC; e += STHREADS) wb[(rank * chunk) * QC + e] = 0.0;
    __syncthreads();
    cta_gemv_cols<QC>(Bc + rank * chunk, S, S, chunk, cc, wb + rank * chunk * QC, 1.0, red);
    for (int e = threadIdx.x; e < chunk * QC; e += STHREADS)
      for (int rr = 0; rr < CN; ++rr)
        if (rr != rank) cl.map_shared_rank(wb, rr)[rank * chunk * QC + e] = wb[rank * chunk * QC + e];
  }
  cl.sync();
  // y = Pi w (composed row interchanges), then L^-1
  const int* pm = nb.pm + (int64_t)k * TP;
  for (int e = threadIdx.x; e < TP * QC; e += STHREADS) y[e] = w[pm[e / QC] * QC + e % QC];
  __syncthreads();
  const double* A = nb.Aug + (int64_t)k * T * T;
  cluster_trsv<QC, false>(cl, A, T, TP, y, part, D);
  if (rank == 0) {
    double* yg = sb.y + (int64_t)(nb.first + k) * TP * sb.q;
    for (int e = threadIdx.x; e < TP * QC; e += STHREADS) yg[(e / QC) * sb.q + q0 + e % QC] = y[e];
  }
  if (!root) {  // c = P cc + L21aug y, rows of c split over the cluster
    double* c = sb.c + (int64_t)v * S * sb.q + q0;
    const int r0 = rank * chunk;
    cta_gemv_rows<QC>(nb.Pn + (int64_t)k * S * TP + (int64_t)r0 * TP, TP, chunk, TP, cc, c + (int64_t)r0 * sb.q,
                      sb.q, false);
    __syncthreads();
    cta_gemv_rows<QC>(A + (int64_t)(TP + r0) * T, T, chunk, TP, y, c + (int64_t)r0 * sb.q, sb.q, true);
  }
  cl.sync();  // keep every CTA's shared memory alive until remote writes are done
}

template <int QC>
__global__ void __cluster_dims__(CN, 1, 1) __launch_bounds__(STHREADS)
    k_node_down_cl(NodeBatch nb, SolveBufs sb, int q0, int root) {
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int k = blockIdx.x / CN;
  extern __shared__ double sm[];
  const int S = nb.s_pad, TP = nb.t_pad, T = nb.T;
  double* u = sm;                // TP x QC
  double* tv = u + TP * QC;      // S x QC
  double* part = tv + S * QC;    // CN x SB x QC
  __shared__ double D[SB][SB + 1];
  const int v = nb.node[k], l = nb.left[k], r = nb.right[k];
  // U and U12aug: the first TP rows, all T columns
  l2_prefetch_rows(nb.Aug + (int64_t)k * T * T, T, 0, TP, T, rank, true);
  const double* yg = sb.y + (int64_t)(nb.first + k) * TP * sb.q;
  for (int e = threadIdx.x; e < TP * QC; e += STHREADS) u[e] = yg[(e / QC) * sb.q + q0 + e % QC];
  if (!root) {
    const double* ti = sb.tin + (int64_t)v * S * sb.q;
    for (int e = threadIdx.x; e < S * QC; e += STHREADS) tv[e] = ti[(e / QC) * sb.q + q0 + e % QC];
  }
  cl.sync();  // every CTA of the cluster is running before any DSMEM write
  const double* A = nb.Aug + (int64_t)k * T * T;
  if (!root) {  // u += U12aug t, rows split over the cluster and broadcast
    const int chunk = TP / CN;
    cluster_rows_bcast<QC>(cl, A + TP, T, rank * chunk, (rank + 1) * chunk, S, tv, u, true);
  }
  cl.sync();
  cluster_trsv<QC, true>(cl, A, T, TP, u, part, D);
  if (rank == 0) {
    double* tl = sb.tin + (int64_t)l * S * sb.q;
    double* tr = sb.tin + (int64_t)r * S * sb.q;
    for (int e = threadIdx.x; e < S * QC; e += STHREADS) {
      const int i = e / QC, q = e % QC;
      tl[(int64_t)i * sb.q + q0 + q] = u[e];
      tr[(int64_t)i * sb.q + q0 + q] = u[S * QC + e];
    }
  }
  cl.sync();
}

template <typename K>
static void set_attr(K kern, size_t bytes) {
  ensure_smem(kern, bytes);
}

void launch_node_up_cluster(const NodeBatch& nb, const SolveBufs& sb, bool root, int q0, int qc, cudaStream_t st) {
  const size_t smem = ((size_t)3 * nb.t_pad + CN * SB + SWARPS * 32) * qc * sizeof(double);
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
  const size_t smem = ((size_t)nb.t_pad + nb.s_pad + CN * SB) * qc * sizeof(double);
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
