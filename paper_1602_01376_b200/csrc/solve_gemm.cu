// Multi-right-hand-side solve building blocks (q >= 8): with many columns the
// telescoping solve is fp64-bound rather than HBM-bound (240
// GFLOP at config 3, q = 32), so the factors are applied as DMMA GEMMs: the
// leaf triangles block by block through their 64x64 diagonal inverses, the
// node triangles through a recursive TRSM whose base case is below. The small
// kernels move right-hand-side blocks between the n x q layout and the per-node
// scratch buffers.
#include "kernels.cuh"

namespace ks {

// B[b] (W x ncols, ld ldb) := op(T)^-1 B[b] for the W x W triangle T[b] (ld lda):
// lower (forward) or upper (backward), unit diagonal or not. One thread per
// column, the column in registers, four partial sums per row (DFMA latency).
template <int W, bool UPPER, bool UNIT>
__global__ void __launch_bounds__(128) k_trsm_rhs(const double* A, int64_t lda, int64_t sa, double* B, int64_t ldb,
                                                 int64_t sb, int ncols) {
  __shared__ double L[W][W + 1];
  __shared__ double rdiag[W];  // 1 / diagonal, formed once (a multiply in the chain)
  const int b = blockIdx.y;
  const double* T = A + (int64_t)b * sa;
  for (int e = threadIdx.x; e < W * W; e += blockDim.x) L[e / W][e % W] = T[(int64_t)(e / W) * lda + e % W];
  if (!UNIT)
    for (int i = threadIdx.x; i < W; i += blockDim.x) rdiag[i] = 1.0 / T[(int64_t)i * lda + i];
  __syncthreads();
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= ncols) return;
  double* X = B + (int64_t)b * sb + col;
  double x[W];
#pragma unroll
  for (int i = 0; i < W; ++i) x[i] = X[(int64_t)i * ldb];
#pragma unroll
  for (int s = 0; s < W; ++s) {
    const int i = UPPER ? W - 1 - s : s;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    if (!UPPER) {
#pragma unroll
      for (int j = 0; j + 3 < i; j += 4) {
        s0 = fma(L[i][j], x[j], s0);
        s1 = fma(L[i][j + 1], x[j + 1], s1);
        s2 = fma(L[i][j + 2], x[j + 2], s2);
        s3 = fma(L[i][j + 3], x[j + 3], s3);
      }
#pragma unroll
      for (int j = i & ~3; j < i; ++j) s0 = fma(L[i][j], x[j], s0);
    } else {
#pragma unroll
      for (int j = i + 1; j + 3 < W; j += 4) {
        s0 = fma(L[i][j], x[j], s0);
        s1 = fma(L[i][j + 1], x[j + 1], s1);
        s2 = fma(L[i][j + 2], x[j + 2], s2);
        s3 = fma(L[i][j + 3], x[j + 3], s3);
      }
#pragma unroll
      for (int j = (W - ((W - i - 1) & 3)); j < W; ++j)
        if (j > i) s0 = fma(L[i][j], x[j], s0);
    }
    double v = x[i] - ((s0 + s1) + (s2 + s3));
    if (!UNIT) v *= rdiag[i];
    x[i] = v;
  }
#pragma unroll
  for (int i = 0; i < W; ++i) X[(int64_t)i * ldb] = x[i];
}

void launch_trsm_rhs(int w, bool upper, bool unit, const double* A, int64_t lda, int64_t sa, double* B, int64_t ldb,
                     int64_t sb, int ncols, int batch, cudaStream_t st) {
  dim3 g((ncols + 127) / 128, batch);
#define KS_T(W_, U_, N_) \
  if (w == W_ && upper == U_ && unit == N_) { k_trsm_rhs<W_, U_, N_><<<g, 128, 0, st>>>(A, lda, sa, B, ldb, sb, ncols); return; }
  KS_T(64, false, true) KS_T(64, true, false) KS_T(32, false, true) KS_T(32, true, false)
  KS_T(16, false, true) KS_T(16, true, false) KS_T(8, false, true) KS_T(8, true, false)
#undef KS_T
}

// Z[leaf] (m_pad x q) <- rows [begin, begin+m) of B (ld ldb), zero padded
__global__ void k_leaf_gather(LeafBatch lb, const double* B, int64_t ldb, double* Z, int q) {
  const int leaf = blockIdx.y;
  const int begin = lb.begin[leaf], m = lb.size[leaf];
  double* z = Z + (int64_t)leaf * lb.m_pad * q;
  const int64_t total = (int64_t)lb.m_pad * q;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / q), c = (int)(e % q);
    z[e] = (r < m) ? B[(int64_t)(begin + r) * ldb + c] : 0.0;
  }
}

__global__ void k_leaf_scatter(LeafBatch lb, const double* Z, double* X, int64_t ldx, int q) {
  const int leaf = blockIdx.y;
  const int begin = lb.begin[leaf], m = lb.size[leaf];
  const double* z = Z + (int64_t)leaf * lb.m_pad * q;
  const int64_t total = (int64_t)m * q;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x)
    X[(int64_t)(begin + e / q) * ldx + e % q] = z[e];
}

void launch_leaf_gather(const LeafBatch& lb, const double* B, int64_t ldb, double* Z, int q, cudaStream_t st) {
  dim3 g(16, lb.count);
  k_leaf_gather<<<g, 256, 0, st>>>(lb, B, ldb, Z, q);
}

void launch_leaf_scatter(const LeafBatch& lb, const double* Z, double* X, int64_t ldx, int q, cudaStream_t st) {
  dim3 g(16, lb.count);
  k_leaf_scatter<<<g, 256, 0, st>>>(lb, Z, X, ldx, q);
}

// Y[k] = Pi W[k] for the second half of each node's 2 s_pad-row block (the S
// rows of the block formulation): rows through S's composed pivot permutation
__global__ void k_permute_rows(NodeBatch nb, const double* W, double* Y, int q) {
  const int k = blockIdx.y;
  const int S = nb.t_pad;
  const int* pm = nb.pm + (int64_t)k * S;
  const double* w = W + (int64_t)(nb.first + k) * nb.zt * q + (int64_t)S * q;
  double* y = Y + (int64_t)(nb.first + k) * nb.zt * q + (int64_t)S * q;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < S * q; e += gridDim.x * blockDim.x)
    y[e] = w[(int64_t)pm[e / q] * q + e % q];
}

void launch_permute_rows(const NodeBatch& nb, const double* W, double* Y, int q, cudaStream_t st) {
  dim3 g(8, nb.count);
  k_permute_rows<<<g, 256, 0, st>>>(nb, W, Y, q);
}

// children's incoming blocks from the node's solved u = [u_l; u_r]
__global__ void k_split_u(NodeBatch nb, const double* U, double* tin, int q) {
  const int k = blockIdx.y;
  const int S = nb.s_pad;
  const double* u = U + (int64_t)(nb.first + k) * nb.zt * q;
  double* tl = tin + (int64_t)nb.left[k] * S * q;
  double* tr = tin + (int64_t)nb.right[k] * S * q;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < S * q; e += gridDim.x * blockDim.x) {
    tl[e] = u[e];
    tr[e] = u[(int64_t)S * q + e];
  }
}

void launch_split_u(const NodeBatch& nb, const double* U, double* tin, int q, cudaStream_t st) {
  dim3 g(8, nb.count);
  k_split_u<<<g, 256, 0, st>>>(nb, U, tin, q);
}

}  // namespace ks
