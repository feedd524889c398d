// Compressed-operator matvec Y = K~ W on the device (reference: hss_matvec,
// compress.py:352-411): upward skeleton weights c = P w (leaves) / P [c_l; c_r]
// (nodes), sibling exchange through the coupling blocks B = K(S_l, S_r), downward
// totals t_child = incoming + (P^T t)[child part], and at the leaves
// Y = K(X_leaf, X_leaf) W + P^T t. P comes from the uploaded coefficients
// (unpadded, rank x |cand|), coupling blocks from the factorization, leaf kernel
// blocks are recomputed on the fly in the reference's difference form. Used for
// residual checks ||(K~ + lam I) u - b|| at full size.
#include "gauss.cuh"
#include "kernels.cuh"
#include "trsv.cuh"

namespace ks {

// rows of P (r x ncand, row-major) times x (ncand x QC, shared) -> out rows (ld q)
template <int QC>
__device__ void p_apply(const double* __restrict__ P, int r, int ncand, const double* x, double* out, int q) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = warp; i < r; i += SWARPS) {
    double acc[QC];
#pragma unroll
    for (int qq = 0; qq < QC; ++qq) acc[qq] = 0.0;
    for (int j = lane; j < ncand; j += 32) {
      const double p = __ldg(P + (int64_t)i * ncand + j);
#pragma unroll
      for (int qq = 0; qq < QC; ++qq) acc[qq] = fma(p, x[j * QC + qq], acc[qq]);
    }
#pragma unroll
    for (int qq = 0; qq < QC; ++qq) {
      const double s = warp_sum(acc[qq]);
      if (lane == 0) out[(int64_t)i * q + qq] = s;
    }
  }
}

template <int QC>
__global__ void __launch_bounds__(STHREADS) k_mv_up_leaf(DevTree t, LeafBatch lb, const double* W, int64_t ldw,
                                                        double* c, int S, int q, int q0) {
  extern __shared__ double x[];
  const int v = lb.node[blockIdx.x], begin = lb.begin[blockIdx.x], m = lb.size[blockIdx.x];
  const int r = t.rank[v];
  if (r == 0) return;
  for (int e = threadIdx.x; e < m * QC; e += STHREADS) x[e] = W[(int64_t)(begin + e / QC) * ldw + q0 + e % QC];
  __syncthreads();
  p_apply<QC>(t.coeff + t.coeff_off[v], r, m, x, c + (int64_t)v * S * q + q0, q);
}

template <int QC>
__global__ void __launch_bounds__(STHREADS) k_mv_up_node(DevTree t, NodeBatch nb, double* c, int S, int q, int q0) {
  extern __shared__ double x[];
  const int v = nb.node[blockIdx.x], l = nb.left[blockIdx.x], rr = nb.right[blockIdx.x];
  const int r = t.rank[v];
  if (r == 0) return;
  const int sl = t.rank[l], ncand = sl + t.rank[rr];
  for (int e = threadIdx.x; e < ncand * QC; e += STHREADS) {
    const int i = e / QC, qq = e % QC;
    x[e] = (i < sl) ? c[((int64_t)l * S + i) * q + q0 + qq] : c[((int64_t)rr * S + (i - sl)) * q + q0 + qq];
  }
  __syncthreads();
  p_apply<QC>(t.coeff + t.coeff_off[v], r, ncand, x, c + (int64_t)v * S * q + q0, q);
}

// incoming[l] = B c_r, incoming[r] = B^T c_l   (compress.py:383-387)
template <int QC>
__global__ void __launch_bounds__(STHREADS) k_mv_couple(DevTree t, NodeBatch nb, const double* c, double* inc, int S,
                                                       int q, int q0) {
  extern __shared__ double sm[];
  double* cl = sm;            // S x QC
  double* cr = sm + S * QC;   // S x QC
  double* ot = cr + S * QC;   // S x QC
  double* red = ot + S * QC;  // SWARPS x 32 x QC
  const int k = blockIdx.x;
  const int l = nb.left[k], r = nb.right[k];
  for (int e = threadIdx.x; e < S * QC; e += STHREADS) {
    const int i = e / QC, qq = e % QC;
    cl[e] = c[((int64_t)l * S + i) * q + q0 + qq];
    cr[e] = c[((int64_t)r * S + i) * q + q0 + qq];
    ot[e] = 0.0;
  }
  __syncthreads();
  const double* B = nb.Bc + (int64_t)k * S * S;
  cta_gemv_rows<QC>(B, S, S, S, cr, inc + (int64_t)l * S * q + q0, q, false);
  cta_gemv_cols<QC>(B, S, S, S, cl, ot, 1.0, red);
  double* ir = inc + (int64_t)r * S * q + q0;
  for (int e = threadIdx.x; e < S * QC; e += STHREADS) ir[(int64_t)(e / QC) * q + e % QC] = ot[e];
}

// tot[child] = inc[child] (+ (P_v^T tot[v])[child part])  (compress.py:389-404)
template <int QC>
__global__ void __launch_bounds__(STHREADS) k_mv_down(DevTree t, NodeBatch nb, const double* inc, double* tot, int S,
                                                     int q, int q0, int has_tot) {
  extern __shared__ double tv[];
  const int k = blockIdx.x;
  const int v = nb.node[k], l = nb.left[k], r = nb.right[k];
  const int sl = t.rank[l], sv = t.rank[v];
  const int ncand = sl + t.rank[r];
  if (has_tot)
    for (int e = threadIdx.x; e < sv * QC; e += STHREADS) tv[e] = tot[((int64_t)v * S + e / QC) * q + q0 + e % QC];
  __syncthreads();
  const double* P = t.coeff + t.coeff_off[v];
  for (int j = threadIdx.x; j < ncand; j += STHREADS) {
    double acc[QC];
#pragma unroll
    for (int qq = 0; qq < QC; ++qq) acc[qq] = 0.0;
    if (has_tot)
      for (int i = 0; i < sv; ++i) {
        const double p = __ldg(P + (int64_t)i * ncand + j);
#pragma unroll
        for (int qq = 0; qq < QC; ++qq) acc[qq] = fma(p, tv[i * QC + qq], acc[qq]);
      }
    const int child = j < sl ? l : r;
    const int i = j < sl ? j : j - sl;
#pragma unroll
    for (int qq = 0; qq < QC; ++qq) {
      const int64_t o = ((int64_t)child * S + i) * q + q0 + qq;
      tot[o] = inc[o] + acc[qq];
    }
  }
}

// Y_leaf = K(X_leaf, X_leaf) W_leaf + P^T tot[leaf]   (compress.py:406-410);
// grid (row tiles of 64, leaves)
template <int QC>
__global__ void __launch_bounds__(256) k_mv_leaf(DevTree t, LeafBatch lb, const double* W, int64_t ldw,
                                                const double* tot, double* Y, int S, int q, int q0, int has_tot) {
  const int leaf = blockIdx.y;
  const int v = lb.node[leaf], begin = lb.begin[leaf], m = lb.size[leaf];
  const int r0 = blockIdx.x * GT;
  if (r0 >= m) return;
  const double den = -2.0 * t.h * t.h;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][QC];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int qq = 0; qq < QC; ++qq) acc[i][qq] = 0.0;
  for (int c0 = 0; c0 < m; c0 += GT) {
    double sq[4][4];
    gauss_tile<false>(t, nullptr, begin, m, nullptr, begin, m, r0, c0, sq);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int cc = c0 + tx + 16 * j;
      if (cc >= m) continue;
      double wv[QC];
#pragma unroll
      for (int qq = 0; qq < QC; ++qq) wv[qq] = W[(int64_t)(begin + cc) * ldw + q0 + qq];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double kv = exp(sq[i][j] / den);
#pragma unroll
        for (int qq = 0; qq < QC; ++qq) acc[i][qq] = fma(kv, wv[qq], acc[i][qq]);
      }
    }
  }
  // reduce over the 16 column threads (tx) of each row
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int qq = 0; qq < QC; ++qq)
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) acc[i][qq] += __shfl_xor_sync(0xffffffffu, acc[i][qq], o);
  if (tx == 0) {
    const int sv = t.rank[v];
    const double* P = t.coeff + t.coeff_off[v];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int rr = r0 + ty + 16 * i;
      if (rr >= m) continue;
      double a[QC];
#pragma unroll
      for (int qq = 0; qq < QC; ++qq) a[qq] = acc[i][qq];
      if (has_tot)
        for (int k2 = 0; k2 < sv; ++k2) {
          const double p = P[(int64_t)k2 * m + rr];
#pragma unroll
          for (int qq = 0; qq < QC; ++qq) a[qq] = fma(p, tot[((int64_t)v * S + k2) * q + q0 + qq], a[qq]);
        }
#pragma unroll
      for (int qq = 0; qq < QC; ++qq) Y[(int64_t)(begin + rr) * q + q0 + qq] = a[qq];
    }
  }
}

template <typename F>
static void chunks(int q, F f) {
  int q0 = 0;
  while (q0 < q) {
    const int qc = (q - q0) >= 4 ? 4 : ((q - q0) >= 2 ? 2 : 1);
    f(q0, qc);
    q0 += qc;
  }
}

template <typename K>
static void smem_attr(K kern, size_t bytes) {
  if (bytes > 48 * 1024) ensure_smem(kern, bytes);
}

#define KS_QC(KERN, GRID, BLOCK, SMEM, ...)                                   \
  chunks(q, [&](int q0, int qc) {                                             \
    if (qc == 4) {                                                            \
      smem_attr(KERN<4>, (SMEM) * 4);                                         \
      KERN<4><<<GRID, BLOCK, (SMEM) * 4, st>>>(__VA_ARGS__);                  \
    } else if (qc == 2) {                                                     \
      smem_attr(KERN<2>, (SMEM) * 2);                                         \
      KERN<2><<<GRID, BLOCK, (SMEM) * 2, st>>>(__VA_ARGS__);                  \
    } else {                                                                  \
      smem_attr(KERN<1>, (SMEM));                                             \
      KERN<1><<<GRID, BLOCK, (SMEM), st>>>(__VA_ARGS__);                      \
    }                                                                         \
  })

void launch_mv_up_leaf(const DevTree& t, const LeafBatch& lb, const double* W, int64_t ldw, double* c, int S, int q,
                       cudaStream_t st) {
  KS_QC(k_mv_up_leaf, lb.count, STHREADS, (size_t)lb.m_pad * sizeof(double), t, lb, W, ldw, c, S, q, q0);
}

void launch_mv_up_node(const DevTree& t, const NodeBatch& nb, double* c, int S, int q, cudaStream_t st) {
  KS_QC(k_mv_up_node, nb.count, STHREADS, (size_t)2 * S * sizeof(double), t, nb, c, S, q, q0);
}

void launch_mv_couple(const DevTree& t, const NodeBatch& nb, const double* c, double* inc, int S, int q,
                      cudaStream_t st) {
  KS_QC(k_mv_couple, nb.count, STHREADS, ((size_t)3 * S + SWARPS * 32) * sizeof(double), t, nb, c, inc, S, q, q0);
}

void launch_mv_down(const DevTree& t, const NodeBatch& nb, const double* inc, double* tot, int S, int q, bool has_tot,
                    cudaStream_t st) {
  KS_QC(k_mv_down, nb.count, STHREADS, (size_t)S * sizeof(double), t, nb, inc, tot, S, q, q0, has_tot ? 1 : 0);
}

void launch_mv_leaf(const DevTree& t, const LeafBatch& lb, const double* W, int64_t ldw, const double* tot, double* Y,
                    int S, int q, bool has_tot, cudaStream_t st) {
  dim3 grid(lb.m_pad / GT, lb.count);
  KS_QC(k_mv_leaf, grid, 256, 0, t, lb, W, ldw, tot, Y, S, q, q0, has_tot ? 1 : 0);
}

// krr_predict partial sums (EPI 3 of the DMMA GEMM) summed over column tiles
__global__ void k_sum_partials(const double* partial, int tiles, int n, double* out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double s = 0.0;
  for (int t = 0; t < tiles; ++t) s += partial[(int64_t)t * n + r];
  out[r] = s;
}

void launch_sum_partials(const double* partial, int tiles, int n, double* out, cudaStream_t st) {
  if (n <= 0) return;
  k_sum_partials<<<(n + 255) / 256, 256, 0, st>>>(partial, tiles, n, out);
}

}  // namespace ks
