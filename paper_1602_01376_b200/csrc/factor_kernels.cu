// Factorization kernels of the Inv-ASKIT hot path (reference: solver.py:92-189).
//
// Leaves (solver.py:123-136): the (m+s) x m trapezoid [[K_leaf + lam I], [P]]
// is assembled in HBM and Cholesky-factored left-looking in 64-column panels
// (panel update = DMMA GEMM, diagonal block = k_potrf64 below, panel TRSM =
// DMMA GEMM with the diagonal block's inverse). The bottom s rows come out as
// L21 = P L^-T, so H = P A^-1 P^T = L21 L21^T is one DMMA SYRK.
//
// Internal nodes (solver.py:138-165): the augmented matrix
//     [[Z, P^T], [-P G, 0]],  Z = I + W G,  W = [[0, B], [B^T, 0]]
// is assembled (coupling B by k_coupling, products by DMMA GEMMs) and LU
// factored with partial pivoting restricted to the first t rows; the trailing
// block is then H = P G Z^-1 P^T (the reference's P M P^T, M = G Z^-1).
#include <cfloat>

#include "kernels.cuh"

namespace ks {

// --------------------------------------------------------------------------
// Gaussian blocks. Difference form exactly as kernels.py:107-111:
//   sq = sum_d (x_d - y_d)^2 ;  k = exp(sq / (-2 h h))
// --------------------------------------------------------------------------
constexpr int GT = 64;   // output tile
constexpr int GD = 32;   // dimension chunk staged in shared memory

template <bool GATHER>
__device__ __forceinline__ void gauss_tile(const DevTree& t, const int* rows_pos, int row_base, int nrows,
                                           const int* cols_pos, int col_base, int ncols, int r0, int c0,
                                           double (&sq)[4][4]) {
  __shared__ double xs[GT][GD + 1];
  __shared__ double ys[GT][GD + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) sq[i][j] = 0.0;
  const int64_t d = t.d;
  for (int d0 = 0; d0 < d; d0 += GD) {
    const int dc = (int)((d - d0) < GD ? (d - d0) : GD);
    for (int e = threadIdx.x; e < GT * GD; e += 256) {
      const int r = e / GD, k = e % GD;
      double xv = 0.0, yv = 0.0;
      if (k < dc) {
        const int rr = r0 + r, cc = c0 + r;
        if (rr < nrows) {
          const int64_t p = GATHER ? rows_pos[rr] : (int64_t)row_base + rr;
          xv = t.coords[p * d + d0 + k];
        }
        if (cc < ncols) {
          const int64_t p = GATHER ? cols_pos[cc] : (int64_t)col_base + cc;
          yv = t.coords[p * d + d0 + k];
        }
      }
      xs[r][k] = xv;
      ys[r][k] = yv;
    }
    __syncthreads();
    for (int k = 0; k < dc; ++k) {
      double xv[4], yv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) xv[i] = xs[ty + 16 * i][k];
#pragma unroll
      for (int j = 0; j < 4; ++j) yv[j] = ys[tx + 16 * j][k];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double df = xv[i] - yv[j];
          sq[i][j] = fma(df, df, sq[i][j]);
        }
    }
    __syncthreads();
  }
}

// Leaf block K(X_leaf, X_leaf) + lam I into the lower triangle of the leaf
// workspace (compress.py:271-272 + solver.py:124); padding rows/cols get the
// identity so the padded Cholesky is blkdiag(L, I) exactly.
__global__ void __launch_bounds__(256) k_leaf_gauss(DevTree t, LeafBatch lb, double lam) {
  const int leaf = blockIdx.y;
  // lower-triangular tile enumeration: tile (ti, tj), tj <= ti
  int ti = (int)((sqrt(8.0 * blockIdx.x + 1.0) - 1.0) * 0.5);
  while ((ti + 1) * (ti + 2) / 2 <= (int)blockIdx.x) ++ti;
  while (ti * (ti + 1) / 2 > (int)blockIdx.x) --ti;
  const int tj = blockIdx.x - ti * (ti + 1) / 2;
  const int r0 = ti * GT, c0 = tj * GT;
  const int begin = lb.begin[leaf], m = lb.size[leaf];
  double sq[4][4];
  gauss_tile<false>(t, nullptr, begin, m, nullptr, begin, m, r0, c0, sq);
  const double den = -2.0 * t.h * t.h;
  double* A = lb.A + (int64_t)leaf * lb.a_stride;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = r0 + ty + 16 * i;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = c0 + tx + 16 * j;
      double v;
      if (c > r)
        v = 0.0;  // upper triangle of diagonal tiles: defined zeros
      else if (r >= m || c >= m)
        v = (r == c) ? 1.0 : 0.0;
      else
        v = exp(sq[i][j] / den) + (r == c ? lam : 0.0);
      A[(int64_t)r * lb.m_pad + c] = v;
    }
  }
}

// P rows of the leaf trapezoid (rows m_pad .. m_pad+s_pad-1), zero padded.
__global__ void k_leaf_copy_p(DevTree t, LeafBatch lb) {
  const int leaf = blockIdx.y;
  const int node = lb.node[leaf], m = lb.size[leaf], r = t.rank[node];
  const double* P = t.coeff + t.coeff_off[node];
  double* A = lb.A + (int64_t)leaf * lb.a_stride + (int64_t)lb.m_pad * lb.m_pad;
  const int64_t total = (int64_t)lb.s_pad * lb.m_pad;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / lb.m_pad), j = (int)(e % lb.m_pad);
    A[e] = (i < r && j < m) ? P[(int64_t)i * m + j] : 0.0;
  }
}

void launch_leaf_assemble(const DevTree& t, const LeafBatch& lb, double lam, cudaStream_t st) {
  const int nt = lb.m_pad / GT;
  dim3 g1(nt * (nt + 1) / 2, lb.count);
  k_leaf_gauss<<<g1, 256, 0, st>>>(t, lb, lam);
  if (lb.s_pad > 0) {
    dim3 g2(64, lb.count);
    k_leaf_copy_p<<<g2, 256, 0, st>>>(t, lb);
  }
}

// --------------------------------------------------------------------------
// 64x64 diagonal-block Cholesky + triangular inverse (one CTA per leaf).
// Failure (pivot <= 0 or non-finite) records the first bad column + 1, as
// _cholesky raises NotSPDError at linalg.py:190-192.
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_potrf64(LeafBatch lb, int j0, double* inv, int* info) {
  const int leaf = blockIdx.x;
  double* A = lb.A + (int64_t)leaf * lb.a_stride + (int64_t)j0 * lb.m_pad + j0;
  const int64_t ld = lb.m_pad;
  extern __shared__ double potrf_sm[];
  double(*a)[65] = reinterpret_cast<double(*)[65]>(potrf_sm);
  double(*x)[65] = reinterpret_cast<double(*)[65]>(potrf_sm + 64 * 65);
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  for (int e = threadIdx.x; e < 64 * 64; e += 256) {
    const int r = e >> 6, c = e & 63;
    a[r][c] = (c <= r) ? A[r * ld + c] : 0.0;
  }
  __syncthreads();
  for (int k = 0; k < 64; ++k) {
    if (threadIdx.x == 0) {
      const double p = a[k][k];
      if (!(p > 0.0) || !isfinite(p)) {
        if (!bad) bad = j0 + k + 1;
        a[k][k] = 1.0;
      } else {
        a[k][k] = sqrt(p);
      }
    }
    __syncthreads();
    const double dk = a[k][k];
    for (int i = k + 1 + threadIdx.x; i < 64; i += 256) a[i][k] /= dk;
    __syncthreads();
    // trailing update of the lower triangle: a[i][j] -= a[i][k] a[j][k], k < j <= i
    const int rem = 63 - k;
    for (int e = threadIdx.x; e < rem * rem; e += 256) {
      const int i = k + 1 + e / rem, j = k + 1 + e % rem;
      if (j <= i) a[i][j] = fma(-a[i][k], a[j][k], a[i][j]);
    }
    __syncthreads();
  }
  // inverse of the lower factor, one column per thread (columns independent)
  if (threadIdx.x < 64) {
    const int j = threadIdx.x;
    for (int i = 0; i < 64; ++i) x[i][j] = 0.0;
    x[j][j] = 1.0 / a[j][j];
    for (int i = j + 1; i < 64; ++i) {
      double s = 0.0;
      for (int k = j; k < i; ++k) s = fma(a[i][k], x[k][j], s);
      x[i][j] = -s / a[i][i];
    }
  }
  __syncthreads();
  double* iv = inv + (int64_t)leaf * 64 * 64;
  for (int e = threadIdx.x; e < 64 * 64; e += 256) {
    const int r = e >> 6, c = e & 63;
    A[r * ld + c] = (c <= r) ? a[r][c] : 0.0;
    iv[e] = x[r][c];
  }
  if (threadIdx.x == 0 && bad && info[leaf] == 0) info[leaf] = bad;
}

void launch_potrf64(const LeafBatch& lb, int j0, double* inv, int* info, cudaStream_t st) {
  constexpr size_t smem = 2 * 64 * 65 * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_potrf64, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  k_potrf64<<<lb.count, 256, smem, st>>>(lb, j0, inv, info);
}

// In-place symmetrization H = (H + H^T)/2 (solver.py:135, :163).
__global__ void k_sym_h(double* H, int64_t stride, const int* idx, int s) {
  double* h = H + (int64_t)idx[blockIdx.y] * stride;
  const int64_t total = (int64_t)s * s;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / s), j = (int)(e % s);
    if (j < i) {
      const double v = 0.5 * (h[(int64_t)i * s + j] + h[(int64_t)j * s + i]);
      h[(int64_t)i * s + j] = v;
      h[(int64_t)j * s + i] = v;
    }
  }
}

void launch_sym_h(double* H, int64_t h_stride, const int* node_idx, int count, int s_pad, cudaStream_t st) {
  if (count <= 0 || s_pad <= 0) return;
  dim3 g(32, count);
  k_sym_h<<<g, 256, 0, st>>>(H, h_stride, node_idx, s_pad);
}

// --------------------------------------------------------------------------
// Internal node assembly
// --------------------------------------------------------------------------
// Coupling B = K(S_l, S_r) (compress.py:281-283), zero padded to s_pad^2.
__global__ void __launch_bounds__(256) k_coupling(DevTree t, NodeBatch nb) {
  const int k = blockIdx.z;
  const int l = nb.left[k], r = nb.right[k];
  const int sl = t.rank[l], sr = t.rank[r];
  const int r0 = blockIdx.y * GT, c0 = blockIdx.x * GT;
  double sq[4][4];
  gauss_tile<true>(t, t.skel_pos + t.skel_off[l], 0, sl, t.skel_pos + t.skel_off[r], 0, sr, r0, c0, sq);
  const double den = -2.0 * t.h * t.h;
  double* B = nb.Bc + (int64_t)k * nb.s_pad * nb.s_pad;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int rr = r0 + ty + 16 * i;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int cc = c0 + tx + 16 * j;
      B[(int64_t)rr * nb.s_pad + cc] = (rr < sl && cc < sr) ? exp(sq[i][j] / den) : 0.0;
    }
  }
}

void launch_coupling(const DevTree& t, const NodeBatch& nb, cudaStream_t st) {
  dim3 g(nb.s_pad / GT, nb.s_pad / GT, nb.count);
  k_coupling<<<g, 256, 0, st>>>(t, nb);
}

// Identity diagonal blocks of Z, P^T (top right), zero bottom-right block, and
// the padded P copy used by the solve. Z12/Z21 and -PG are written by GEMMs.
// Padded candidate index i' maps to the reference's cand index
// (cand = [skel_l; skel_r], compress.py:213): i' < s_pad -> i' (if < s_l),
// i' >= s_pad -> s_l + (i' - s_pad) (if < s_r).
__global__ void k_aug_init(DevTree t, NodeBatch nb) {
  const int k = blockIdx.y;
  const int v = nb.node[k], l = nb.left[k], r = nb.right[k];
  const int sl = t.rank[l], sr = t.rank[r], sv = t.rank[v];
  const int S = nb.s_pad, TP = nb.t_pad, T = nb.T;
  const double* P = t.coeff + t.coeff_off[v];
  const int cand = sl + sr;
  double* A = nb.Aug + (int64_t)k * T * T;
  double* Pn = nb.Pn + (int64_t)k * S * TP;
  // (a) identity blocks of Z: rows/cols in the same half
  const int64_t n_id = 2LL * S * S;
  // (b) P^T block: TP x S at (0, TP);  (c) zero block S x S at (TP, TP);  (d) Pn: S x TP
  const int64_t n_pt = (int64_t)TP * S, n_z = (int64_t)S * S, n_pn = (int64_t)S * TP;
  const int64_t total = n_id + n_pt + n_z + n_pn;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    if (e < n_id) {
      const int half = (int)(e / ((int64_t)S * S));
      const int64_t f = e % ((int64_t)S * S);
      const int i = (int)(f / S), j = (int)(f % S);
      A[(int64_t)(half * S + i) * T + half * S + j] = (i == j) ? 1.0 : 0.0;
      continue;
    }
    int64_t f = e - n_id;
    if (f < n_pt) {
      const int i = (int)(f / S), j = (int)(f % S);  // P^T[i][j] = P[j][i']
      const int ci = (i < S) ? (i < sl ? i : -1) : (i - S < sr ? sl + (i - S) : -1);
      A[(int64_t)i * T + TP + j] = (ci >= 0 && j < sv) ? P[(int64_t)j * cand + ci] : 0.0;
      continue;
    }
    f -= n_pt;
    if (f < n_z) {
      const int i = (int)(f / S), j = (int)(f % S);
      A[(int64_t)(TP + i) * T + TP + j] = 0.0;
      continue;
    }
    f -= n_z;
    {
      const int j = (int)(f / TP), i = (int)(f % TP);
      const int ci = (i < S) ? (i < sl ? i : -1) : (i - S < sr ? sl + (i - S) : -1);
      Pn[f] = (ci >= 0 && j < sv) ? P[(int64_t)j * cand + ci] : 0.0;
    }
  }
}

void launch_aug_init(const DevTree& t, const NodeBatch& nb, cudaStream_t st) {
  dim3 g(128, nb.count);
  k_aug_init<<<g, 256, 0, st>>>(t, nb);
}

// 1-norm of Z (max column abs sum, linalg.py:176), before the LU overwrites it.
__global__ void k_colnorm1(NodeBatch nb) {
  const int k = blockIdx.x;
  const double* A = nb.Aug + (int64_t)k * nb.T * nb.T;
  double best = 0.0;
  for (int j = threadIdx.x; j < nb.t_pad; j += blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < nb.t_pad; ++i) s += fabs(A[(int64_t)i * nb.T + j]);
    best = fmax(best, s);
  }
  __shared__ double red[256];
  red[threadIdx.x] = best;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) nb.norm1[k] = red[0];
}

void launch_colnorm1(const DevTree&, const NodeBatch& nb, cudaStream_t st) {
  k_colnorm1<<<nb.count, 256, 0, st>>>(nb);
}

// --------------------------------------------------------------------------
// LU with partial pivoting restricted to rows < t_pad (linalg.py:199-213 on
// the Z block; the -PG rows are eliminated but never chosen as pivots).
// Base panel: W columns [c0, c0+W), rows [c0, T), staged column-major in smem.
// --------------------------------------------------------------------------
template <int W>
__global__ void __launch_bounds__(512) k_lu_panel(NodeBatch nb, int c0) {
  extern __shared__ double sp[];  // W x ldp
  const int k = blockIdx.x;
  const int T = nb.T;
  double* A = nb.Aug + (int64_t)k * T * T;
  const int rows = T - c0;
  const int ldp = rows + 1;
  const int plim = nb.t_pad - c0;  // pivot rows are local rows [kk, plim)
  __shared__ double rv[16];
  __shared__ int ri[16];
  __shared__ int s_piv;
  for (int e = threadIdx.x; e < rows * W; e += blockDim.x) {
    const int r = e / W, j = e % W;
    sp[j * ldp + r] = A[(int64_t)(c0 + r) * T + c0 + j];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int kk = 0; kk < W; ++kk) {
    double* col = sp + kk * ldp;
    // argmax |col[r]|, r in [kk, plim), first index on ties (np.argmax)
    double bv = -1.0;
    int bi = 0x7fffffff;
    for (int r = kk + threadIdx.x; r < plim; r += blockDim.x) {
      const double a = fabs(col[r]);
      if (a > bv) { bv = a; bi = r; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) { rv[warp] = bv; ri[warp] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = rv[0];
      int i = ri[0];
      for (int w = 1; w < nw; ++w)
        if (rv[w] > b || (rv[w] == b && ri[w] < i)) { b = rv[w]; i = ri[w]; }
      if (!(b > 0.0)) {  // exactly zero pivot column (SingularMatrixError)
        if (nb.info[k] == 0) nb.info[k] = c0 + kk + 1;
        i = kk;
      }
      s_piv = i;
      nb.piv[(int64_t)k * nb.t_pad + c0 + kk] = c0 + i;
    }
    __syncthreads();
    const int p = s_piv;
    if (p != kk && threadIdx.x < W) {
      double* cj = sp + threadIdx.x * ldp;
      const double tmp = cj[kk];
      cj[kk] = cj[p];
      cj[p] = tmp;
    }
    __syncthreads();
    const double pv = col[kk];
    const double piv_ok = (pv != 0.0) ? pv : 1.0;
    for (int r = kk + 1 + threadIdx.x; r < rows; r += blockDim.x) {
      const double l = col[r] / piv_ok;
      col[r] = l;
#pragma unroll 4
      for (int j = kk + 1; j < W; ++j) sp[j * ldp + r] = fma(-l, sp[j * ldp + kk], sp[j * ldp + r]);
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < rows * W; e += blockDim.x) {
    const int r = e / W, j = e % W;
    A[(int64_t)(c0 + r) * T + c0 + j] = sp[j * ldp + r];
  }
}

void launch_lu_panel(const NodeBatch& nb, int c0, int w, cudaStream_t st) {
  const int rows = nb.T - c0;
  const size_t smem = (size_t)w * (rows + 1) * sizeof(double);
  if (w == 32) {
    cudaFuncSetAttribute(k_lu_panel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_lu_panel<32><<<nb.count, 512, smem, st>>>(nb, c0);
  } else {
    cudaFuncSetAttribute(k_lu_panel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_lu_panel<16><<<nb.count, 512, smem, st>>>(nb, c0);
  }
}

// Apply the panel's row interchanges to every column outside the panel
// (LAPACK getrf convention: L keeps later swaps; linalg.py:209).
__global__ void k_lu_swap(NodeBatch nb, int c0, int w) {
  const int k = blockIdx.y;
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  const int T = nb.T;
  if (col >= T || (col >= c0 && col < c0 + w)) return;
  double* A = nb.Aug + (int64_t)k * T * T;
  const int* piv = nb.piv + (int64_t)k * nb.t_pad;
  for (int kk = 0; kk < w; ++kk) {
    const int r1 = c0 + kk, r2 = piv[r1];
    if (r1 != r2) {
      const double a = A[(int64_t)r1 * T + col];
      A[(int64_t)r1 * T + col] = A[(int64_t)r2 * T + col];
      A[(int64_t)r2 * T + col] = a;
    }
  }
}

void launch_lu_swap(const NodeBatch& nb, int c0, int w, cudaStream_t st) {
  dim3 g((nb.T + 127) / 128, nb.count);
  k_lu_swap<<<g, 128, 0, st>>>(nb, c0, w);
}

// B := L^-1 B for the unit-lower W x W block at (r0, r0), B = rows r0..r0+W,
// columns [c0, c0+ncols). One thread per column, x held in registers.
template <int W>
__global__ void __launch_bounds__(128) k_trsm_ul(NodeBatch nb, int r0, int c0, int ncols) {
  const int k = blockIdx.y;
  const int T = nb.T;
  double* A = nb.Aug + (int64_t)k * T * T;
  __shared__ double L[W][W + 1];
  for (int e = threadIdx.x; e < W * W; e += blockDim.x) {
    const int i = e / W, j = e % W;
    L[i][j] = A[(int64_t)(r0 + i) * T + r0 + j];
  }
  __syncthreads();
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= ncols) return;
  double* B = A + (int64_t)r0 * T + c0 + col;
  double x[W];
#pragma unroll
  for (int i = 0; i < W; ++i) x[i] = B[(int64_t)i * T];
#pragma unroll
  for (int i = 1; i < W; ++i) {
    double s = x[i];
#pragma unroll
    for (int j = 0; j < i; ++j) s = fma(-L[i][j], x[j], s);
    x[i] = s;
  }
#pragma unroll
  for (int i = 0; i < W; ++i) B[(int64_t)i * T] = x[i];
}

void launch_trsm_unit_lower(const NodeBatch& nb, int r0, int w, int c0, int ncols, cudaStream_t st) {
  if (ncols <= 0) return;
  dim3 g((ncols + 127) / 128, nb.count);
  if (w == 16) k_trsm_ul<16><<<g, 128, 0, st>>>(nb, r0, c0, ncols);
  else if (w == 32) k_trsm_ul<32><<<g, 128, 0, st>>>(nb, r0, c0, ncols);
  else k_trsm_ul<64><<<g, 128, 0, st>>>(nb, r0, c0, ncols);
}

// --------------------------------------------------------------------------
// Hager 1-norm condition estimate of Z (linalg.py:282-304), one warp per node,
// on the LU factors in place. Only real (unpadded) indices take part.
// --------------------------------------------------------------------------
struct ZView {
  const double* A;
  int T, n;
  const int* piv;
  __device__ double at(int i, int j) const { return A[(int64_t)i * T + j]; }
};

__device__ void warp_lu_solve(const ZView& z, double* v) {  // Z v = b (in place)
  const int lane = threadIdx.x & 31;
  for (int k = 0; k < z.n; ++k) {  // row swaps
    const int p = z.piv[k];
    if (p != k && lane == 0) { const double t = v[k]; v[k] = v[p]; v[p] = t; }
    __syncwarp();
  }
  for (int i = 0; i < z.n; ++i) {  // unit lower, rows
    double s = 0.0;
    for (int c = lane; c < i; c += 32) s = fma(z.at(i, c), v[c], s);
    s = warp_sum(s);
    if (lane == 0) v[i] -= s;
    __syncwarp();
  }
  for (int i = z.n - 1; i >= 0; --i) {  // upper, rows
    double s = 0.0;
    for (int c = i + 1 + lane; c < z.n; c += 32) s = fma(z.at(i, c), v[c], s);
    s = warp_sum(s);
    if (lane == 0) v[i] = (v[i] - s) / z.at(i, i);
    __syncwarp();
  }
}

__device__ void warp_lu_solve_t(const ZView& z, double* v) {  // Z^T v = b (in place)
  const int lane = threadIdx.x & 31;
  for (int k = 0; k < z.n; ++k) {  // U^T w = b: forward, right-looking on rows of U
    if (lane == 0) v[k] /= z.at(k, k);
    __syncwarp();
    const double vk = v[k];
    for (int i = k + 1 + lane; i < z.n; i += 32) v[i] = fma(-z.at(k, i), vk, v[i]);
    __syncwarp();
  }
  for (int k = z.n - 1; k >= 0; --k) {  // L^T x = w: backward, unit, rows of L
    const double vk = v[k];
    for (int i = lane; i < k; i += 32) v[i] = fma(-z.at(k, i), vk, v[i]);
    __syncwarp();
  }
  for (int k = z.n - 1; k >= 0; --k) {  // undo swaps in reverse
    const int p = z.piv[k];
    if (p != k && lane == 0) { const double t = v[k]; v[k] = v[p]; v[p] = t; }
    __syncwarp();
  }
}

__global__ void __launch_bounds__(32) k_hager(DevTree t, NodeBatch nb) {
  extern __shared__ double hv[];  // 3 x t_pad
  const int k = blockIdx.x;
  const int lane = threadIdx.x;
  const int TP = nb.t_pad, S = nb.s_pad;
  const int sl = t.rank[nb.left[k]], sr = t.rank[nb.right[k]];
  const int n = sl + sr;
  ZView z{nb.Aug + (int64_t)k * nb.T * nb.T, nb.T, TP, nb.piv + (int64_t)k * TP};
  double* x = hv;
  double* y = hv + TP;
  double* w = hv + 2 * TP;
  auto real = [&](int i) { return i < S ? (i < sl) : (i - S < sr); };
  if (n == 0) { if (lane == 0) nb.cond[k] = 0.0; return; }
  for (int i = lane; i < TP; i += 32) x[i] = real(i) ? 1.0 / n : 0.0;
  __syncwarp();
  double est = 0.0;
  for (int it = 0; it < 5; ++it) {
    for (int i = lane; i < TP; i += 32) y[i] = x[i];
    __syncwarp();
    warp_lu_solve(z, y);
    double s = 0.0;
    for (int i = lane; i < TP; i += 32) s += real(i) ? fabs(y[i]) : 0.0;
    est = warp_sum(s);
    for (int i = lane; i < TP; i += 32) w[i] = real(i) ? (y[i] >= 0.0 ? 1.0 : -1.0) : 0.0;
    __syncwarp();
    warp_lu_solve_t(z, w);
    // j = argmax |z| (first on ties, in reference index order), z.x
    double bv = -1.0, dot = 0.0;
    int bi = 0x7fffffff;
    for (int i = lane; i < TP; i += 32) {
      if (!real(i)) continue;
      const double a = fabs(w[i]);
      const int ri = i < S ? i : sl + (i - S);
      if (a > bv || (a == bv && ri < bi)) { bv = a; bi = ri; }
      dot = fma(w[i], x[i], dot);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    dot = warp_sum(dot);
    if (bv <= dot) break;
    const int jp = bi < sl ? bi : S + (bi - sl);  // back to padded index
    for (int i = lane; i < TP; i += 32) x[i] = (i == jp) ? 1.0 : 0.0;
    __syncwarp();
  }
  if (lane == 0) nb.cond[k] = isfinite(est) ? nb.norm1[k] * est : INFINITY;
}

void launch_hager(const DevTree& t, const NodeBatch& nb, cudaStream_t st) {
  k_hager<<<nb.count, 32, 3 * nb.t_pad * sizeof(double), st>>>(t, nb);
}

// H = sym(trailing block) -> Hbuf[node] (solver.py:163).
__global__ void k_extract_h(NodeBatch nb, double* H, int64_t stride) {
  const int k = blockIdx.y;
  const int S = nb.s_pad, T = nb.T, TP = nb.t_pad;
  const double* A = nb.Aug + (int64_t)k * T * T + (int64_t)TP * T + TP;
  double* h = H + (int64_t)nb.node[k] * stride;
  const int64_t total = (int64_t)S * S;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / S), j = (int)(e % S);
    h[e] = 0.5 * (A[(int64_t)i * T + j] + A[(int64_t)j * T + i]);
  }
}

void launch_extract_h(const NodeBatch& nb, double* H, int64_t h_stride, cudaStream_t st) {
  dim3 g(32, nb.count);
  k_extract_h<<<g, 256, 0, st>>>(nb, H, h_stride);
}

}  // namespace ks
