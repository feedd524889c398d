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
#include <algorithm>
#include <cfloat>
#include <vector>

#include "gauss.cuh"
#include "kernels.cuh"
#include "lu_panel.cuh"
#include "trsv.cuh"

namespace ks {

// --------------------------------------------------------------------------
// Gaussian blocks. Difference form exactly as kernels.py:107-111:
//   sq = sum_d (x_d - y_d)^2 ;  k = exp(sq / (-2 h h))
// --------------------------------------------------------------------------
// Points to tree order: dst[i] = src[perm[i]] (PartitionTree.perm, tree.py:231-234).
__global__ void k_gather_rows(const double* src, const int64_t* perm, int64_t n, int64_t d, double* dst) {
  const int64_t total = n * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / d, k = e % d;
    dst[e] = src[perm[i] * d + k];
  }
}

void launch_gather_rows(const double* src, const int64_t* perm, int64_t n, int64_t d, double* dst, cudaStream_t st) {
  k_gather_rows<<<1184, 256, 0, st>>>(src, perm, n, d, dst);
}

// Leaf block K(X_leaf, X_leaf) + lam I into the lower triangle of the leaf
// workspace (compress.py:271-272 + solver.py:124); padding rows/cols get the
// identity so the padded Cholesky is blkdiag(L, I) exactly.
__global__ void __launch_bounds__(256) k_leaf_gauss(DevTree t, LeafBatch lb, const double* lam_p) {
  const double lam = *lam_p;
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
  pdl_wait();
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

__global__ void k_row_sqnorms(const double* X, int64_t n, int64_t d, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t k = 0; k < d; ++k) s = fma(X[i * d + k], X[i * d + k], s);
    out[i] = s;
  }
}

void launch_row_sqnorms(const double* X, int64_t n, int64_t d, double* out, cudaStream_t st) {
  k_row_sqnorms<<<1184, 128, 0, st>>>(X, n, d, out);
}

void launch_leaf_copy_p(const DevTree& t, const LeafBatch& lb, cudaStream_t st) {
  if (lb.s_pad > 0) {
    dim3 g2(64, lb.count);
    launch_pdl(k_leaf_copy_p, g2, dim3(256), 0, st, t, lb);
  }
}

void launch_leaf_assemble(const DevTree& t, const LeafBatch& lb, const double* lam, cudaStream_t st) {
  const int nt = lb.m_pad / GT;
  dim3 g1(nt * (nt + 1) / 2, lb.count);
  k_leaf_gauss<<<g1, 256, 0, st>>>(t, lb, lam);
  if (lb.s_pad > 0) {
    dim3 g2(64, lb.count);
    launch_pdl(k_leaf_copy_p, g2, dim3(256), 0, st, t, lb);
  }
}

// --------------------------------------------------------------------------
// 64x64 diagonal-block Cholesky + triangular inverse (one CTA per leaf).
// Failure (pivot <= 0 or non-finite) records the first bad column + 1, as
// _cholesky raises NotSPDError at linalg.py:190-192.
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 6) k_potrf64(LeafBatch lb, int j0, double* inv, int* info) {
  pdl_wait();
  const int leaf = blockIdx.x;
  double* A = lb.A + (int64_t)leaf * lb.a_stride + (int64_t)j0 * lb.m_pad + j0;
  const int64_t ld = lb.m_pad;
  // one 64 x 65 tile: L in the lower triangle, X = L^-1 (also lower) stored
  // transposed in the strict upper triangle (x[i][j] at a[j][i], i > j) with its
  // diagonal in xd: 34 KB, so six CTAs share an SM
  extern __shared__ double potrf_sm[];
  double(*a)[65] = reinterpret_cast<double(*)[65]>(potrf_sm);
  double* xd = potrf_sm + 64 * 65;
  __shared__ int bad;
  {  // all 16 loads per thread in flight
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = threadIdx.x + u * 256, r = e >> 6, c = e & 63;
      v[u] = (c <= r) ? A[r * ld + c] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = threadIdx.x + u * 256, r = e >> 6, c = e & 63;
      a[r][c] = v[u];
    }
    if (threadIdx.x < 64) xd[threadIdx.x] = 1.0;
  }
  if (threadIdx.x == 0) bad = 0x7fffffff;
  __syncthreads();
  // symmetric right-looking elimination, one barrier per column:
  //   a[i][j] -= a[i][k] a[j][k] / p_k  (k < j <= i),  p_k = a[k][k] at step k;
  // afterwards L[k][k] = sqrt(p_k), L[i][k] = a[i][k] / sqrt(p_k)
  // (_cholesky, linalg.py:185-196; a non-positive p_k is NotSPDError, :190-192)
  // 1/p_k leaves the chain: the next pivot p_{k+1} = a[k+1][k+1] - a[k+1][k]^2/p_k
  // is formed (by the thread that also writes it) and inverted at the start of
  // step k, while the other threads update; rpiv[k] holds 1/p_k
  __shared__ double rpiv[64];
  if (threadIdx.x == 0) {
    double p0 = a[0][0];
    if (!(p0 > 0.0) || !isfinite(p0)) p0 = 1.0;  // recorded below; keep the block finite
    rpiv[0] = 1.0 / p0;
  }
  __syncthreads();
  for (int k = 0; k < 63; ++k) {
    const double rp = rpiv[k];
    const int ti = threadIdx.x >> 4, tj = threadIdx.x & 15;
    if (threadIdx.x == 0) {  // the same arithmetic as the (k+1, k+1) update below
      const double l1 = a[k + 1][k] * rp;
      double pn = fma(-l1, a[k + 1][k], a[k + 1][k + 1]);
      if (!(pn > 0.0) || !isfinite(pn)) pn = 1.0;
      rpiv[k + 1] = 1.0 / pn;
    }
    // 16 x 16 thread grid over the trailing lower triangle, no index division
    for (int i = k + 1 + ti; i < 64; i += 16) {
      const double li = a[i][k] * rp;
      for (int j = k + 1 + tj; j <= i; j += 16) a[i][j] = fma(-li, a[j][k], a[i][j]);
    }
    __syncthreads();
  }
  if (threadIdx.x < 64) {
    const double p = a[threadIdx.x][threadIdx.x];
    if (!(p > 0.0) || !isfinite(p)) atomicMin(&bad, (int)threadIdx.x);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 64 * 64; e += 256) {  // scale columns (diagonal last)
    const int r = e >> 6, c = e & 63;
    if (c >= r) continue;
    double p = a[c][c];
    if (!(p > 0.0) || !isfinite(p)) p = 1.0;
    a[r][c] = a[r][c] / sqrt(p);
  }
  __syncthreads();
  if (threadIdx.x < 64) {
    double p = a[threadIdx.x][threadIdx.x];
    if (!(p > 0.0) || !isfinite(p)) p = 1.0;
    a[threadIdx.x][threadIdx.x] = sqrt(p);
  }
  __syncthreads();
  // X = L^-1 right-looking: rows below k lose L[i][k] X[k] / L[k][k], then row
  // k is scaled; one barrier per step. x[i][j] (i > j) lives at a[j][i].
  if (threadIdx.x < 64) rpiv[threadIdx.x] = 1.0 / a[threadIdx.x][threadIdx.x];  // 1 / L[k][k], all at once
  __syncthreads();
  for (int k = 0; k < 64; ++k) {
    const double rk = rpiv[k];
    const int cols = k + 1;
    const int ti = threadIdx.x >> 4, tj = threadIdx.x & 15;
    for (int i = k + 1 + ti; i < 64; i += 16) {
      const double li = a[i][k] * rk;
      for (int j = tj; j < cols; j += 16) {
        const double xkj = (j == k) ? xd[k] : a[j][k];
        a[j][i] = fma(-li, xkj, a[j][i]);
      }
    }
    __syncthreads();
    if (threadIdx.x < cols) {
      if (threadIdx.x == k) xd[k] *= rk;
      else a[threadIdx.x][k] *= rk;
    }
  }
  __syncthreads();
  double* iv = inv + ((int64_t)leaf * (lb.m_pad / 64) + j0 / 64) * 64 * 64;
#pragma unroll 4
  for (int e = threadIdx.x; e < 64 * 64; e += 256) {
    const int r = e >> 6, c = e & 63;
    A[r * ld + c] = (c <= r) ? a[r][c] : 0.0;
    iv[e] = (c < r) ? a[c][r] : (c == r ? xd[r] : 0.0);
  }
  if (threadIdx.x == 0 && bad != 0x7fffffff && info[leaf] == 0) info[leaf] = j0 + bad + 1;
}

void launch_potrf64(const LeafBatch& lb, int j0, double* inv, int* info, cudaStream_t st) {
  constexpr size_t smem = (64 * 65 + 64) * sizeof(double);
  ensure_smem(k_potrf64, smem);
  launch_pdl(k_potrf64, dim3(lb.count), dim3(256), smem, st, lb, j0, inv, info);
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

// Upper triangle := lower triangle (SYRK computed on lower tiles only).
__global__ void k_mirror_lower(double* H, int64_t stride, const int* idx, int s) {
  pdl_wait();
  double* h = H + (int64_t)idx[blockIdx.y] * stride;
  const int64_t total = (int64_t)s * s;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / s), j = (int)(e % s);
    if (j > i) h[e] = h[(int64_t)j * s + i];
  }
}

void launch_mirror_lower(double* H, int64_t h_stride, const int* node_idx, int count, int s_pad, cudaStream_t st) {
  if (count <= 0 || s_pad <= 0) return;
  dim3 g(32, count);
  launch_pdl(k_mirror_lower, g, dim3(256), 0, st, H, h_stride, node_idx, s_pad);
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
  pdl_wait();
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
  launch_pdl(k_coupling, g, dim3(256), 0, st, t, nb);
}

// Identity diagonal blocks of Z, P^T (top right), zero bottom-right block, and
// the padded P copy used by the solve. Z12/Z21 and -PG are written by GEMMs.
// Padded candidate index i' maps to the reference's cand index
// (cand = [skel_l; skel_r], compress.py:213): i' < s_pad -> i' (if < s_l),
// i' >= s_pad -> s_l + (i' - s_pad) (if < s_r).
__device__ __forceinline__ int cand_index(int i, int S, int sl, int sr) {
  return (i < S) ? (i < sl ? i : -1) : (i - S < sr ? sl + (i - S) : -1);
}

// one CTA per row: rows [0, TP) the identity diagonal blocks of Z, rows
// [TP, T) the zero bottom-right block, then the S rows of the padded P copy
__global__ void __launch_bounds__(256) k_aug_init(DevTree t, NodeBatch nb) {
  pdl_wait();
  const int k = blockIdx.y, row = blockIdx.x;
  const int S = nb.s_pad, TP = nb.t_pad, T = nb.T;
  double* A = nb.Aug + (int64_t)k * T * T;
  if (row < TP) {  // (a) identity block of Z: row i, columns of its half
    const int half = row / S, i = row - half * S;
    double* out = A + (int64_t)row * T + half * S;
    for (int j = threadIdx.x; j < S; j += 256) out[j] = (i == j) ? 1.0 : 0.0;
    return;
  }
  if (row < T) {  // (c) zero block S x S at (TP, TP)
    double* out = A + (int64_t)row * T + TP;
    for (int j = threadIdx.x; j < S; j += 256) out[j] = 0.0;
    return;
  }
  // (d) Pn row j: P[j][cand(i)] for the padded candidate index i
  const int j = row - T;
  const int v = nb.node[k], sl = t.rank[nb.left[k]], sr = t.rank[nb.right[k]], sv = t.rank[v];
  const double* P = t.coeff + t.coeff_off[v] + (int64_t)j * (sl + sr);
  double* out = nb.Pn + (int64_t)k * S * TP + (int64_t)j * TP;
  for (int i = threadIdx.x; i < TP; i += 256) {
    const int ci = cand_index(i, S, sl, sr);
    out[i] = (ci >= 0 && j < sv) ? P[ci] : 0.0;
  }
}

// (b) the P^T block (TP x S at (0, TP)) through 32 x 32 shared-memory tiles:
// reads along P's rows, writes along Aug's rows
__global__ void __launch_bounds__(256) k_aug_pt(DevTree t, NodeBatch nb) {
  pdl_wait();
  __shared__ double tile[32][33];
  const int k = blockIdx.z;
  const int S = nb.s_pad, TP = nb.t_pad, T = nb.T;
  const int v = nb.node[k], sl = t.rank[nb.left[k]], sr = t.rank[nb.right[k]], sv = t.rank[v];
  const double* P = t.coeff + t.coeff_off[v];
  const int cand = sl + sr;
  const int j0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  {
    const int ci = cand_index(i0 + tx, S, sl, sr);
    for (int jj = ty; jj < 32; jj += 8) {
      const int j = j0 + jj;
      tile[jj][tx] = (ci >= 0 && j < sv) ? P[(int64_t)j * cand + ci] : 0.0;
    }
  }
  __syncthreads();
  double* A = nb.Aug + (int64_t)k * T * T;
  for (int ii = ty; ii < 32; ii += 8) A[(int64_t)(i0 + ii) * T + TP + j0 + tx] = tile[tx][ii];
}

void launch_aug_init(const DevTree& t, const NodeBatch& nb, cudaStream_t st) {
  launch_pdl(k_aug_init, dim3(nb.T + nb.s_pad, nb.count), dim3(256), 0, st, t, nb);
  launch_pdl(k_aug_pt, dim3(nb.s_pad / 32, nb.t_pad / 32, nb.count), dim3(256), 0, st, t, nb);
}

// 1-norm of Z (max column abs sum, linalg.py:176), before the LU overwrites it.
// 32 columns per CTA, rows split over 8 warps; the max over column tiles goes
// through an integer atomicMax on the (non-negative) double's bit pattern.
__global__ void __launch_bounds__(256) k_colnorm1(NodeBatch nb) {
  pdl_wait();
  const int k = blockIdx.y;
  const double* A = nb.Aug + (int64_t)k * nb.T * nb.T;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * 32 + lane;
  __shared__ double red[8][33];
  double s = 0.0;
  if (c < nb.t_pad)
#pragma unroll 8
    for (int i = warp; i < nb.t_pad; i += 8) s += fabs(A[(int64_t)i * nb.T + c]);
  red[warp][lane] = s;
  __syncthreads();
  if (warp == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w][lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t = fmax(t, __shfl_xor_sync(0xffffffffu, t, o));
    if (lane == 0) atomicMax(reinterpret_cast<unsigned long long*>(nb.norm1 + k), __double_as_longlong(t));
  }
}

void launch_colnorm1(const DevTree&, const NodeBatch& nb, cudaStream_t st) {
  cudaMemsetAsync(nb.norm1, 0, sizeof(double) * nb.count, st);
  dim3 g((nb.t_pad + 31) / 32, nb.count);
  launch_pdl(k_colnorm1, g, dim3(256), 0, st, nb);
}

// --------------------------------------------------------------------------
// LU with partial pivoting restricted to rows < t_pad (linalg.py:199-213 on
// the Z block; the -PG rows are eliminated but never chosen as pivots): one
// W-column panel per launch and node (k_lu_panel2). The candidate rows live in
// registers and never move inside the panel; each thread tracks its rows'
// LOGICAL positions (the reference's swap sequence, swaps[k] = p). The column
// loop is lu_panel.cuh (shared with the persistent LU of lu_slab.cu); then the
// rows go back to their logical positions (coalesced), the augmented rows are
// eliminated against the panel's U rows (coalesced through shared memory), and
// the panel's row interchanges are applied to every column outside it (all
// loads of a column chunk, one barrier, all stores).
// --------------------------------------------------------------------------
// probe hook (ks_probe_panel): clock64 stamps of CTA 0 at phase boundaries
__device__ long long* g_panel_clk = nullptr;
#define PANEL_STAMP(i)                                                   \
  do {                                                                   \
    if (clk && threadIdx.x == 0) clk[i] = clock64();                     \
  } while (0)

template <int W, int RPT, int NT, int MINB = 1>
__global__ void __launch_bounds__(NT, MINB) k_lu_panel2(NodeBatch nb, int c0, int pr0, int pc0, int ph, int pcols) {
  pdl_wait();
  long long* clk = blockIdx.x == 0 ? g_panel_clk : nullptr;
  PANEL_STAMP(0);
  constexpr int NW = NT / 32;
  constexpr int CB = 4;
  constexpr int FS = W + 2;
  static_assert(NW <= 32 && W % CB == 0, "panel shape");
  const int k = blockIdx.x;
  const int T = nb.T;
  double* A = nb.Aug + (int64_t)k * T * T;
  if (ph > 0) {  // U12 of the preceding fused merge (k_lu_merge), disjoint from this panel
    const double* sc = nb.scratch + (int64_t)k * 32 * 64;
    for (int e = threadIdx.x; e < ph * pcols; e += NT) {
      const int i = e / pcols, j = e % pcols;
      A[(int64_t)(pr0 + i) * T + pc0 + j] = sc[i * 64 + j];
    }
  }
  const int rows = nb.t_pad - c0;
  extern __shared__ __align__(16) double fin[];  // rows x FS finished values
  __shared__ PanelShared<NW, W> ps;
  __shared__ double u11[W][W + 1];
  double a[RPT][W];
  int pos[RPT];
  bool done[RPT];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int r = threadIdx.x + i * NT;
    pos[i] = r;
    done[i] = (r >= rows);
    const double2* src = reinterpret_cast<const double2*>(A + (int64_t)(c0 + (r < rows ? r : 0)) * T + c0);
#pragma unroll
    for (int j = 0; j < W / 2; ++j) {
      const double2 v = (r < rows) ? src[j] : make_double2(0.0, 0.0);
      a[i][2 * j] = v.x;
      a[i][2 * j + 1] = v.y;
    }
  }
  PANEL_STAMP(1);
  {
    const int nact = panel_warps(rows, NT);
    if ((int)(threadIdx.x >> 5) < nact)
      panel_columns<W, RPT, NT, (W <= 16 ? W : 16)>(a, pos, done, ps, fin, FS, rows, nb.piv + (int64_t)k * nb.t_pad + c0,
                                                  c0, nb.info + k, c0, nact);
  }
  __syncthreads();
  PANEL_STAMP(20);
  // panel rows back to their logical positions (coalesced: W/2 threads per
  // row); the pivot rows (U) to u11
  __shared__ int spos[RPT * NT];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int r = threadIdx.x + i * NT;
    if (r >= rows) continue;
    spos[r] = pos[i];
    if (pos[i] < W) {
#pragma unroll
      for (int j = 0; j < W; ++j) u11[pos[i]][j] = fin[r * FS + j];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < rows * (W / 2); e += NT) {
    const int r = e / (W / 2), j2 = 2 * (e % (W / 2));
    *reinterpret_cast<double2*>(A + (int64_t)(c0 + spos[r]) * T + c0 + j2) =
        *reinterpret_cast<const double2*>(fin + r * FS + j2);
  }
  // the augmented rows, eliminated against the panel's pivot rows; loaded and
  // stored W/2 lanes per row (coalesced) through the finished-value buffer
  __syncthreads();  // fin is free once the panel rows are written back
  PANEL_STAMP(21);
  const int naug = T - nb.t_pad;
  for (int e = threadIdx.x; e < naug * (W / 2); e += NT) {
    const int r = e / (W / 2), j2 = 2 * (e % (W / 2));
    *reinterpret_cast<double2*>(fin + r * FS + j2) =
        *reinterpret_cast<const double2*>(A + (int64_t)(nb.t_pad + r) * T + c0 + j2);
  }
  __syncthreads();
  for (int r = threadIdx.x; r < naug; r += NT) {
    double2* row = reinterpret_cast<double2*>(fin + r * FS);
    const double* ut = &u11[0][0];
    asm volatile("" : "+l"(ut));
    double x[W];
#pragma unroll
    for (int j = 0; j < W / 2; ++j) {
      const double2 v = row[j];
      x[2 * j] = v.x;
      x[2 * j + 1] = v.y;
    }
#pragma unroll
    for (int kk = 0; kk < W; ++kk) {
      const double l = x[kk] * ps.urcp[kk];
      x[kk] = l;
#pragma unroll
      for (int j = kk + 1; j < W; ++j) x[j] = fma(-l, ut[kk * (W + 1) + j], x[j]);
    }
#pragma unroll
    for (int j = 0; j < W / 2; ++j) row[j] = make_double2(x[2 * j], x[2 * j + 1]);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < naug * (W / 2); e += NT) {
    const int r = e / (W / 2), j2 = 2 * (e % (W / 2));
    *reinterpret_cast<double2*>(A + (int64_t)(nb.t_pad + r) * T + c0 + j2) =
        *reinterpret_cast<const double2*>(fin + r * FS + j2);
  }
  // the same row interchanges for every column outside the panel
  __shared__ int msrc[RPT * NT < 2 * W ? RPT * NT : 2 * W], mdst[RPT * NT < 2 * W ? RPT * NT : 2 * W];
  __shared__ int nmove;
  if (threadIdx.x == 0) nmove = 0;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int r = threadIdx.x + i * NT;
    if (r < rows && pos[i] != r) {
      const int slot = atomicAdd(&nmove, 1);
      msrc[slot] = c0 + r;
      mdst[slot] = c0 + pos[i];
    }
  }
  __syncthreads();
  PANEL_STAMP(22);
  const int nm = nmove;
  const int npair = (T - W) / 2;  // column pairs outside the panel
  constexpr int PER = 12;         // double2 per thread per chunk
  for (int e0 = 0; e0 < nm * npair; e0 += PER * NT) {
    double2 v[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = e0 + u * NT + threadIdx.x;
      if (e < nm * npair) {
        const int m = e / npair, x = 2 * (e % npair);
        const int col = x < c0 ? x : x + W;
        v[u] = *reinterpret_cast<const double2*>(A + (int64_t)msrc[m] * T + col);
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = e0 + u * NT + threadIdx.x;
      if (e < nm * npair) {
        const int m = e / npair, x = 2 * (e % npair);
        const int col = x < c0 ? x : x + W;
        *reinterpret_cast<double2*>(A + (int64_t)mdst[m] * T + col) = v[u];
      }
    }
  }
  PANEL_STAMP(23);
  if (clk && threadIdx.x == 0) clk[24] = nm;
}

template <int W, int RPT, int NT, int MINB = 1>
static void launch_panel(const NodeBatch& nb, int c0, cudaStream_t st, const int* pend) {
  const size_t smem = (size_t)std::max(nb.t_pad - c0, nb.T - nb.t_pad) * (W + 2) * sizeof(double);
  ensure_smem(k_lu_panel2<W, RPT, NT, MINB>, smem);
  launch_pdl(k_lu_panel2<W, RPT, NT, MINB>, dim3(nb.count), dim3(NT), smem, st, nb, c0, pend[0], pend[1], pend[2],
             pend[3]);
}

template <int W>
static void launch_panel_w(const NodeBatch& nb, int c0, cudaStream_t st, const int* pend) {
  // 512 threads (16 warps hide the per-column latency), rows in registers.
  // (A 256-thread, two-CTAs-per-SM variant for batches wider than the GPU
  // measured no better: the two node-group streams already fill the SMs.)
  const int rows = nb.t_pad - c0;
  if constexpr (W == 32) {  // 32 columns in registers: one row per thread, t_pad <= 512
    launch_panel<W, 1, 512>(nb, c0, st, pend);
  } else {
    if (rows <= 512) launch_panel<W, 1, 512>(nb, c0, st, pend);
    else if (rows <= 1024) launch_panel<W, 2, 512>(nb, c0, st, pend);
    else if constexpr (W <= 8) {
      if (rows <= 1536) launch_panel<W, 3, 512>(nb, c0, st, pend);
      else launch_panel<W, 4, 512>(nb, c0, st, pend);
    }
  }
}

void launch_lu_panel(const NodeBatch& nb, int c0, int w, cudaStream_t st, const int* pend) {
  static const int none[4] = {0, 0, 0, 0};
  if (!pend) pend = none;
  if (w == 32) launch_panel_w<32>(nb, c0, st, pend);
  else if (w == 16) launch_panel_w<16>(nb, c0, st, pend);
  else launch_panel_w<8>(nb, c0, st, pend);
}

// B := L^-1 B for the unit-lower W x W block at (r0, r0), B = rows r0..r0+W,
// columns [c0, c0+ncols). One thread per column, x held in registers.
template <int W>
__global__ void __launch_bounds__(128) k_trsm_ul(NodeBatch nb, int r0, int c0, int ncols) {
  pdl_wait();
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
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;  // 4 chains: DFMA latency, not issue, bounds this loop
#pragma unroll
    for (int j = 0; j + 3 < i; j += 4) {
      s0 = fma(L[i][j], x[j], s0);
      s1 = fma(L[i][j + 1], x[j + 1], s1);
      s2 = fma(L[i][j + 2], x[j + 2], s2);
      s3 = fma(L[i][j + 3], x[j + 3], s3);
    }
#pragma unroll
    for (int j = i & ~3; j < i; ++j) s0 = fma(L[i][j], x[j], s0);
    x[i] -= (s0 + s1) + (s2 + s3);
  }
#pragma unroll
  for (int i = 0; i < W; ++i) B[(int64_t)i * T] = x[i];
}

void launch_trsm_unit_lower(const NodeBatch& nb, int r0, int w, int c0, int ncols, cudaStream_t st) {
  if (ncols <= 0) return;
  dim3 g((ncols + 127) / 128, nb.count);
  if (w == 8) launch_pdl(k_trsm_ul<8>, g, dim3(128), 0, st, nb, r0, c0, ncols);
  else if (w == 16) launch_pdl(k_trsm_ul<16>, g, dim3(128), 0, st, nb, r0, c0, ncols);
  else if (w == 32) launch_pdl(k_trsm_ul<32>, g, dim3(128), 0, st, nb, r0, c0, ncols);
  else launch_pdl(k_trsm_ul<64>, g, dim3(128), 0, st, nb, r0, c0, ncols);
}

// --------------------------------------------------------------------------
// Hager 1-norm condition estimate of Z (linalg.py:282-304), one CTA per node,
// on the LU factors in place (blocked CTA triangular solves, trsv.cuh). Only
// real (unpadded) indices take part, in the reference's index order.
// --------------------------------------------------------------------------
__device__ __forceinline__ void block_argmax(double& bv, int& bi, double* rv, int* ri) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  if (lane == 0) { rv[warp] = bv; ri[warp] = bi; }
  __syncthreads();
  bv = rv[0];
  bi = ri[0];
  for (int w = 1; w < SWARPS; ++w)
    if (rv[w] > bv || (rv[w] == bv && ri[w] < bi)) { bv = rv[w]; bi = ri[w]; }
  __syncthreads();
}

__device__ __forceinline__ double block_sum(double v, double* rv) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  v = warp_sum(v);
  if (lane == 0) rv[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < SWARPS; ++w) s += rv[w];
  __syncthreads();
  return s;
}

__global__ void __launch_bounds__(STHREADS) k_hager(DevTree t, NodeBatch nb) {
  extern __shared__ double hv[];  // x, y, w (t_pad each) + red (SWARPS*32) ; int perm (t_pad)
  __shared__ double D[SB][SB + 1];
  __shared__ double rv[SWARPS];
  __shared__ int ri[SWARPS];
  const int k = blockIdx.x;
  const int TP = nb.t_pad, S = nb.s_pad, T = nb.T;
  const int sl = t.rank[nb.left[k]], sr = t.rank[nb.right[k]];
  const int n = sl + sr;
  const double* A = nb.Aug + (int64_t)k * T * T;
  double* x = hv;
  double* y = hv + TP;
  double* w = hv + 2 * TP;
  double* red = hv + 3 * TP;
  int* pm = reinterpret_cast<int*>(red + SWARPS * 32);  // (Pi v)[i] = v[pm[i]]
  if (n == 0) {
    if (threadIdx.x == 0) nb.cond[k] = 0.0;
    return;
  }
  for (int i = threadIdx.x; i < TP; i += STHREADS) pm[i] = nb.pm[(int64_t)k * TP + i];  // composed swaps
  auto real = [&](int i) { return i < S ? (i < sl) : (i - S < sr); };
  for (int i = threadIdx.x; i < TP; i += STHREADS) x[i] = real(i) ? 1.0 / n : 0.0;
  __syncthreads();
  double est = 0.0;
  for (int it = 0; it < 5; ++it) {
    // y = Z^-1 x   (dense_solve: swaps, unit L, U)
    for (int i = threadIdx.x; i < TP; i += STHREADS) y[i] = x[pm[i]];
    __syncthreads();
    cta_trsv_rows<1, false, true>(A, T, TP, y, D);
    cta_trsv_rows<1, true, false>(A, T, TP, y, D);
    double s = 0.0;
    for (int i = threadIdx.x; i < TP; i += STHREADS) s += real(i) ? fabs(y[i]) : 0.0;
    est = block_sum(s, rv);
    // z = Z^-T sign(y)   (solve_transposed: U^T, unit L^T, undo swaps)
    for (int i = threadIdx.x; i < TP; i += STHREADS) w[i] = real(i) ? (y[i] >= 0.0 ? 1.0 : -1.0) : 0.0;
    __syncthreads();
    cta_trsv_trans<1, true, false>(A, T, TP, w, D, red);
    cta_trsv_trans<1, false, true>(A, T, TP, w, D, red);
    for (int i = threadIdx.x; i < TP; i += STHREADS) y[pm[i]] = w[i];  // y <- z (unpermuted)
    __syncthreads();
    // j = argmax |z| (first in reference order on ties), z . x
    double bv = -1.0, dot = 0.0;
    int bi = 0x7fffffff;
    for (int i = threadIdx.x; i < TP; i += STHREADS) {
      if (!real(i)) continue;
      const double a = fabs(y[i]);
      const int r = i < S ? i : sl + (i - S);
      if (a > bv || (a == bv && r < bi)) { bv = a; bi = r; }
      dot = fma(y[i], x[i], dot);
    }
    block_argmax(bv, bi, rv, ri);
    dot = block_sum(dot, rv);
    if (bv <= dot) break;
    const int jp = bi < sl ? bi : S + (bi - sl);
    for (int i = threadIdx.x; i < TP; i += STHREADS) x[i] = (i == jp) ? 1.0 : 0.0;
    __syncthreads();
  }
  if (threadIdx.x == 0) nb.cond[k] = isfinite(est) ? nb.norm1[k] * est : INFINITY;
}

static void launch_hager_blocked(const DevTree& t, const NodeBatch& nb, cudaStream_t st) {
  const size_t smem = sizeof(double) * (3 * nb.t_pad + SWARPS * 32) + sizeof(int) * nb.t_pad;
  ensure_smem(k_hager, smem);
  k_hager<<<nb.count, STHREADS, smem, st>>>(t, nb);
}

// --------------------------------------------------------------------------
// The same estimate with thread-owned vectors (t_pad <= 1024): thread i owns
// entry i of every vector. A triangular solve walks SB-row blocks; the
// coefficients coupling the next block to each thread's entry are loaded one
// step ahead, the diagonal block goes through its inverse (precomputed by
// k_diag_inv, staged in shared memory) as an SB-wide shuffle GEMV, so a block
// step is a handful of dependent operations and one barrier.
// --------------------------------------------------------------------------
enum { SOLVE_L = 0, SOLVE_U = 1, SOLVE_UT = 2, SOLVE_LT = 3 };

// inverses of the SB x SB diagonal blocks of unit-lower L (which 0) and upper
// U (which 1) of every node's Z factors: dinv[node][which][b][s][t]
template <int SB>
__global__ void __launch_bounds__(256) k_diag_inv(NodeBatch nb, double* dinv) {
  const int k = blockIdx.x, which = blockIdx.y;
  const int TP = nb.t_pad, T = nb.T;
  const double* A = nb.Aug + (int64_t)k * T * T;
  double* out = dinv + ((int64_t)(nb.first + k) * 2 + which) * TP * SB;
  for (int task = threadIdx.x; task < TP; task += 256) {
    const int b = task / SB, j = task % SB;  // column j of block b's inverse
    const int r0 = b * SB;
    double x[SB];
    if (which == 0) {
#pragma unroll
      for (int s2 = 0; s2 < SB; ++s2) {
        double v = (s2 == j) ? 1.0 : 0.0;
#pragma unroll
        for (int t2 = 0; t2 < s2; ++t2)
          if (t2 >= j) v = fma(-A[(int64_t)(r0 + s2) * T + r0 + t2], x[t2], v);
        x[s2] = (s2 < j) ? 0.0 : v;
      }
    } else {
#pragma unroll
      for (int s2 = SB - 1; s2 >= 0; --s2) {
        double v = (s2 == j) ? 1.0 : 0.0;
#pragma unroll
        for (int t2 = s2 + 1; t2 < SB; ++t2)
          if (t2 <= j) v = fma(-A[(int64_t)(r0 + s2) * T + r0 + t2], x[t2], v);
        x[s2] = (s2 > j) ? 0.0 : v / A[(int64_t)(r0 + s2) * T + r0 + s2];
      }
    }
#pragma unroll
    for (int s2 = 0; s2 < SB; ++s2) out[(int64_t)b * SB * SB + s2 * SB + j] = x[s2];
  }
}

// v (thread i's entry) <- M^-1 v for M = L (unit lower), U, U^T or L^T of the
// packed factors in A (rows of length lda); di: the matching diagonal-block
// inverses in shared memory; xs: a shared broadcast buffer (n entries).
// COLMAJ: A is the column-major copy of the factors (At[j][i] = A[i][j]), so
// the non-transposed solves read it down columns like the transposed ones
// (coalesced across the threads that own consecutive entries)
template <int SB, int NT, int MODE, bool COLMAJ = false>
__device__ __forceinline__ double own_solve(const double* __restrict__ A, int64_t lda, int n, const double* di, double v,
                            double* xs) {
  constexpr bool ASC = (MODE == SOLVE_L || MODE == SOLVE_UT);
  constexpr bool TRANS = (MODE == SOLVE_UT || MODE == SOLVE_LT);
  constexpr bool COLACC = TRANS || COLMAJ;
  const int i = threadIdx.x, lane = i & 31;
  const bool own = i < n;
  const int nblk = n / SB;
  double cur[SB], nxt[SB];
  auto load = [&](int b, double (&c)[SB]) {
    const int r0 = b * SB;
    const bool need = own && (ASC ? i >= r0 + SB : i < r0);  // solved after block b
    if (COLACC) {
      const double* p = A + (int64_t)r0 * lda + (own ? i : 0);
#pragma unroll
      for (int j = 0; j < SB; ++j, p += lda) c[j] = need ? __ldg(p) : 0.0;
    } else {
      const double2* p = reinterpret_cast<const double2*>(A + (int64_t)(own ? i : 0) * lda + r0);
#pragma unroll
      for (int j = 0; j < SB / 2; ++j) {
        const double2 u = need ? __ldg(p + j) : make_double2(0.0, 0.0);
        c[2 * j] = u.x;
        c[2 * j + 1] = u.y;
      }
    }
  };
  load(ASC ? 0 : nblk - 1, cur);
  __syncthreads();  // xs may still be read by the caller's previous phase
#pragma unroll 1
  for (int step = 0; step < nblk; ++step) {
    const int b = ASC ? step : nblk - 1 - step;
    if (step + 1 < nblk) load(ASC ? b + 1 : b - 1, nxt);
    const int r0 = b * SB;
    if ((i >> 5) == (r0 >> 5)) {  // the warp holding block b: x_b = D_b^-1 v_b
      const int base = r0 & 31, s2 = lane - base;
      const bool inb = own && s2 >= 0 && s2 < SB;
      const double* d = di + (int64_t)b * SB * SB;
      double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
      for (int t2 = 0; t2 < SB; t2 += 2) {
        const double v0 = __shfl_sync(0xffffffffu, v, base + t2);
        const double v1 = __shfl_sync(0xffffffffu, v, base + t2 + 1);
        if (inb) {
          acc0 = fma(TRANS ? d[t2 * SB + s2] : d[s2 * SB + t2], v0, acc0);
          acc1 = fma(TRANS ? d[(t2 + 1) * SB + s2] : d[s2 * SB + t2 + 1], v1, acc1);
        }
      }
      if (inb) {
        v = acc0 + acc1;
        xs[i] = v;
      }
    }
    __syncthreads();
    const bool after = own && (ASC ? i >= r0 + SB : i < r0);
    if (after) {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int j = 0; j < SB; j += 2) {
        s0 = fma(cur[j], xs[r0 + j], s0);
        s1 = fma(cur[j + 1], xs[r0 + j + 1], s1);
      }
      v -= s0 + s1;
    }
#pragma unroll
    for (int j = 0; j < SB; ++j) cur[j] = nxt[j];
  }
  return v;
}

// The non-transposed solves (L, U) with the coefficient loads coalesced: each
// thread needs the 8 coefficients of its own row, but one row per lane makes
// every load instruction touch 32 cache lines (the L1 tag lookups, not the
// bytes, bound the step). Here the CTA loads the block's row segments 4 lanes
// per row (8 lines per instruction), one step ahead, and stages them through
// shared memory (cb: 2 x NT x 10 doubles); the step's barrier publishes them.
template <int NT, int MODE>
__device__ __forceinline__ double own_solve_rows(const double* __restrict__ A, int64_t lda, int n, const double* di,
                                                 double v, double* xs, double* cb) {
  constexpr int SB = 8, CS = 10;  // 8 coefficients per row, padded row stride (16 B aligned, conflict-free)
  constexpr bool ASC = (MODE == SOLVE_L);
  static_assert(MODE == SOLVE_L || MODE == SOLVE_U, "non-transposed solves only");
  const int i = threadIdx.x, lane = i & 31;
  const bool own = i < n;
  const int nblk = n / SB;
  double2 ld[4];
  auto issue = [&](int b) {
    const int r0 = b * SB;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = threadIdx.x + u * NT, row = c >> 2, part = c & 3;
      const bool need = row < n && (ASC ? row >= r0 + SB : row < r0);
      ld[u] = need ? ldg2(A + (int64_t)row * lda + r0 + 2 * part) : make_double2(0.0, 0.0);
    }
  };
  auto stage = [&](int st) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = threadIdx.x + u * NT, row = c >> 2, part = c & 3;
      if (row < NT) *reinterpret_cast<double2*>(cb + ((int64_t)st * NT + row) * CS + 2 * part) = ld[u];
    }
  };
  __syncthreads();  // xs and cb may still be read by the caller's previous phase
  issue(ASC ? 0 : nblk - 1);
  stage(0);
#pragma unroll 1
  for (int step = 0; step < nblk; ++step) {
    const int b = ASC ? step : nblk - 1 - step;
    if (step + 1 < nblk) issue(ASC ? b + 1 : b - 1);
    const int r0 = b * SB;
    if ((i >> 5) == (r0 >> 5)) {  // the warp holding block b: x_b = D_b^-1 v_b
      const int base = r0 & 31, s2 = lane - base;
      const bool inb = own && s2 >= 0 && s2 < SB;
      const double* d = di + (int64_t)b * SB * SB;
      double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
      for (int t2 = 0; t2 < SB; t2 += 2) {
        const double v0 = __shfl_sync(0xffffffffu, v, base + t2);
        const double v1 = __shfl_sync(0xffffffffu, v, base + t2 + 1);
        if (inb) {
          acc0 = fma(d[s2 * SB + t2], v0, acc0);
          acc1 = fma(d[s2 * SB + t2 + 1], v1, acc1);
        }
      }
      if (inb) {
        v = acc0 + acc1;
        xs[i] = v;
      }
    }
    __syncthreads();
    const bool after = own && (ASC ? i >= r0 + SB : i < r0);
    if (after) {
      const double* c = cb + ((int64_t)(step & 1) * NT + i) * CS;
      double q0 = 0.0, q1 = 0.0;
#pragma unroll
      for (int j = 0; j < SB; j += 2) {
        const double2 cc = *reinterpret_cast<const double2*>(c + j);
        q0 = fma(cc.x, xs[r0 + j], q0);
        q1 = fma(cc.y, xs[r0 + j + 1], q1);
      }
      v -= q0 + q1;
    }
    if (step + 1 < nblk) stage((step + 1) & 1);
  }
  return v;
}

template <int NT>
__device__ __forceinline__ double nt_sum(double v, double* red) {
  constexpr int NWp = NT / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < NWp; ++w) s += red[w];
  return s;
}

template <int NT>
__device__ __forceinline__ void nt_argmax(double& bv, int& bi, double* red, int* redi) {
  constexpr int NWp = NT / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  __syncthreads();
  if (lane == 0) { red[warp] = bv; redi[warp] = bi; }
  __syncthreads();
  bv = red[0];
  bi = redi[0];
#pragma unroll
  for (int w = 1; w < NWp; ++w)
    if (red[w] > bv || (red[w] == bv && redi[w] < bi)) { bv = red[w]; bi = redi[w]; }
}

template <int SB, int NT, bool COLMAJ>
__global__ void __launch_bounds__(NT, 1) k_hager_own(DevTree t, NodeBatch nb, const double* dinv, const double* lut) {
  extern __shared__ __align__(16) double hs[];
  // persistent over nodes: the grid may be smaller than the batch so that the
  // estimate leaves SMs free for the factorization it overlaps
  for (int k = blockIdx.x; k < nb.count; k += gridDim.x) {
  __syncthreads();
  const int TP = nb.t_pad, S = nb.s_pad, T = nb.T;
  const int sl = t.rank[nb.left[k]], sr = t.rank[nb.right[k]];
  const int n = sl + sr;
  if (n == 0) {
    if (threadIdx.x == 0) nb.cond[k] = 0.0;
    continue;
  }
  double* dL = hs;                 // TP x SB
  double* dU = hs + TP * SB;       // TP x SB
  double* xs = dU + TP * SB;       // TP
  double* red = xs + TP;           // NT / 32
  int* redi = reinterpret_cast<int*>(red + NT / 32);
  int* pm = redi + NT / 32;        // TP: composed swaps, (Pi v)[i] = v[pm[i]]
  const double* A = nb.Aug + (int64_t)k * T * T;
  {
    const double2* src = reinterpret_cast<const double2*>(dinv + (int64_t)(nb.first + k) * 2 * TP * SB);
    double2* dst = reinterpret_cast<double2*>(hs);
    for (int e = threadIdx.x; e < TP * SB; e += NT) dst[e] = src[e];
    for (int e = threadIdx.x; e < TP; e += NT) pm[e] = nb.pm[(int64_t)k * TP + e];
  }
  const int i = threadIdx.x;
  const bool own = i < TP;
  const bool real = own && (i < S ? (i < sl) : (i - S < sr));
  const int ref = i < S ? i : sl + (i - S);  // reference index order
  double x = real ? 1.0 / n : 0.0;
  double est = 0.0;
  __syncthreads();
  for (int it = 0; it < 5; ++it) {
    // y = Z^-1 x   (dense_solve: swaps, unit L, U)
    if (own) xs[i] = x;
    __syncthreads();
    double y = own ? xs[pm[i]] : 0.0;
    if constexpr (COLMAJ) {
      const double* At = lut + (int64_t)(nb.first + k) * TP * TP;
      y = own_solve<SB, NT, SOLVE_L, true>(At, TP, TP, dL, y, xs);
      y = own_solve<SB, NT, SOLVE_U, true>(At, TP, TP, dU, y, xs);
    } else if constexpr (SB == 8 && NT == 512) {
      double* cb = reinterpret_cast<double*>(pm + TP);  // 2 x NT x 10 staged coefficients
      y = own_solve_rows<NT, SOLVE_L>(A, T, TP, dL, y, xs, cb);
      y = own_solve_rows<NT, SOLVE_U>(A, T, TP, dU, y, xs, cb);
    } else {
      y = own_solve<SB, NT, SOLVE_L>(A, T, TP, dL, y, xs);
      y = own_solve<SB, NT, SOLVE_U>(A, T, TP, dU, y, xs);
    }
    est = nt_sum<NT>(real ? fabs(y) : 0.0, red);
    // z = Z^-T sign(y)   (solve_transposed: U^T, unit L^T, undo swaps)
    double w = real ? (y >= 0.0 ? 1.0 : -1.0) : 0.0;
    w = own_solve<SB, NT, SOLVE_UT>(A, T, TP, dU, w, xs);
    w = own_solve<SB, NT, SOLVE_LT>(A, T, TP, dL, w, xs);
    __syncthreads();
    if (own) xs[pm[i]] = w;
    __syncthreads();
    const double z = own ? xs[i] : 0.0;
    // j = argmax |z| (first in reference order on ties), z . x
    double bv = real ? fabs(z) : -1.0;
    int bi = real ? ref : 0x7fffffff;
    nt_argmax<NT>(bv, bi, red, redi);
    const double dot = nt_sum<NT>(real ? z * x : 0.0, red);
    if (bv <= dot) break;
    const int jp = bi < sl ? bi : S + (bi - sl);
    x = (i == jp) ? 1.0 : 0.0;
  }
  if (threadIdx.x == 0) nb.cond[k] = isfinite(est) ? nb.norm1[k] * est : INFINITY;
  }
}

// column-major copy of each node's Z factors (L\U, t_pad x t_pad) for the
// estimator's non-transposed solves: lut[first + k] = Z_k^T
__global__ void __launch_bounds__(256) k_lu_transpose(NodeBatch nb, double* lut) {
  __shared__ double tt[32][33];
  const int k = blockIdx.z, TP = nb.t_pad, T = nb.T;
  const double* A = nb.Aug + (int64_t)k * T * T;
  double* At = lut + (int64_t)(nb.first + k) * TP * TP;
  const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 32; r += 8) tt[r][tx] = A[(int64_t)(i0 + r) * T + j0 + tx];
  __syncthreads();
  for (int r = ty; r < 32; r += 8) At[(int64_t)(j0 + r) * TP + i0 + tx] = tt[tx][r];
}

template <int SB, int NT, bool COLMAJ>
static void launch_hager_own(const DevTree& t, const NodeBatch& nb, double* dinv, double* lut, int max_ctas,
                             cudaStream_t st) {
  dim3 g(nb.count, 2);
  k_diag_inv<SB><<<g, 256, 0, st>>>(nb, dinv);
  if (COLMAJ) k_lu_transpose<<<dim3(nb.t_pad / 32, nb.t_pad / 32, nb.count), 256, 0, st>>>(nb, lut);
  size_t smem = sizeof(double) * (2 * (size_t)nb.t_pad * SB + nb.t_pad + 2 * NT / 32) + sizeof(int) * nb.t_pad;
  if (!COLMAJ && SB == 8 && NT == 512) smem = (smem + 15) / 16 * 16 + sizeof(double) * 2 * NT * 10;
  ensure_smem(k_hager_own<SB, NT, COLMAJ>, smem);
  k_hager_own<SB, NT, COLMAJ><<<std::min(nb.count, max_ctas), NT, smem, st>>>(t, nb, dinv, lut);
}

int hager_launches(const NodeBatch& nb) { return (nb.t_pad <= 512 && nb.count < 64) ? 3 : (nb.t_pad <= 1024 ? 2 : 1); }

void launch_hager(const DevTree& t, const NodeBatch& nb, double* dinv, double* lut, int max_ctas, cudaStream_t st) {
  const char* e = std::getenv("KS_HAGER_IMPL");
  if (e && e[0] == 'b') {
    launch_hager_blocked(t, nb, st);
    return;
  }
  if (nb.t_pad <= 512) {
    // the column-major copy pays for itself where the factors are still in L2
    // (narrow levels); for wide levels the extra HBM pass costs more than it saves
    if (lut && nb.count < 64) launch_hager_own<8, 512, true>(t, nb, dinv, lut, max_ctas, st);
    else launch_hager_own<8, 512, false>(t, nb, dinv, lut, max_ctas, st);
  } else if (nb.t_pad <= 1024) launch_hager_own<8, 1024, false>(t, nb, dinv, nullptr, max_ctas, st);
  else launch_hager_blocked(t, nb, st);
}

// LU fallback for leaves whose Cholesky failed (solver.py:125-131): the
// augmented matrix [[A, -P^T], [P, 0]], A = K(X_leaf, X_leaf) + lam I (both
// triangles), with the leaf's padded identity; its LU restricted to the first
// m_pad pivots leaves the Schur complement P A^-1 P^T = H in the trailing block.
// fb: count = failed leaves, node = their node ids, t_pad = m_pad, T = m_pad + s_pad.
__global__ void __launch_bounds__(256) k_fb_assemble(DevTree t, NodeBatch fb, const int* begin, const int* size,
                                                     const double* lam_p) {
  const int k = blockIdx.z;
  const int v = fb.node[k], b0 = begin[k], m = size[k];
  const int TP = fb.t_pad, T = fb.T, S = T - TP;
  double* A = fb.Aug + (int64_t)k * T * T;
  const int r0 = blockIdx.y * GT, c0 = blockIdx.x * GT;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  if (r0 < TP && c0 < TP) {
    double sq[4][4];
    gauss_tile<false>(t, nullptr, b0, m, nullptr, b0, m, r0, c0, sq);
    const double den = -2.0 * t.h * t.h, lam = *lam_p;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = r0 + ty + 16 * i, c = c0 + tx + 16 * j;
        double val;
        if (r >= m || c >= m) val = (r == c) ? 1.0 : 0.0;
        else val = exp(sq[i][j] / den) + (r == c ? lam : 0.0);
        A[(int64_t)r * T + c] = val;
      }
    return;
  }
  // P blocks: rows TP.. = P (cols < TP), cols TP.. = -P^T (rows < TP), zero corner
  const int rank = t.rank[v];
  const double* P = t.coeff + t.coeff_off[v];
  for (int e = threadIdx.x; e < GT * GT; e += 256) {
    const int r = r0 + e / GT, c = c0 + e % GT;
    if (r >= T || c >= T) continue;
    double val = 0.0;
    if (r >= TP && c < TP) {
      const int i = r - TP;
      val = (i < rank && c < m) ? P[(int64_t)i * m + c] : 0.0;
    } else if (r < TP && c >= TP) {
      const int i = c - TP;
      val = (i < rank && r < m) ? -P[(int64_t)i * m + r] : 0.0;
    }
    A[(int64_t)r * T + c] = val;
  }
  (void)S;
}

void launch_fb_assemble(const DevTree& t, const NodeBatch& fb, const int* begin, const int* size, const double* lam,
                        cudaStream_t st) {
  const int nt = (fb.T + GT - 1) / GT;
  dim3 g(nt, nt, fb.count);
  k_fb_assemble<<<g, 256, 0, st>>>(t, fb, begin, size, lam);
}

// Composed row interchanges of each node's LU: (Pi v)[i] = v[pm[i]], from the
// LAPACK-style swap sequence (linalg.py:250-253). One warp per node.
__global__ void __launch_bounds__(1024) k_compose_perm(NodeBatch nb) {
  pdl_wait();
  const int k = blockIdx.x;
  const int TP = nb.t_pad;
  const int* piv = nb.piv + (int64_t)k * TP;
  int* pm = nb.pm + (int64_t)k * TP;
  extern __shared__ __align__(16) int ps[];
  for (int i = threadIdx.x; i < TP; i += blockDim.x) ps[i] = piv[i];
  __syncthreads();
  // every thread follows one row through the swap sequence: the row that
  // starts at r ends at f(r), so pm[f(r)] = r (same result as swapping pm);
  // t_pad is a multiple of 64, the swaps are read four at a time
  for (int r = threadIdx.x; r < TP; r += blockDim.x) {
    int f = r;
    const int4* p4 = reinterpret_cast<const int4*>(ps);
    for (int i = 0; i < TP / 4; ++i) {
      const int4 q = p4[i];
      const int i0 = 4 * i;
      f = (f == i0) ? q.x : (f == q.x ? i0 : f);
      f = (f == i0 + 1) ? q.y : (f == q.y ? i0 + 1 : f);
      f = (f == i0 + 2) ? q.z : (f == q.z ? i0 + 2 : f);
      f = (f == i0 + 3) ? q.w : (f == q.w ? i0 + 3 : f);
    }
    pm[f] = r;
  }
}

void launch_compose_perm(const NodeBatch& nb, cudaStream_t st) {
  launch_pdl(k_compose_perm, dim3(nb.count), dim3(std::min(1024, nb.t_pad)), sizeof(int) * nb.t_pad, st, nb);
}

// H = sym(trailing block) -> Hbuf[node] (solver.py:163): 32 x 32 tiles, the
// transposed tile through shared memory so both reads run along rows.
__global__ void __launch_bounds__(256) k_extract_h(NodeBatch nb, double* H, int64_t stride) {
  pdl_wait();
  __shared__ double tt[32][33];
  const int k = blockIdx.z;
  const int S = nb.s_pad, T = nb.T, TP = nb.t_pad;
  const double* A = nb.Aug + (int64_t)k * T * T + (int64_t)TP * T + TP;
  double* h = H + (int64_t)nb.node[k] * stride;
  const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 32; r += 8) tt[r][tx] = A[(int64_t)(j0 + r) * T + i0 + tx];  // A[j][i]
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int i = i0 + r, j = j0 + tx;
    h[(int64_t)i * S + j] = 0.5 * (A[(int64_t)i * T + j] + tt[tx][r]);
  }
}

void launch_extract_h(const NodeBatch& nb, double* H, int64_t h_stride, cudaStream_t st) {
  launch_pdl(k_extract_h, dim3(nb.s_pad / 32, nb.s_pad / 32, nb.count), dim3(256), 0, st, nb, H, h_stride);
}

}  // namespace ks

namespace ks {

// ---------------------------------------------------------------------------
// Fused recursive-LU merge for a left block of width H <= 32 (rlu in capi.cu):
//   U12 = L11^-1 A12   (L11 unit lower H x H at (c0, c0), A12 = rows [c0, c0+H),
//                       columns [c0+H, c0+w))
//   A22 -= L21 U12      (rows [c0+H, T), same columns)
// One CTA per (64-column tile, 64-row tile, node): every CTA solves its U12
// tile in shared memory (row tile 0 writes it back), then the DMMA update.
// Replaces a TRSM launch plus a GEMM launch per merge.
// ---------------------------------------------------------------------------
template <int H>
__global__ void __launch_bounds__(128) k_lu_merge(NodeBatch nb, int c0, int w) {
  constexpr int BM = 64, BN = 64;
  constexpr int A_LD = H + 4, B_LD = BN + 4;
  __shared__ double Ls[H][H + 1];
  __shared__ __align__(16) double Us[H][B_LD];
  __shared__ __align__(16) double As[BM][A_LD];
  const int k = blockIdx.z;
  const int T = nb.T;
  double* A = nb.Aug + (int64_t)k * T * T;
  const int n0 = c0 + H + blockIdx.x * BN;  // first column of the tile
  const int m0 = c0 + H + blockIdx.y * BM;  // first row of the A22 tile
  const int ncol = min(BN, c0 + w - n0);
  const int mrow = min(BM, T - m0);
  // L21 tile (rows m0.., cols c0..c0+H) through cp.async
  for (int e = threadIdx.x; e < BM * (H / 2); e += 128) {
    const int r = e / (H / 2), cc = (e % (H / 2)) * 2;
    const bool ok = r < mrow;
    cp_async16(&As[r][cc], ok ? A + (int64_t)(m0 + r) * T + c0 + cc : A, ok ? 16 : 0);
  }
  cp_async_commit();
  for (int e = threadIdx.x; e < H * H; e += 128) Ls[e / H][e % H] = A[(int64_t)(c0 + e / H) * T + c0 + e % H];
  for (int e = threadIdx.x; e < H * BN; e += 128) {
    const int i = e / BN, j = e % BN;
    Us[i][j] = (j < ncol) ? A[(int64_t)(c0 + i) * T + n0 + j] : 0.0;
  }
  __syncthreads();
  if (threadIdx.x < BN) {  // forward substitution, one column per thread
    const int j = threadIdx.x;
    for (int i = 1; i < H; ++i) {
      double s0 = 0.0, s1 = 0.0;
      int kk = 0;
      for (; kk + 1 < i; kk += 2) {
        s0 = fma(Ls[i][kk], Us[kk][j], s0);
        s1 = fma(Ls[i][kk + 1], Us[kk + 1][j], s1);
      }
      if (kk < i) s0 = fma(Ls[i][kk], Us[kk][j], s0);
      Us[i][j] -= s0 + s1;
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  // U12 cannot overwrite A12 here (other row tiles may still read A12): it goes
  // to the node's scratch and the next panel kernel of this node copies it in
  if (blockIdx.y == 0) {
    double* sc = nb.scratch + (int64_t)k * 32 * 64;
    for (int e = threadIdx.x; e < H * BN; e += 128) {
      const int i = e / BN, j = e % BN;
      if (j < ncol) sc[i * 64 + blockIdx.x * BN + j] = Us[i][j];
    }
  }
  if (mrow <= 0) return;
  // DMMA: 4 warps as 2 x 2, warp tile 32 x 32
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm0 = (warp >> 1) * 32, wn0 = (warp & 1) * 32;
  const int gq = lane >> 2, tq = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int kk = 0; kk < H; kk += 4) {
    double af[4], bf[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) af[i] = As[wm0 + i * 8 + gq][kk + tq];
#pragma unroll
    for (int j = 0; j < 4; ++j) bf[j] = Us[kk + tq][wn0 + j * 8 + gq];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = wm0 + i * 8 + gq;
    if (r >= mrow) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = wn0 + j * 8 + 2 * tq;
      if (c >= ncol) continue;
      double2* p = reinterpret_cast<double2*>(A + (int64_t)(m0 + r) * T + n0 + c);
      double2 v = *p;
      v.x -= acc[i][j][0];
      v.y -= acc[i][j][1];
      *p = v;
    }
  }
}

void launch_lu_merge(const NodeBatch& nb, int c0, int h, int w, cudaStream_t st) {
  dim3 g((w - h + 63) / 64, (nb.T - c0 - h + 63) / 64, nb.count);
  if (h == 16) k_lu_merge<16><<<g, 128, 0, st>>>(nb, c0, w);
  else k_lu_merge<32><<<g, 128, 0, st>>>(nb, c0, w);
}

}  // namespace ks

// ---------------------------------------------------------------------------
// Probe (tools/panel_probe.py): one LU panel (columns [0, w)) on `count`
// random nodes of order T (pivot rows < tp), timed per launch with events;
// clk receives CTA 0's clock64 stamps of the last launch (25 entries).
// ---------------------------------------------------------------------------
#include "../../include/invaskit_probe.h"

extern "C" int ks_probe_panel(int T, int tp, int w, int count, int reps, double* ms, long long* clk) {
  using namespace ks;
  const size_t nA = (size_t)count * T * T;
  std::vector<double> h(nA);
  uint64_t st = 88172645463325252ull;
  for (auto& x : h) {
    st ^= st << 13; st ^= st >> 7; st ^= st << 17;
    x = (double)(st >> 11) * (1.0 / 9007199254740992.0) - 0.5;
  }
  double *A = nullptr, *A0 = nullptr, *scratch = nullptr, *norm1 = nullptr, *cond = nullptr;
  int *piv = nullptr, *info = nullptr, *moves = nullptr, *pm = nullptr;
  long long* dclk = nullptr;
  cudaMalloc(&A, nA * 8); cudaMalloc(&A0, nA * 8);
  cudaMalloc(&scratch, (size_t)count * 32 * 64 * 8);
  cudaMalloc(&piv, (size_t)count * tp * 4); cudaMalloc(&info, count * 4);
  cudaMalloc(&moves, (size_t)count * 129 * 4); cudaMalloc(&pm, (size_t)count * tp * 4);
  cudaMalloc(&norm1, count * 8); cudaMalloc(&cond, count * 8);
  cudaMalloc(&dclk, 64 * 8);
  cudaMemcpy(A0, h.data(), nA * 8, cudaMemcpyHostToDevice);
  cudaMemset(info, 0, count * 4);
  cudaMemset(dclk, 0, 64 * 8);
  NodeBatch nb{};
  nb.count = count; nb.first = 0; nb.s_pad = T - tp; nb.t_pad = tp; nb.T = T;
  nb.Aug = A; nb.piv = piv; nb.info = info; nb.moves = moves; nb.pm = pm; nb.scratch = scratch;
  nb.norm1 = norm1; nb.cond = cond;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  std::vector<float> t;
  for (int r = 0; r < reps; ++r) {
    cudaMemcpy(A, A0, nA * 8, cudaMemcpyDeviceToDevice);
    long long* p = (r == reps - 1) ? dclk : nullptr;
    cudaMemcpyToSymbol(g_panel_clk, &p, sizeof(p));
    cudaDeviceSynchronize();
    cudaEventRecord(e0, 0);
    launch_lu_panel(nb, 0, w, 0, nullptr);
    cudaEventRecord(e1, 0);
    cudaEventSynchronize(e1);
    float x = 0.f;
    cudaEventElapsedTime(&x, e0, e1);
    t.push_back(x);
  }
  long long* z = nullptr;
  cudaMemcpyToSymbol(g_panel_clk, &z, sizeof(z));
  cudaError_t err = cudaDeviceSynchronize();
  std::sort(t.begin(), t.end());
  ms[0] = t[0]; ms[1] = t[t.size() / 2];
  cudaMemcpy(clk, dclk, 64 * 8, cudaMemcpyDeviceToHost);
  cudaFree(A); cudaFree(A0); cudaFree(scratch); cudaFree(piv); cudaFree(info); cudaFree(moves); cudaFree(pm);
  cudaFree(norm1); cudaFree(cond); cudaFree(dclk);
  cudaEventDestroy(e0); cudaEventDestroy(e1);
  return err == cudaSuccess ? 0 : 5;
}
