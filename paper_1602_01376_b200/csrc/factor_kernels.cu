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
// 64x64 diagonal-block Cholesky + triangular inverse (one CTA per leaf),
// blocked by 16 columns so the critical path is ~20 barriers instead of one
// per column:
//   for each 16-column block kb: warp 0 factors the 16x16 diagonal block in
//   registers (lane i owns row i; per column one broadcast of the pivot, a
//   reciprocal square root and one shuffle per remaining column: _cholesky's
//   column order within the block, linalg.py:185-196, with l_jj = p * rsqrt(p))
//   and inverts it with the stored reciprocals; all threads then form the
//   block's rows below (L21 = A21 L11^-T) and update the trailing lower
//   triangle; finally the off-diagonal blocks of X = L^-1 by block rows.
// Failure (pivot <= 0 or non-finite) records the first bad column + 1, as
// _cholesky raises NotSPDError at linalg.py:190-192 (the block stays finite).
// X lives transposed in the strict upper triangle of the tile (x[i][j] at
// a[j][i], i > j) with its diagonal in xd; the current block's inverse also
// densely in xi (zeros above its diagonal).
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 4) k_potrf64(LeafBatch lb, int j0, double* inv, int* info) {
  pdl_wait();
  const int leaf = blockIdx.x;
  double* A = lb.A + (int64_t)leaf * lb.a_stride + (int64_t)j0 * lb.m_pad + j0;
  const int64_t ld = lb.m_pad;
  extern __shared__ double potrf_sm[];
  double(*a)[65] = reinterpret_cast<double(*)[65]>(potrf_sm);
  double* xd = potrf_sm + 64 * 65;
  double(*t)[17] = reinterpret_cast<double(*)[17]>(xd + 64);  // 48 x 17 scratch
  double(*xi)[17] = reinterpret_cast<double(*)[17]>(xd + 64 + 48 * 17);  // 16 x 17: the block's inverse
  __shared__ int bad;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
  }
  if (threadIdx.x == 0) bad = 0x7fffffff;
  __syncthreads();
#pragma unroll 1
  for (int kb = 0; kb < 64; kb += 16) {
    if (warp == 0) {
      // (1) the 16 x 16 diagonal block: lane i < 16 owns row kb + i (the upper
      // part of r and lanes >= 16 carry unused values: no predication)
      const int row = kb + (lane & 15);
      double r[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) r[k] = a[row][kb + k];
      double rinv = 0.0;  // lane j: 1 / l_jj
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        double p = __shfl_sync(0xffffffffu, r[j], j);
        if (!(p > 0.0) || !isfinite(p)) {  // warp-uniform
          if (lane == 0) atomicMin(&bad, kb + j);
          p = 1.0;
          if (lane == j) r[j] = 1.0;
        }
        const double rl = rsqrt(p);
        const double cj = r[j] * rl;  // lane j: l_jj = p / sqrt(p); lanes > j: column j of L
        r[j] = cj;
        if (lane == j) rinv = rl;
#pragma unroll
        for (int k = j + 1; k < 16; ++k) r[k] = fma(-cj, __shfl_sync(0xffffffffu, cj, k), r[k]);
      }
      if (lane < 16) {
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (k <= lane) a[row][kb + k] = r[k];
        t[0][lane] = rinv;  // scratch row 0: the reciprocal diagonal
      }
      __syncwarp();
      // inverse of the diagonal block: lane c < 16 solves column c of L11 x = e_c
      if (lane < 16) {
        const int c = lane;
        double x[16];
#pragma unroll
        for (int rr = 0; rr < 16; ++rr) {
          double s = (rr == c) ? 1.0 : 0.0;
#pragma unroll
          for (int k = 0; k < rr; ++k) s = fma(-a[kb + rr][kb + k], x[k], s);  // x[k] = 0 for k < c
          x[rr] = s * t[0][rr];
        }
#pragma unroll
        for (int rr = 0; rr < 16; ++rr) {
          xi[rr][c] = x[rr];
          if (rr == c) xd[kb + c] = x[rr];
          else if (rr > c) a[kb + c][kb + rr] = x[rr];
        }
      }
    }
    __syncthreads();
    const int nr = 48 - kb;  // rows below the block
    if (nr > 0) {
      // (2) L21 = A21 L11^-T: t[r][j] = sum_{k <= j} A[kb+16+r][kb+k] X11[j][k]
      for (int e = threadIdx.x; e < nr * 16; e += 256) {
        const int rr = e >> 4, j = e & 15;
        const double* ar = a[kb + 16 + rr] + kb;
        const double* xj = xi[j];
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < 16; ++k) s = fma(ar[k], xj[k], s);  // xj[k] = 0 for k > j
        t[rr][j] = s;
      }
      __syncthreads();
      // (3) trailing lower triangle: a[r][c] -= sum_k L[r][k] L[c][k]; L21 back into a
      for (int e = threadIdx.x; e < nr * nr; e += 256) {
        const int rr = e / nr, cc = e - rr * nr;
        if (cc > rr) continue;
        double s = a[kb + 16 + rr][kb + 16 + cc];
#pragma unroll
        for (int k = 0; k < 16; ++k) s = fma(-t[rr][k], t[cc][k], s);
        a[kb + 16 + rr][kb + 16 + cc] = s;
      }
      for (int e = threadIdx.x; e < nr * 16; e += 256) a[kb + 16 + (e >> 4)][kb + (e & 15)] = t[e >> 4][e & 15];
      __syncthreads();
    }
  }
  // (4) off-diagonal blocks of X = L^-1 by block rows:
  //     X[bi][bj] = -X[bi][bi] sum_{k = bj..bi-1} L[bi][k] X[k][bj]
  //     (X[k][c] for k > c is a[c][k], X[c][c] is xd[c])
#pragma unroll 1
  for (int bi = 1; bi < 4; ++bi) {
    double(*tt)[16] = reinterpret_cast<double(*)[16]>(&t[0][0]);  // bi x 16 x 16 (<= 768 doubles)
    for (int e = threadIdx.x; e < bi * 256; e += 256) {
      const int bj = e >> 8, rl = (e >> 4) & 15, cl = e & 15;
      const int r = bi * 16 + rl, c = bj * 16 + cl;
      const double* lr = a[r];
      const double* xc = a[c];
      double s = lr[c] * xd[c];
      for (int k = c + 1; k < bi * 16; ++k) s = fma(lr[k], xc[k], s);
      tt[bj * 16 + rl][cl] = s;
    }
    __syncthreads();
    double xo[3];
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const int e = threadIdx.x + u * 256;
      xo[u] = 0.0;
      if (e < bi * 256) {
        const int bj = e >> 8, rl = (e >> 4) & 15, cl = e & 15;
        const int r = bi * 16 + rl;
        double s = xd[r] * tt[bj * 16 + rl][cl];
        for (int m = 0; m < rl; ++m) s = fma(a[bi * 16 + m][r], tt[bj * 16 + m][cl], s);
        xo[u] = -s;
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const int e = threadIdx.x + u * 256;
      if (e < bi * 256) {
        const int bj = e >> 8, rl = (e >> 4) & 15, cl = e & 15;
        a[bj * 16 + cl][bi * 16 + rl] = xo[u];  // X[r][c] at a[c][r]
      }
    }
    __syncthreads();
  }
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
  constexpr size_t smem = (64 * 65 + 64 + 48 * 17 + 16 * 17) * sizeof(double);
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

void launch_sym_h(double* H, int64_t h_stride, const int* node_idx, int count, int s_pad, cudaStream_t st) {
  if (count <= 0 || s_pad <= 0) return;
  dim3 g(32, count);
  k_sym_h<<<g, 256, 0, st>>>(H, h_stride, node_idx, s_pad);
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

