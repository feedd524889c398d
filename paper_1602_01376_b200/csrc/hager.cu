// Hager 1-norm condition estimate of Z (cond1_estimate, linalg.py:282-304;
// threshold solver.py:150-152) on the block factors of the node step
// (node_kernels.cu): Z = [[I, X], [Y, I]] = [[I, 0], [Y, I]] [[I, X], [0, S]],
// S = Pi^T L U. The estimator's solves become
//
//   y = Z^-1 x :   v2 = x2 - Y x1;  y2 = U^-1 L^-1 Pi v2;  y1 = x1 - X y2
//   z = Z^-T w :   a2 = Pi^T L^-T U^-T (w2 - X^T w1);  z2 = a2;  z1 = w1 - Y^T a2
//
// with the reference's iteration (5 steps, the same break rule and argmax
// first-occurrence tie rule, in the reference's index order: the left child's
// skeleton entries, then the right child's). One CTA per node (persistent over
// the batch); thread i owns entry i of both halves of every vector. The
// triangular solves (size s_pad, half of Z's order) walk 8-row blocks with the
// next block's coefficients loaded one step ahead and the diagonal blocks
// applied through their inverses (k_diag_inv); the X / Y products are
// coalesced GEMVs (warp per row, or thread per column).
#include <cstdlib>
#include <algorithm>

#include "kernels.cuh"
#include "trsv.cuh"

namespace ks {

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


// out[r] = sum_j M[r][j] xin[j] for r < n (M row-major, ld n, n % 64 == 0):
// a warp per 4 rows, 16-byte loads along the rows; every load of a row group
// is issued before the first FMA (up to 16 in flight per lane: the GEMV is
// bound by the loads a single CTA keeps in flight, not by bandwidth)
template <int NT>
__device__ __forceinline__ void gemv_rows_smem(const double* __restrict__ M, int n, const double* xin, double* out) {
  constexpr int NW = NT / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int segs = n >> 6;  // 64-column segments: one double2 per lane each
  for (int r0 = warp * 4; r0 < n; r0 += NW * 4) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int sg0 = 0; sg0 < segs; sg0 += 4) {
      double2 a[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int g = 0; g < 4; ++g)
          a[u][g] = (sg0 + g < segs) ? ldg2(M + (int64_t)(r0 + u) * n + (sg0 + g) * 64 + 2 * lane)
                                     : make_double2(0.0, 0.0);
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        if (sg0 + g < segs) {
          const int c = (sg0 + g) * 64 + 2 * lane;
          const double x0 = xin[c], x1 = xin[c + 1];
#pragma unroll
          for (int u = 0; u < 4; ++u) acc[u] = fma(a[u][g].x, x0, fma(a[u][g].y, x1, acc[u]));
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double v = warp_sum(acc[u]);
      if (lane == 0) out[r0 + u] = v;
    }
  }
}

// sum_r M[r][i] xin[r] for this thread's column i < n (coalesced across
// threads), 16 loads in flight per thread
__device__ __forceinline__ double gemv_col_own(const double* __restrict__ M, int n, const double* xin, int i) {
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  if (i < n) {
    const double* p = M + i;
    for (int r = 0; r < n; r += 16) {
      double a[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) a[u] = __ldg(p + (int64_t)(r + u) * n);
#pragma unroll
      for (int u = 0; u < 16; ++u) acc[u & 3] = fma(a[u], xin[r + u], acc[u & 3]);
    }
  }
  return (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

// nb: the LU view (t_pad = s_pad = S, T = 2 S); dinv: the diagonal-block
// inverses of L and U of S; lut (COLMAJ): column-major copies of S's factors.
template <int NT, bool COLMAJ>
__global__ void __launch_bounds__(NT, 1) k_hager_blk(DevTree t, NodeBatch nb, const double* dinv, const double* lut) {
  constexpr int SBk = 8;
  extern __shared__ __align__(16) double hs[];
  const int S = nb.s_pad, T = nb.T;
  double* dL = hs;                 // S x 8
  double* dU = dL + S * SBk;       // S x 8
  double* xs = dU + S * SBk;       // S: the solves' broadcast buffer
  double* xa = xs + S;             // S: GEMV operand
  double* rb = xa + S;             // S: GEMV result
  double* red = rb + S;            // NT / 32
  int* redi = reinterpret_cast<int*>(red + NT / 32);
  int* pm = redi + NT / 32;        // S: composed swaps of S's LU, (Pi v)[i] = v[pm[i]]
  double* cb = reinterpret_cast<double*>(pm + S + (S & 1));  // 2 x NT x 10 staged coefficients
  const int i = threadIdx.x;
  const bool own = i < S;
  for (int k = blockIdx.x; k < nb.count; k += gridDim.x) {
    __syncthreads();
    const int sl = t.rank[nb.left[k]], sr = t.rank[nb.right[k]];
    const int n = sl + sr;
    if (n == 0) {
      if (threadIdx.x == 0) nb.cond[k] = 0.0;
      continue;
    }
    const double* A = nb.Aug + (int64_t)k * T * T;
    const double* X = nb.XY + (int64_t)k * 2 * S * S;
    const double* Y = X + (int64_t)S * S;
    {
      const double2* src = reinterpret_cast<const double2*>(dinv + (int64_t)(nb.first + k) * 2 * S * SBk);
      double2* dst = reinterpret_cast<double2*>(hs);
      for (int e = threadIdx.x; e < S * SBk; e += NT) dst[e] = src[e];
      for (int e = threadIdx.x; e < S; e += NT) pm[e] = nb.pm[(int64_t)k * S + e];
    }
    const bool r1 = own && i < sl, r2 = own && i < sr;  // real entries of the two halves
    double x1 = r1 ? 1.0 / n : 0.0, x2 = r2 ? 1.0 / n : 0.0;
    double est = 0.0;
    __syncthreads();
    for (int it = 0; it < 5; ++it) {
      // ---- y = Z^-1 x (dense_solve)
      if (own) xa[i] = x1;
      __syncthreads();
      gemv_rows_smem<NT>(Y, S, xa, rb);
      __syncthreads();
      const double v2 = own ? x2 - rb[i] : 0.0;
      if (own) xs[i] = v2;
      __syncthreads();
      double y2 = own ? xs[pm[i]] : 0.0;
      if constexpr (COLMAJ) {
        const double* At = lut + (int64_t)(nb.first + k) * S * S;
        y2 = own_solve<SBk, NT, SOLVE_L, true>(At, S, S, dL, y2, xs);
        y2 = own_solve<SBk, NT, SOLVE_U, true>(At, S, S, dU, y2, xs);
      } else if constexpr (NT <= 512) {  // staged row segments (cb), see own_solve_rows
        y2 = own_solve_rows<NT, SOLVE_L>(A, T, S, dL, y2, xs, cb);
        y2 = own_solve_rows<NT, SOLVE_U>(A, T, S, dU, y2, xs, cb);
      } else {
        y2 = own_solve<SBk, NT, SOLVE_L>(A, T, S, dL, y2, xs);
        y2 = own_solve<SBk, NT, SOLVE_U>(A, T, S, dU, y2, xs);
      }
      __syncthreads();
      if (own) xa[i] = y2;
      __syncthreads();
      gemv_rows_smem<NT>(X, S, xa, rb);
      __syncthreads();
      const double y1 = own ? x1 - rb[i] : 0.0;
      est = nt_sum<NT>((r1 ? fabs(y1) : 0.0) + (r2 ? fabs(y2) : 0.0), red);
      // ---- z = Z^-T sign(y) (solve_transposed)
      const double w1 = r1 ? (y1 >= 0.0 ? 1.0 : -1.0) : 0.0;
      const double w2 = r2 ? (y2 >= 0.0 ? 1.0 : -1.0) : 0.0;
      if (own) xa[i] = w1;
      __syncthreads();
      double a2 = own ? w2 - gemv_col_own(X, S, xa, i) : 0.0;
      a2 = own_solve<SBk, NT, SOLVE_UT>(A, T, S, dU, a2, xs);
      a2 = own_solve<SBk, NT, SOLVE_LT>(A, T, S, dL, a2, xs);
      __syncthreads();
      if (own) xs[pm[i]] = a2;
      __syncthreads();
      const double z2 = own ? xs[i] : 0.0;
      if (own) xa[i] = z2;
      __syncthreads();
      const double z1 = own ? w1 - gemv_col_own(Y, S, xa, i) : 0.0;
      // ---- j = argmax |z| (first in reference order on ties), z . x
      double bv = -1.0;
      int bi = 0x7fffffff;
      if (r1) { bv = fabs(z1); bi = i; }
      if (r2 && fabs(z2) > bv) { bv = fabs(z2); bi = sl + i; }
      nt_argmax<NT>(bv, bi, red, redi);
      const double dot = nt_sum<NT>((r1 ? z1 * x1 : 0.0) + (r2 ? z2 * x2 : 0.0), red);
      if (bv <= dot) break;
      x1 = (r1 && bi == i) ? 1.0 : 0.0;
      x2 = (r2 && bi == sl + i) ? 1.0 : 0.0;
    }
    if (threadIdx.x == 0) nb.cond[k] = isfinite(est) ? nb.norm1[k] * est : INFINITY;
  }
}

void launch_diag_inv(const NodeBatch& nb, double* dinv, cudaStream_t st) {
  k_diag_inv<8><<<dim3(nb.count, 2), 256, 0, st>>>(nb, dinv);
}

template <int NT, bool COLMAJ>
static void launch_hager_blk(const DevTree& t, const NodeBatch& nb, double* dinv, double* lut, int max_ctas,
                             cudaStream_t st) {
  const int S = nb.s_pad;
  launch_diag_inv(nb, dinv, st);
  if (COLMAJ) k_lu_transpose<<<dim3(S / 32, S / 32, nb.count), 256, 0, st>>>(nb, lut);
  size_t smem = sizeof(double) * (2 * (size_t)S * 8 + 3 * (size_t)S + NT / 32) + sizeof(int) * (NT / 32 + S + (S & 1));
  if (NT <= 512) smem = (smem + 15) / 16 * 16 + sizeof(double) * 2 * NT * 10;
  ensure_smem(k_hager_blk<NT, COLMAJ>, smem);
  k_hager_blk<NT, COLMAJ><<<std::min(nb.count, max_ctas), NT, smem, st>>>(t, nb, dinv, lut);
}

int hager_launches(const NodeBatch& nb) { return (nb.t_pad <= 512 && nb.count < 64) ? 3 : 2; }

// nb.t_pad = s_pad <= 1024. The column-major copy pays for itself where the
// factors are still in L2 (narrow levels); for wide levels the extra HBM pass
// costs more than it saves.
void launch_hager(const DevTree& t, const NodeBatch& nb, double* dinv, double* lut, int max_ctas, cudaStream_t st) {
  const int abl = std::getenv("KS_ABLATE") ? std::atoi(std::getenv("KS_ABLATE")) : 0;  // timing experiment (tools/ablate.py)
  if (abl & 256) return;
  const int S = nb.t_pad;
  const bool cm = lut && nb.count < 64 && S <= 512;
  if (S <= 256) {
    if (cm) launch_hager_blk<256, true>(t, nb, dinv, lut, max_ctas, st);
    else launch_hager_blk<256, false>(t, nb, dinv, lut, max_ctas, st);
  } else if (S <= 512) {
    if (cm) launch_hager_blk<512, true>(t, nb, dinv, lut, max_ctas, st);
    else launch_hager_blk<512, false>(t, nb, dinv, lut, max_ctas, st);
  } else {
    launch_hager_blk<1024, false>(t, nb, dinv, nullptr, max_ctas, st);
  }
}

}  // namespace ks
