// CTA-level (256 threads) blocked triangular solves and GEMVs on matrices in
// global memory with vectors in shared memory; used by the solve kernels and
// by the Hager condition estimator. Rows of A are contiguous (ld = lda).
#pragma once

#include "common.cuh"

namespace ks {

constexpr int SB = 32;       // diagonal block of the blocked triangular solves
constexpr int STHREADS = 256;
constexpr int SWARPS = STHREADS / 32;

// Row-oriented blocked triangular solve, in place on the shared vector x (n x QC):
// lower (ascending blocks) or upper (descending), unit or not. Rows of A are
// contiguous (ld = lda); n is a multiple of SB.
template <int QC, bool UPPER, bool UNIT>
__device__ void cta_trsv_rows(const double* __restrict__ A, int64_t lda, int n, double* x, double (*D)[SB + 1]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = n / SB;
  for (int s = 0; s < nb; ++s) {
    const int bi = UPPER ? nb - 1 - s : s;
    const int r0 = bi * SB;
    const int cb = UPPER ? r0 + SB : 0, ce = UPPER ? n : r0;
    // 1) off-diagonal GEMV: 4 rows per warp
    {
      double acc[4][QC];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < QC; ++q) acc[i][q] = 0.0;
      const int rb = r0 + warp * 4;
      for (int c = cb + lane; c < ce; c += 32) {
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
          if (lane == 0) x[(rb + i) * QC + q] -= v;
        }
    }
    // 2) diagonal block to shared memory
    for (int e = threadIdx.x; e < SB * SB; e += STHREADS) {
      const int i = e / SB, j = e % SB;
      D[i][j] = A[(int64_t)(r0 + i) * lda + r0 + j];
    }
    __syncthreads();
    // 3) one warp: column-oriented substitution, lane r owns row r0+r
    if (warp == 0) {
      double v[QC];
#pragma unroll
      for (int q = 0; q < QC; ++q) v[q] = x[(r0 + lane) * QC + q];
#pragma unroll 4
      for (int s2 = 0; s2 < SB; ++s2) {
        const int c = UPPER ? SB - 1 - s2 : s2;
        if (!UNIT && lane == c) {
#pragma unroll
          for (int q = 0; q < QC; ++q) v[q] /= D[c][c];
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
      for (int q = 0; q < QC; ++q) x[(r0 + lane) * QC + q] = v[q];
    }
    __syncthreads();
  }
}

// y[r] = sum_c A[r][c] x[c] for rows [0, nrows): warps over rows, lanes over c.
template <int QC>
__device__ void cta_gemv_rows(const double* __restrict__ A, int64_t lda, int nrows, int ncols, const double* x,
                              double* out, int64_t ldo, bool accumulate) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int rb = warp * 4; rb < nrows; rb += SWARPS * 4) {
    double acc[4][QC];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int q = 0; q < QC; ++q) acc[i][q] = 0.0;
    for (int c = lane; c < ncols; c += 32) {
      double a[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = (rb + i < nrows) ? __ldg(A + (int64_t)(rb + i) * lda + c) : 0.0;
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
        if (lane == 0 && rb + i < nrows) {
          double* o = out + (int64_t)(rb + i) * ldo + q;
          *o = accumulate ? *o + v : v;
        }
      }
  }
}

// out[c] (+)= sum_r A[r][c] x[r] for columns [0, ncols): lanes over c, warps
// over r, cross-warp reduction in shared memory. red: SWARPS x 32 x QC.
template <int QC>
__device__ void cta_gemv_cols(const double* __restrict__ A, int64_t lda, int nrows, int ncols, const double* x,
                              double* out, double sign, double* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c0 = 0; c0 < ncols; c0 += 32) {
    const int c = c0 + lane;
    double acc[QC];
#pragma unroll
    for (int q = 0; q < QC; ++q) acc[q] = 0.0;
    if (c < ncols) {
      for (int r = warp; r < nrows; r += SWARPS) {
        const double a = __ldg(A + (int64_t)r * lda + c);
#pragma unroll
        for (int q = 0; q < QC; ++q) acc[q] = fma(a, x[r * QC + q], acc[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < QC; ++q) red[(warp * 32 + lane) * QC + q] = acc[q];
    __syncthreads();
    if (warp == 0 && c < ncols) {
#pragma unroll
      for (int q = 0; q < QC; ++q) {
        double s = 0.0;
        for (int w = 0; w < SWARPS; ++w) s += red[(w * 32 + lane) * QC + q];
        out[c * QC + q] += sign * s;
      }
    }
    __syncthreads();
  }
}


// Transposed blocked triangular solve op(A)^T x = b, in place on x (n x QC):
// FORWARD: A upper, A^T lower, blocks ascending (U^T w = b, linalg.py:257);
// !FORWARD: A lower, A^T upper, blocks descending (L^T x = b, linalg.py:235-243,
// :258). The off-diagonal part reads 32-wide row segments of A (coalesced) and
// reduces across warps in shared memory. red: SWARPS x 32 x QC.
template <int QC, bool FORWARD, bool UNIT>
__device__ void cta_trsv_trans(const double* __restrict__ A, int64_t lda, int n, double* x, double (*D)[SB + 1],
                               double* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = n / SB;
  for (int s = 0; s < nb; ++s) {
    const int bi = FORWARD ? s : nb - 1 - s;
    const int r0 = bi * SB;
    const int kb = FORWARD ? 0 : r0 + SB, ke = FORWARD ? r0 : n;
    {
      double acc[QC];
#pragma unroll
      for (int q = 0; q < QC; ++q) acc[q] = 0.0;
      for (int k = kb + warp; k < ke; k += SWARPS) {
        const double a = __ldg(A + (int64_t)k * lda + r0 + lane);
#pragma unroll
        for (int q = 0; q < QC; ++q) acc[q] = fma(a, x[k * QC + q], acc[q]);
      }
#pragma unroll
      for (int q = 0; q < QC; ++q) red[(warp * 32 + lane) * QC + q] = acc[q];
    }
    for (int e = threadIdx.x; e < SB * SB; e += STHREADS) {
      const int i = e / SB, j = e % SB;
      D[i][j] = A[(int64_t)(r0 + i) * lda + r0 + j];
    }
    __syncthreads();
    if (warp == 0) {
      double v[QC];
#pragma unroll
      for (int q = 0; q < QC; ++q) {
        double sum = 0.0;
        for (int w = 0; w < SWARPS; ++w) sum += red[(w * 32 + lane) * QC + q];
        v[q] = x[(r0 + lane) * QC + q] - sum;
      }
#pragma unroll 4
      for (int s2 = 0; s2 < SB; ++s2) {
        const int c = FORWARD ? s2 : SB - 1 - s2;
        if (!UNIT && lane == c) {
#pragma unroll
          for (int q = 0; q < QC; ++q) v[q] /= D[c][c];
        }
        const double dl = D[c][lane];  // (A^T)[lane][c] = A[c][lane]
        const bool upd = FORWARD ? (lane > c) : (lane < c);
#pragma unroll
        for (int q = 0; q < QC; ++q) {
          const double xc = __shfl_sync(0xffffffffu, v[q], c);
          if (upd) v[q] = fma(-dl, xc, v[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < QC; ++q) x[(r0 + lane) * QC + q] = v[q];
    }
    __syncthreads();
  }
}

}  // namespace ks
