// CTA-level (256 threads) blocked triangular solves and GEMVs on matrices in
// global memory with vectors in shared memory; used by the solve kernels and
// by the Hager condition estimator. Rows of A are contiguous (ld = lda, even).
//
// These loops stream factor rows from HBM once per pass, so they are written
// for memory-level parallelism: 16-byte loads, several independent loads per
// lane in flight, and the next diagonal block fetched into registers while the
// off-diagonal GEMV of the current block runs.
#pragma once

#include "common.cuh"

namespace ks {

constexpr int SB = 32;       // diagonal block of the blocked triangular solves
constexpr int STHREADS = 256;
constexpr int SWARPS = STHREADS / 32;

__device__ __forceinline__ double2 ldg2(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }

// acc[i][q] += sum_{c in [cb, ce)} A[rb+i][c] x[c][q], i < 4, for one warp.
// [cb, ce) is a multiple of 32 wide and starts even; partial sums per lane.
template <int QC>
__device__ __forceinline__ void warp_rows4(const double* __restrict__ A, int64_t lda, int rb, int nrows, int cb,
                                           int ce, const double* x, double (&acc)[4][QC]) {
  const int lane = threadIdx.x & 31;
  int c = cb + 2 * lane;
  for (; c + 64 < ce; c += 128) {  // two 64-column strips per iteration: 8 loads in flight
    double2 a0[4], a1[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool ok = rb + i < nrows;
      a0[i] = ok ? ldg2(A + (int64_t)(rb + i) * lda + c) : make_double2(0.0, 0.0);
      a1[i] = ok ? ldg2(A + (int64_t)(rb + i) * lda + c + 64) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int q = 0; q < QC; ++q) {
      const double x0 = x[c * QC + q], x1 = x[(c + 1) * QC + q];
      const double x2 = x[(c + 64) * QC + q], x3 = x[(c + 65) * QC + q];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[i][q] = fma(a0[i].x, x0, acc[i][q]);
        acc[i][q] = fma(a0[i].y, x1, acc[i][q]);
        acc[i][q] = fma(a1[i].x, x2, acc[i][q]);
        acc[i][q] = fma(a1[i].y, x3, acc[i][q]);
      }
    }
  }
  for (; c < ce; c += 64) {
    double2 a0[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
      a0[i] = (rb + i < nrows) ? ldg2(A + (int64_t)(rb + i) * lda + c) : make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < QC; ++q) {
      const double x0 = x[c * QC + q], x1 = x[(c + 1) * QC + q];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[i][q] = fma(a0[i].x, x0, acc[i][q]);
        acc[i][q] = fma(a0[i].y, x1, acc[i][q]);
      }
    }
  }
}

// Row-oriented blocked triangular solve, in place on the shared vector x (n x QC):
// lower (ascending blocks) or upper (descending), unit or not. n is a multiple of SB.
template <int QC, bool UPPER, bool UNIT>
__device__ void cta_trsv_rows(const double* __restrict__ A, int64_t lda, int n, double* x, double (*D)[SB + 1]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = n / SB;
  for (int s = 0; s < nb; ++s) {
    const int bi = UPPER ? nb - 1 - s : s;
    const int r0 = bi * SB;
    const int cb = UPPER ? r0 + SB : 0, ce = UPPER ? n : r0;
    // diagonal block: issue its loads first, store after the GEMV
    double dreg[SB * SB / STHREADS];
#pragma unroll
    for (int u = 0; u < SB * SB / STHREADS; ++u) {
      const int e = threadIdx.x + u * STHREADS;
      dreg[u] = A[(int64_t)(r0 + e / SB) * lda + r0 + e % SB];
    }
    {
      double acc[4][QC];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < QC; ++q) acc[i][q] = 0.0;
      const int rb = r0 + warp * 4;
      warp_rows4<QC>(A, lda, rb, n, cb, ce, x, acc);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < QC; ++q) {
          const double v = warp_sum(acc[i][q]);
          if (lane == 0) x[(rb + i) * QC + q] -= v;
        }
    }
#pragma unroll
    for (int u = 0; u < SB * SB / STHREADS; ++u) {
      const int e = threadIdx.x + u * STHREADS;
      D[e / SB][e % SB] = dreg[u];
    }
    __syncthreads();
    // one warp: column-oriented substitution, lane r owns row r0+r
    if (warp == 0) {
      double v[QC];
#pragma unroll
      for (int q = 0; q < QC; ++q) v[q] = x[(r0 + lane) * QC + q];
      const double rd = UNIT ? 1.0 : 1.0 / D[lane][lane];  // (multiply in the chain)
#pragma unroll 4
      for (int s2 = 0; s2 < SB; ++s2) {
        const int c = UPPER ? SB - 1 - s2 : s2;
        if (!UNIT && lane == c) {
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
      for (int q = 0; q < QC; ++q) x[(r0 + lane) * QC + q] = v[q];
    }
    __syncthreads();
  }
}

// y[r] (+)= sum_c A[r][c] x[c] for rows [0, nrows): warps over rows, lanes over c.
// ncols is a multiple of 32.
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
    warp_rows4<QC>(A, lda, rb, nrows, 0, ncols, x, acc);
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

// acc[q] += sum_{k in [kb, ke), k = warp (mod SWARPS)} A[k][col] x[k][q]: 8 loads in flight.
template <int QC>
__device__ __forceinline__ void warp_cols(const double* __restrict__ A, int64_t lda, int kb, int ke, int col,
                                          const double* x, double (&acc)[QC]) {
  const int warp = threadIdx.x >> 5;
  int k = kb + warp;
  for (; k + 7 * SWARPS < ke; k += 8 * SWARPS) {
    double a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = __ldg(A + (int64_t)(k + u * SWARPS) * lda + col);
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int q = 0; q < QC; ++q) acc[q] = fma(a[u], x[(k + u * SWARPS) * QC + q], acc[q]);
  }
  for (; k < ke; k += SWARPS) {
    const double a = __ldg(A + (int64_t)k * lda + col);
#pragma unroll
    for (int q = 0; q < QC; ++q) acc[q] = fma(a, x[k * QC + q], acc[q]);
  }
}

// out[c] += sign * sum_r A[r][c] x[r] for columns [0, ncols): lanes over c, warps
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
    if (c < ncols) warp_cols<QC>(A, lda, 0, nrows, c, x, acc);
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
    double dreg[SB * SB / STHREADS];
#pragma unroll
    for (int u = 0; u < SB * SB / STHREADS; ++u) {
      const int e = threadIdx.x + u * STHREADS;
      dreg[u] = A[(int64_t)(r0 + e / SB) * lda + r0 + e % SB];
    }
    {
      double acc[QC];
#pragma unroll
      for (int q = 0; q < QC; ++q) acc[q] = 0.0;
      warp_cols<QC>(A, lda, kb, ke, r0 + lane, x, acc);
#pragma unroll
      for (int q = 0; q < QC; ++q) red[(warp * 32 + lane) * QC + q] = acc[q];
    }
#pragma unroll
    for (int u = 0; u < SB * SB / STHREADS; ++u) {
      const int e = threadIdx.x + u * STHREADS;
      D[e / SB][e % SB] = dreg[u];
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
      const double rd = UNIT ? 1.0 : 1.0 / D[lane][lane];  // (multiply in the chain)
#pragma unroll 4
      for (int s2 = 0; s2 < SB; ++s2) {
        const int c = FORWARD ? s2 : SB - 1 - s2;
        if (!UNIT && lane == c) {
#pragma unroll
          for (int q = 0; q < QC; ++q) v[q] *= rd;
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
