// Tiled Gaussian-kernel block in the reference's difference form
// (kernels.py:107-111): sq[i][j] = sum_d (x_i - y_j)^2 for a 64 x 64 tile,
// coordinates staged through shared memory 32 dimensions at a time.
// 256 threads; thread (ty, tx) owns rows ty + 16 i and columns tx + 16 j.
#pragma once

#include "kernels.cuh"

namespace ks {

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


}  // namespace ks
