// Cost of the LU panel's per-column step, built up piece by piece (cycles per
// column, one CTA of NT threads, one register row of W values per thread).
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1602_01376_b200/csrc/lu_panel.cuh"
using namespace ks;

template <int W, int NT, int CB>
__global__ void __launch_bounds__(NT, 1) k_real(const double* in, double* out, long long* cyc, int ncols, int* piv, int* info) {
  constexpr int NW = NT / 32;
  __shared__ PanelShared<NW, W> ps;
  extern __shared__ double fin[];
  double a[1][W];
  int pos[1];
  bool done[1];
  long long tot = 0;
#pragma unroll 1
  for (int rep = 0; rep < ncols / W; ++rep) {
#pragma unroll
    for (int j = 0; j < W; ++j) a[0][j] = in[threadIdx.x * W + j];
    pos[0] = threadIdx.x;
    done[0] = false;
    __syncthreads();
    long long t0 = clock64();
    panel_columns<W, 1, NT, CB>(a, pos, done, ps, fin, W + 2, NT, piv, 0, info, 0, NT / 32);
    __syncthreads();
    tot += clock64() - t0;
  }
  if (threadIdx.x == 0) cyc[4] = tot;
  out[threadIdx.x] = a[0][0] + fin[threadIdx.x];
}

template <int W, int NT, int MODE>
__global__ void __launch_bounds__(NT, 1) k_col(const double* in, double* out, long long* cyc, int ncols) {
  constexpr int NW = NT / 32;
  __shared__ PanelShared<NW, W> ps;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double a[W];
#pragma unroll
  for (int j = 0; j < W; ++j) a[j] = in[threadIdx.x * W + j];
  int pos = threadIdx.x;
  bool done = false;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int rep = 0; rep < ncols / W; ++rep) {
#pragma unroll
    for (int c = 0; c < W; ++c) {
      const int buf = c & 1;
      const double v = fabs(a[c]);
      const unsigned bh = done ? 0u : (unsigned)__double2hiint(v) + 1u, bl = (unsigned)__double2loint(v);
      double rc = 1.0;
      if (MODE >= 2) rc = 1.0 / a[c];
      const int wl = warp_winner3(bh, bl, pos);
      if (lane == wl) {
        if (MODE >= 3) {
#pragma unroll
          for (int j = c + 1; j < W; ++j) ps.cand[buf][warp][j] = a[j];
        }
        PivRec q; q.hi = bh; q.lo = bl; q.pos = pos; q.pad = 0; q.rcp = rc; q.pad2 = 0.0;
        ps.rec[buf][warp] = q;
      }
      __syncthreads();
      unsigned qh = 0u, ql = 0u; int qp = 0x7fffffff; double qr = 0.0;
      if (lane < NW) { const PivRec& q = ps.rec[buf][lane]; qh = q.hi; ql = q.lo; qp = q.pos; qr = q.rcp; }
      const int ww = warp_winner3(qh, ql, qp);
      const int bpos = __shfl_sync(0xffffffffu, qp, ww);
      const double rcp = __shfl_sync(0xffffffffu, qr, ww);
      if (MODE >= 1) {
        const bool is_piv = !done && pos == bpos;
        done = done || is_piv;
      }
      if (MODE >= 3 && !done) {
        const double l = a[c] * rcp;
        a[c] = l;
#pragma unroll
        for (int j = c + 1; j < W; ++j) a[j] = fma(-l, ps.cand[buf][ww][j], a[j]);
      } else {
        a[(c + 1) % W] += rcp * 1e-300 + (double)bpos * 1e-300;
      }
    }
    done = false;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[MODE] = t1 - t0;
  double s = 0;
#pragma unroll
  for (int j = 0; j < W; ++j) s += a[j];
  out[threadIdx.x] = s;
}

int main() {
  const int NT = 512, W = 16, ncols = 256;
  double *in, *out; long long* cyc;
  cudaMalloc(&in, NT * W * 8); cudaMalloc(&out, NT * 8); cudaMalloc(&cyc, 8 * 8);
  double h[NT * W];
  unsigned s = 1;
  for (auto& x : h) { s = s * 1664525u + 1013904223u; x = (s >> 8) * (1.0 / 16777216.0) - 0.5; }
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  long long c[8];
  for (int r = 0; r < 2; ++r) {
    k_col<W, NT, 0><<<1, NT>>>(in, out, cyc, ncols);
    k_col<W, NT, 1><<<1, NT>>>(in, out, cyc, ncols);
    k_col<W, NT, 2><<<1, NT>>>(in, out, cyc, ncols);
    k_col<W, NT, 3><<<1, NT>>>(in, out, cyc, ncols);
  }
  int *piv, *info;
  cudaMalloc(&piv, 64 * 4); cudaMalloc(&info, 4); cudaMemset(info, 0, 4);
  cudaFuncSetAttribute(k_real<W, NT, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, NT * (W + 2) * 8);
  cudaFuncSetAttribute(k_real<W, NT, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, NT * (W + 2) * 8);
  for (int r = 0; r < 2; ++r) k_real<W, NT, 4><<<1, NT, NT * (W + 2) * 8>>>(in, out, cyc, ncols, piv, info);
  cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  printf("panel_columns CB=4: %.0f cycles/column\n", c[4] / (double)ncols);
  for (int r = 0; r < 2; ++r) k_real<W, NT, 16><<<1, NT, NT * (W + 2) * 8>>>(in, out, cyc, ncols, piv, info);
  cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  printf("panel_columns CB=16: %.0f cycles/column\n", c[4] / (double)ncols);
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  printf("NT=%d W=%d cycles/column: search+BAR %.0f  +done %.0f  +div %.0f  +publish/update %.0f\n", NT, W,
         c[0] / (double)ncols, c[1] / (double)ncols, c[2] / (double)ncols, c[3] / (double)ncols);
  return 0;
}
