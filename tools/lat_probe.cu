// Latency probe: dependent DFMA / DADD / SHFL(double) chains, 512-thread
// barrier round trip, LDS->DFMA->STS->BAR loop (the estimator's block step).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat(double* out, long long* cyc, int n) {
  __shared__ double xs[512];
  double a = out[threadIdx.x], b = 1.0000001, c = 1e-9;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) { a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0);
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) { a = a + c; a = a + c; a = a + c; a = a + c; }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = (t1 - t0);
  // SHFL double chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    a = __shfl_sync(0xffffffffu, a, (threadIdx.x + 1) & 31); a = __shfl_sync(0xffffffffu, a, (threadIdx.x + 3) & 31);
    a = __shfl_sync(0xffffffffu, a, (threadIdx.x + 5) & 31); a = __shfl_sync(0xffffffffu, a, (threadIdx.x + 7) & 31);
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = (t1 - t0);
  // barrier only
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < n; ++i) { __syncthreads(); __syncthreads(); __syncthreads(); __syncthreads(); }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = (t1 - t0);
  // STS -> BAR -> LDS -> DFMA chain (one block step of a broadcast solve)
  xs[threadIdx.x] = a;
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < 4 * n; ++i) {
    const int src = i & 511;
    if (threadIdx.x == (src & 511)) xs[src] = a;
    __syncthreads();
    a = fma(xs[src], b, a);
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = (t1 - t0);
  out[threadIdx.x] = a;
}

int main() {
  double* d; long long* c; long long h[5];
  cudaMalloc(&d, 512 * sizeof(double)); cudaMemset(d, 0, 512 * sizeof(double));
  cudaMalloc(&c, 5 * sizeof(long long));
  const int n = 1000;
  for (int nt : {32, 512}) {
    k_lat<<<1, nt>>>(d, c, n);
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    printf("threads %d: DFMA %.1f  DADD %.1f  SHFL.f64 %.1f  BAR %.1f  STS-BAR-LDS-DFMA %.1f cyc/op\n", nt,
           h[0] / (4.0 * n), h[1] / (4.0 * n), h[2] / (4.0 * n), h[3] / (4.0 * n), h[4] / (4.0 * n));
  }
  return 0;
}
