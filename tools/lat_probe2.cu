// Latency probe 2: dependent chains of the LU panel's per-column primitives.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat2(double* out, long long* cyc, int n) {
  __shared__ double xs[512 * 4];
  unsigned u = threadIdx.x * 2654435761u;
  double a = out[threadIdx.x] + 1.5, b = 1.0000001;
  long long t0, t1;
  // CREDUX max chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    u = __reduce_max_sync(0xffffffffu, u) ^ threadIdx.x;
    u = __reduce_max_sync(0xffffffffu, u) ^ threadIdx.x;
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  // ballot + popc + ffs chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    unsigned m = __ballot_sync(0xffffffffu, (u >> (threadIdx.x & 7)) & 1);
    u = (unsigned)__popc(m) + (unsigned)__ffs(m) + u;
    m = __ballot_sync(0xffffffffu, (u >> (threadIdx.x & 7)) & 1);
    u = (unsigned)__popc(m) + (unsigned)__ffs(m) + u;
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = t1 - t0;
  // fp64 division chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) { a = b / a; a = b / a; }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = t1 - t0;
  // LDS.64 dependent chain (pointer chase through smem)
  xs[threadIdx.x] = (double)((threadIdx.x + 1) & 511);
  __syncthreads();
  int idx = threadIdx.x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { idx = (int)xs[idx]; idx = (int)xs[idx]; }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = t1 - t0;
  // shfl int chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) { idx = __shfl_sync(0xffffffffu, idx, (threadIdx.x + 1) & 31); idx = __shfl_sync(0xffffffffu, idx, (idx + 3) & 31); }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = t1 - t0;
  // STS + BAR + LDS (winner publish round trip)
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if ((threadIdx.x & 31) == (idx & 31)) xs[threadIdx.x >> 5] = a;
    __syncthreads();
    a = xs[(idx >> 5) & 15] + a;
    idx += 1;
    __syncthreads();
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = t1 - t0;
  out[threadIdx.x] = a + u + idx;
}

int main() {
  double* d; long long* c; long long h[6];
  cudaMalloc(&d, 512 * sizeof(double)); cudaMemset(d, 0, 512 * sizeof(double));
  cudaMalloc(&c, 6 * sizeof(long long));
  const int n = 1000;
  for (int nt : {32, 512}) {
    k_lat2<<<1, nt>>>(d, c, n);
    k_lat2<<<1, nt>>>(d, c, n);
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    printf("threads %d: CREDUX %.1f  BALLOT+POPC+FFS %.1f  DDIV %.1f  LDS-chase %.1f  SHFL.i32 %.1f  STS-BAR-LDS-BAR %.1f cyc/op\n",
           nt, h[0] / (2.0 * n), h[1] / (2.0 * n), h[2] / (2.0 * n), h[3] / (2.0 * n), h[4] / (2.0 * n), h[5] / (1.0 * n));
  }
  return 0;
}
