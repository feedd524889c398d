// Microbenchmark: fp64 issue rates on sm_100a (DFMA vs mma.sync f64 shapes).
// Used once to pick the inner-product primitive of the factorization kernels.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void mma884_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void mma1684_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = 0.5, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = i + j;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[0] = s;
}

__global__ void mma1688_kernel(double* out, int iters) {
  double a[4], b0 = 1.0 - threadIdx.x * 1e-4, b1 = 0.25;
  for (int i = 0; i < 4; ++i) a[i] = threadIdx.x * 1e-3 + i;
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = i + j;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b0), "d"(b1));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[0] = s;
}

__global__ void mma16816_kernel(double* out, int iters) {
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - threadIdx.x * 1e-4 * i;
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = i + j;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[0] = s;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  double* out; CK(cudaMalloc(&out, 8));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock %d kHz\n", sms, clk);
  for (int wpb : {4, 8, 16}) {
    int blocks = sms * 4, threads = 32 * wpb, iters = 4096;
    double fl;
    float ms = timeit([&] { dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); });
    fl = 2.0 * 16 * iters * (double)blocks * threads;
    printf("DFMA        wpb=%2d  %.2f TFLOP/s  (%.3f ms)\n", wpb, fl / ms / 1e9, ms);
    ms = timeit([&] { mma884_kernel<<<blocks, threads>>>(out, iters); });
    fl = 2.0 * 8 * 8 * 4 * 8 * (double)iters * blocks * wpb;
    printf("DMMA 8x8x4   wpb=%2d  %.2f TFLOP/s\n", wpb, fl / ms / 1e9);
    ms = timeit([&] { mma1684_kernel<<<blocks, threads>>>(out, iters); });
    fl = 2.0 * 16 * 8 * 4 * 4 * (double)iters * blocks * wpb;
    printf("DMMA 16x8x4  wpb=%2d  %.2f TFLOP/s\n", wpb, fl / ms / 1e9);
    ms = timeit([&] { mma1688_kernel<<<blocks, threads>>>(out, iters); });
    fl = 2.0 * 16 * 8 * 8 * 4 * (double)iters * blocks * wpb;
    printf("DMMA 16x8x8  wpb=%2d  %.2f TFLOP/s\n", wpb, fl / ms / 1e9);
    ms = timeit([&] { mma16816_kernel<<<blocks, threads>>>(out, iters / 2); });
    fl = 2.0 * 16 * 8 * 16 * 4 * (double)(iters / 2) * blocks * wpb;
    printf("DMMA 16x8x16 wpb=%2d  %.2f TFLOP/s\n", wpb, fl / ms / 1e9);
  }
  CK(cudaGetLastError());
  return 0;
}
