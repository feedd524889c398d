// Cycles per block step of the condition estimator's triangular solves
#include <cstdio>
// (own_solve in factor_kernels.cu) on one warm 768 x 768 augmented matrix.
#include "../paper_1602_01376_b200/csrc/factor_kernels.cu"

template <int MODE>
__global__ void __launch_bounds__(512, 1) k_probe(const double* A, const double* dinv, long long* cyc, int reps) {
  extern __shared__ __align__(16) double hs[];
  constexpr int SB = 8, NT = 512, TP = 512, T = 768;
  double* dL = hs;
  double* xs = hs + TP * SB;
  for (int e = threadIdx.x; e < TP * SB; e += NT) dL[e] = dinv[e];
  double v = 1.0 / (1 + threadIdx.x);
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) v = ks::own_solve<SB, NT, MODE>(A, T, TP, dL, v, xs) * 1e-3 + 1.0;
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[MODE] = (t1 - t0) / reps;
  if (v == 12345.0) cyc[7] = 1;
}

int main() {
  const int T = 768, TP = 512, SB = 8;
  std::vector<double> h((size_t)T * T), d((size_t)TP * SB);
  for (int i = 0; i < T; ++i)
    for (int j = 0; j < T; ++j) h[(size_t)i * T + j] = (i == j) ? 2.0 : 1e-3 * ((i * 7 + j * 13) % 17 - 8);
  for (size_t e = 0; e < d.size(); ++e) d[e] = ((e / SB) % SB == e % SB) ? 0.5 : 0.0;
  double *A, *D; long long* c;
  cudaMalloc(&A, h.size() * 8); cudaMalloc(&D, d.size() * 8); cudaMalloc(&c, 8 * 8);
  cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(D, d.data(), d.size() * 8, cudaMemcpyHostToDevice);
  const size_t smem = (TP * SB + TP + 64) * 8;
  cudaFuncSetAttribute(k_probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_probe<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  long long hc[8] = {0};
  for (int it = 0; it < 2; ++it) {
    k_probe<0><<<1, 512, smem>>>(A, D, c, 10);
    k_probe<1><<<1, 512, smem>>>(A, D, c, 10);
    k_probe<2><<<1, 512, smem>>>(A, D, c, 10);
    k_probe<3><<<1, 512, smem>>>(A, D, c, 10);
  }
  cudaMemcpy(hc, c, sizeof(hc), cudaMemcpyDeviceToHost);
  printf("err %s; cycles per solve (64 block steps): L %lld  U %lld  UT %lld  LT %lld -> per step %.0f %.0f %.0f %.0f\n",
         cudaGetErrorString(cudaDeviceSynchronize()), hc[0], hc[1], hc[2], hc[3], hc[0] / 64.0, hc[1] / 64.0,
         hc[2] / 64.0, hc[3] / 64.0);
  return 0;
}
