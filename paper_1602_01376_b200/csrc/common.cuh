// Shared device helpers for libinvaskit (sm_100a only).
#pragma once

#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

#include <cuda_runtime.h>
#include <stdint.h>

#if defined(__CUDA_ARCH__) && !defined(__CUDA_ARCH_FEAT_SM100_ALL)
#error "libinvaskit is built for sm_100a only (-gencode arch=compute_100a,code=sm_100a)"
#endif

namespace ks {

constexpr int kWarp = 32;

// Raise a kernel's dynamic shared-memory ceiling to at least `bytes` on the
// current device. Cached per (device, kernel) -- the attribute is per device,
// and the call is not free -- and thread-safe (solves may run concurrently).
inline cudaError_t ensure_smem(const void* kern, size_t bytes, int carveout = -1) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> seen;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  auto it = seen.find({dev, kern});
  if (it != seen.end() && bytes <= it->second) return cudaSuccess;
  if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes)) != cudaSuccess)
    return e;
  if (carveout >= 0 && it == seen.end()) cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
  seen[{dev, kern}] = bytes;
  return cudaSuccess;
}
template <typename K>
inline cudaError_t ensure_smem(K* kern, size_t bytes, int carveout = -1) {
  return ensure_smem(reinterpret_cast<const void*>(kern), bytes, carveout);
}

// fp64 tensor-core MMA: D(8x8) += A(8x4, row) * B(4x8, col). On sm_100a this is
// DMMA.8x8x4 in SASS (the m16n8k{4,8,16} forms lower to sequences of it).
// Fragment layout, g = lane>>2, t = lane&3:
//   a = A[g][t]   b = B[t][g]   d0 = D[g][2t]   d1 = D[g][2t+1]
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 16-byte async global->shared copy; src_bytes == 0 zero-fills the destination.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// exp(x) for x <= 0 (the Gaussian kernel's argument, kernels.py:107-111) on
// the FMA pipe only: x = k ln2 + r (Cody-Waite, k = rint(x log2 e) by the
// 1.5*2^52 shift), exp(r) by its degree-13 Taylor polynomial (|r| <= ln2/2:
// truncation < 5e-18 relative), times 2^k through the exponent bits (two steps
// below 2^-1022, so subnormal results round once). Within ~1 ulp of exp().
// Taylor coefficients 1/n!, n = 13..2, as constant-bank operands of the DFMAs
static __constant__ double kExpTaylor[12] = {1.6059043836821613e-10, 2.08767569878681e-09, 2.505210838544172e-08,
                                             2.755731922398589e-07,  2.7557319223985893e-06, 2.48015873015873e-05,
                                             1.984126984126984e-04,  1.388888888888889e-03,  8.333333333333333e-03,
                                             4.1666666666666664e-02, 1.6666666666666666e-01, 0.5};
// cf: the Taylor coefficients held in registers by a caller that evaluates
// many exponentials (no constant reloads per call)
__device__ __forceinline__ double exp_neg(double x, const double (&cf)[12]) {
  if (!(x > -745.2)) return x < 0.0 ? 0.0 : x;  // underflow (NaN passes through)
  const double shift = 6755399441055744.0;
  const double kd = fma(x, 1.4426950408889634, shift);
  const double k = kd - shift;
  const int ki = __double2loint(kd);
  double r = fma(k, -6.93147180559945286227e-01, x);
  r = fma(k, -2.31904681384629955842e-17, r);
  double p = cf[0];
#pragma unroll
  for (int n = 1; n < 12; ++n) p = fma(p, r, cf[n]);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  if (ki >= -1022) return p * __hiloint2double((ki + 1023) << 20, 0);
  return p * __hiloint2double((ki + 1623) << 20, 0) * 2.4099198651028841e-181;  // 2^(k+600) * 2^-600
}
__device__ __forceinline__ void exp_coeffs(double (&cf)[12]) {
#pragma unroll
  for (int n = 0; n < 12; ++n) cf[n] = kExpTaylor[n];
}
__device__ __forceinline__ double exp_neg(double x) {
  double cf[12];
  exp_coeffs(cf);
  return exp_neg(x, cf);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Batched operand addressing: matrix b of a batch lives at base + idx[b] * stride
// (idx == nullptr means idx[b] = b).
struct Operand {
  const double* ptr;
  int64_t ld;
  int64_t stride;
  const int* idx;
  __device__ __forceinline__ const double* at(int b) const {
    return ptr + (idx ? (int64_t)idx[b] : (int64_t)b) * stride;
  }
};
struct OperandW {
  double* ptr;
  int64_t ld;
  int64_t stride;
  const int* idx;
  __device__ __forceinline__ double* at(int b) const {
    return ptr + (idx ? (int64_t)idx[b] : (int64_t)b) * stride;
  }
};


// Programmatic dependent launch: kernels of the factorization's dependent chain
// start with pdl_wait() (a no-op unless launched with the PDL attribute) and are
// launched through launch_pdl, so the next kernel's launch and CTA setup
// overlap the tail of the previous one. KS_PDL=0 turns the attribute off.
__device__ __forceinline__ void pdl_wait() {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 900)
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

inline bool pdl_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("KS_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

}  // namespace ks
