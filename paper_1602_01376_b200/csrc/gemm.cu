// Tile-shape selection and instantiation of the batched DMMA GEMM.
#include <cudaTypedefs.h>

#include <cstdlib>

#include "gemm.cuh"

namespace ks {

namespace {

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

bool tma_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("KS_TMA");
    return !(e && e[0] == '0');
  }();
  return on;
}

// 3-D map (cols, rows, batch) of a row-major operand: boxes of box_cols x
// box_rows. cols = K with 16-wide boxes and the 128-byte swizzle (gemm.cuh
// swz128) for A and B^T; cols = N with 8-wide unswizzled boxes for B.
bool encode_operand(CUtensorMap* m, const Operand& o, int rows, int cols, int batch, int box_cols, int box_rows,
                    bool swizzle) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = tmap_encoder();
  if (!enc || o.idx || !o.ptr) return false;
  if ((reinterpret_cast<uintptr_t>(o.ptr) & 15) || (o.ld & 1) || o.ld < cols) return false;
  int64_t bstride = o.stride;
  if (batch == 1 && bstride == 0) bstride = o.ld * rows;
  if (bstride <= 0 || (bstride & 1)) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)batch};
  const cuuint64_t strides[2] = {(cuuint64_t)o.ld * 8, (cuuint64_t)bstride * 8};
  const cuuint32_t box[3] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(o.ptr), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BM, int BN, int WM, int WN, bool TA, bool TB, int STAGES, int EPI = 0>
cudaError_t launch(const GemmArgs& g0, cudaStream_t st) {
  using Cfg = GemmCfg<BM, BN, WM, WN, TA, TB, STAGES>;
  auto kern = k_gemm<BM, BN, WM, WN, TA, TB, STAGES, EPI>;
  constexpr size_t smem = (EPI == 2 && Cfg::SMEM_EPI2 > Cfg::SMEM) ? Cfg::SMEM_EPI2 : Cfg::SMEM;
  static_assert(Cfg::SMEM >= (size_t)STAGES * (BM + BN) * Cfg::BK * 8 + 1024 + 8 * STAGES, "TMA ring fits");
  GemmArgs g = g0;
  g.use_tma = 0;
  if constexpr (!TA) {  // TMA tiles where both operands are strided batches
    if (tma_enabled() && encode_operand(&g.tma_a, g.A, g.M, g.K, g.batch, 16, BM, true) &&
        (TB ? encode_operand(&g.tma_b, g.B, g.N, g.K, g.batch, 16, BN, true)
            : encode_operand(&g.tma_b, g.B, g.K, g.N, g.batch, 8, 16, false)))
      g.use_tma = 1;
  }
  if (cudaError_t e = ensure_smem(kern, smem)) return e;
  dim3 grid((g.N + BN - 1) / BN, (g.M + BM - 1) / BM, g.batch);
  launch_pdl(kern, grid, dim3(Cfg::THREADS), smem, st, g);
  return cudaGetLastError();
}

static int variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("KS_GEMM_VARIANT");  // tile-shape experiments (tools/gemm_probe.py)
    v = e ? std::atoi(e) : 0;
  }
  return v;
}

template <bool TA, bool TB>
cudaError_t dispatch(const GemmArgs& g, cudaStream_t st) {
  switch (variant()) {
    case 1: return launch<128, 64, 2, 2, TA, TB, 3>(g, st);
    case 2: return launch<128, 64, 4, 2, TA, TB, 4>(g, st);
    case 3: return launch<128, 128, 2, 4, TA, TB, 4>(g, st);
    case 4: return launch<128, 128, 4, 2, TA, TB, 3>(g, st);
    case 5: return launch<64, 64, 2, 2, TA, TB, 4>(g, st);
    default: break;
  }
  // Large output tiles when there is enough work to fill the 148 SMs with
  // them; otherwise narrower tiles (N <= 64 panels, small per-node blocks).
  // measured on B200 with tools/gemm_variants.py: N <= 64 panels keep 128x64
  // tiles (8 warps, 32x32 warp tiles); wider outputs use 64x32 warp tiles
  // (128x64 CTA tiles) when K is long and 64x64 tiles with 4 stages otherwise
  if (g.tri == 2 && (g.N <= 64 || g.M != g.N)) {
    GemmArgs t = g;
    t.tri = 0;
    return dispatch<TA, TB>(t, st);
  }
  if (g.N <= 16) return launch<128, 16, 4, 1, TA, TB, 3>(g, st);
  if (g.N <= 32) return launch<128, 32, 4, 1, TA, TB, 3>(g, st);
  if (g.N <= 64) {
    if (g.M >= 128 && (long)((g.M + 127) / 128) * g.batch >= 2 * 148)
      return launch<128, 64, 4, 2, TA, TB, 3>(g, st);
    return launch<64, 64, 2, 2, TA, TB, 4>(g, st);
  }
  const long tiles = (long)((g.M + 127) / 128) * ((g.N + 63) / 64) * g.batch;
  if (g.K >= 512 && tiles >= 2 * 148) return launch<128, 64, 2, 2, TA, TB, 3>(g, st);
  return launch<64, 64, 2, 2, TA, TB, 4>(g, st);
}

template <int BM, int BN, int WM, int WN, int STAGES, bool TB = false, int EPI = 0>
cudaError_t launch_group(const GemmGroup& gg, cudaStream_t st) {
  using Cfg = GemmCfg<BM, BN, WM, WN, false, TB, STAGES>;
  auto kern = k_gemm_group<BM, BN, WM, WN, false, TB, STAGES, EPI>;
  if (cudaError_t e = ensure_smem(kern, Cfg::SMEM)) return e;
  const GemmArgs& g = gg.p[0];
  GemmGroup gt = gg;
  for (int i = 0; i < gt.count; ++i) {  // TMA per problem where both operands are strided batches
    GemmArgs& q = gt.p[i];
    q.use_tma = tma_enabled() && encode_operand(&q.tma_a, q.A, q.M, q.K, q.batch, 16, BM, true) &&
                (TB ? encode_operand(&q.tma_b, q.B, q.N, q.K, q.batch, 16, BN, true)
                    : encode_operand(&q.tma_b, q.B, q.K, q.N, q.batch, 8, 16, false));
  }
  dim3 grid((g.N + BN - 1) / BN, (g.M + BM - 1) / BM, g.batch * gg.count);
  launch_pdl(kern, grid, dim3(Cfg::THREADS), Cfg::SMEM, st, gt);
  return cudaGetLastError();
}

}  // namespace

cudaError_t gemm_group(const GemmGroup& gg, cudaStream_t st) {
  if (gg.count < 1 || gg.count > kGroupMax) return cudaErrorInvalidValue;
  const GemmArgs& g = gg.p[0];
  if (g.M <= 0 || g.N <= 0 || g.batch <= 0) return cudaSuccess;
  for (int i = 0; i < gg.count; ++i) {
    const GemmArgs& q = gg.p[i];
    if (q.M != g.M || q.N != g.N || q.K != g.K || q.batch != g.batch || q.tri == 1) return cudaErrorInvalidValue;
    if (q.tri == 2 && q.M != q.N) return cudaErrorInvalidValue;
    if (((q.M | q.N | q.K) & 1) || q.K <= 0 || ((q.A.ld | q.B.ld | q.C.ld) & 1)) return cudaErrorInvalidValue;
  }
  // the same shape choice as gemm() for these products (K = s_pad < 512)
  const long tiles = (long)((g.M + 127) / 128) * ((g.N + 63) / 64) * g.batch * gg.count;
  if (g.K >= 512 && tiles >= 2 * 148) return launch_group<128, 64, 2, 2, 3>(gg, st);
  return launch_group<64, 64, 2, 2, 4>(gg, st);
}

cudaError_t gemm_group_coupling(const GemmGroup& gg, cudaStream_t st) {
  if (gg.count < 1 || gg.count > kGroupMax) return cudaErrorInvalidValue;
  const GemmArgs& g = gg.p[0];
  if (g.M <= 0 || g.N <= 0 || g.batch <= 0) return cudaSuccess;
  for (int i = 0; i < gg.count; ++i) {
    const GemmArgs& q = gg.p[i];
    if (q.M != g.M || q.N != g.N || q.K != g.K || q.batch != g.batch) return cudaErrorInvalidValue;
    if (((q.M | q.N | q.K) & 1) || q.K <= 0 || ((q.A.ld | q.B.ld | q.C.ld) & 1)) return cudaErrorInvalidValue;
  }
  return launch_group<64, 64, 2, 2, 4, true, 4>(gg, st);
}

cudaError_t gemm_gauss(const GemmArgs& g, cudaStream_t st) {
  if ((g.K & 1) || (g.A.ld & 1) || (g.C.ld & 1)) return cudaErrorInvalidValue;
  GemmArgs t = g;
  t.tri = 1;
  // K = d is small and the exp epilogue dominates: small tiles, 2 stages, many warps per SM
  return launch<64, 64, 2, 4, false, true, 2, 1>(t, st);
}

cudaError_t gemm_small_tile(const GemmArgs& g, cudaStream_t st) {
  // one 64 x 64 output per batch entry with a long K (leaf diagonal-block
  // updates): 8 warps per tile so one tile keeps the tensor pipe busier
  if (g.M != 64 || g.N != 64 || (g.K & 1) || g.K <= 0 || ((g.A.ld | g.B.ld | g.C.ld) & 1)) return gemm(g, false, true, st);
  const char* e = std::getenv("KS_DIAG_TILE");
  if (e && e[0] == '0') return gemm(g, false, true, st);
  return launch<64, 64, 2, 4, false, true, 4>(g, st);
}

cudaError_t gemm_syrk(const GemmArgs& g, cudaStream_t st) {
  if (g.M <= 0 || g.batch <= 0) return cudaSuccess;
  if (g.M != g.N || ((g.M | g.K) & 1) || g.K <= 0 || ((g.A.ld | g.B.ld | g.C.ld) & 1) || g.beta != 0.0)
    return cudaErrorInvalidValue;
  GemmArgs t = g;
  t.tri = 1;
  // 64 x 64 tiles: 10 of the 16 tiles of a 256 x 256 block are computed (6 of 8 with 128 x 64)
  return launch<64, 64, 2, 2, false, true, 4, 5>(t, st);
}

cudaError_t gemm_update_trsm(const GemmArgs& g, cudaStream_t st) {
  if (g.M <= 0 || g.batch <= 0) return cudaSuccess;
  if (g.N != 64 || (g.K & 1) || g.K <= 0 || ((g.A.ld | g.B.ld | g.C.ld | g.E.ld) & 1)) return cudaErrorInvalidValue;
  return launch<128, 64, 4, 2, false, true, 3, 2>(g, st);
}

cudaError_t gemm_krr(const GemmArgs& g, int* tiles, cudaStream_t st) {
  *tiles = (g.N + 63) / 64;
  if (g.M <= 0 || g.N <= 0) return cudaSuccess;
  if ((g.K & 1) || g.K <= 0 || ((g.A.ld | g.B.ld) & 1)) return cudaErrorInvalidValue;
  return launch<64, 64, 2, 2, false, true, 3, 3>(g, st);
}

cudaError_t gemm(const GemmArgs& g, bool ta, bool tb, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0 || g.batch <= 0) return cudaSuccess;
  if ((g.M | g.N | g.K) & 1) return cudaErrorInvalidValue;
  if ((g.A.ld | g.B.ld | g.C.ld) & 1) return cudaErrorInvalidValue;
  if (g.K <= 0) return cudaErrorInvalidValue;
  if (!ta && !tb) return dispatch<false, false>(g, st);
  if (!ta && tb) return dispatch<false, true>(g, st);
  if (ta && !tb) return dispatch<true, false>(g, st);
  return dispatch<true, true>(g, st);
}

}  // namespace ks
