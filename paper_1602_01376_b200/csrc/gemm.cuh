// Batched fp64 GEMM on the DMMA tensor pipe (mma.sync m8n8k4 f64 -> DMMA.8x8x4).
//
//   C[b] = alpha * op(A[b]) * op(B[b]) + beta * C[b]      (row-major storage)
//   op(A) = A (M x K, K contiguous)  or  A^T (A stored K x M)      [TA]
//   op(B) = B (K x N, N contiguous)  or  B^T (B stored N x K)      [TB]
//
// This is the workhorse of the factorization: the leaf Cholesky panel updates
// and panel TRSMs, the leaf SYRK H = L21 L21^T, the Z / -PG assembly products
// and the trailing updates of the recursive LU all run through it.
//
// Tiles are staged global->shared with a cp.async multistage pipeline; shared
// tiles are padded so that every DMMA fragment load (8-byte, half-warp phases)
// is bank-conflict free: a leading dimension == 4 (mod 16) doubles.
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace ks {

// Optional fused epilogues (template EPI):
//   0  C = alpha*AB + beta*C
//   1  Gaussian kernel block from the Gram matrix G = X X^T of a leaf
//      (kernels.py:107-111 in GEMM form): C[r][c] = exp(max(xx_r + xx_c - 2G, 0)
//      / (-2 h h)) for r > c, 1 + lam on the diagonal (r == c: distance exactly 0,
//      kernel exactly 1, solver.py:124), identity on padded rows/columns
//      (r or c >= size[b]) and 0 above the diagonal.
//   2  panel TRSM folded into a panel update (N == BN == 64):
//      C = (alpha*AB + beta*C) * E^T, E[b] a 64 x 64 LOWER TRIANGULAR block (the
//      inverse of the panel's diagonal Cholesky factor): the updated tile is staged
//      in shared memory and multiplied on the tensor pipe before it is stored
//      (only the k <= c terms: E's zeros are skipped).
struct GaussEpi {
  const double* xx;   // squared norms of the points, tree order
  const int* begin;   // per batch: first point of the leaf
  const int* size;    // per batch: points in the leaf
  const double* lam;  // device scalar
  double h;
};

//   3  dense Gaussian cross-kernel matvec (krr_predict, solver.py:273-301):
//      per row r of the tile, sum_c exp(max(xx_r + yy_c - 2G, 0) / (-2 h h)) w_c
//      over the tile's valid columns -> partial[blockIdx.x][r] (no C written).
struct KrrEpi {
  const double* xx;  // squared norms of the test points (rows)
  const double* yy;  // squared norms of the training points (columns)
  const double* w;   // weights (columns)
  double* partial;   // n_col_tiles x M
  double den;        // 1 / (-2 h h)
};

//   5  SYRK C = alpha * A A^T (BM == BN, tri = 1): tiles strictly above the diagonal
//      are skipped, tiles below it also store their transpose, diagonal tiles
//      compute both halves (the two sums have the same terms in the same order, so
//      C is symmetric bit for bit: the reference's 0.5 (H + H^T), solver.py:135, is
//      the identity on it).
//   4  coupling block B = K(S_l, S_r) from the Gram product of gathered skeleton
//      coordinates (kernels.py:107-111 in GEMM form, compress.py:281-283):
//      C[r][c] = exp(max(xa_r + xb_c - 2G, 0) / (-2 h h)) for r < rank(na[b]),
//      c < rank(nb[b]), else 0 (the zero padding to s_pad).
struct CoupEpi {
  const double* xa;   // squared norms of the A rows, per batch entry (stride xs)
  const double* xb;   // squared norms of the B rows
  int64_t xs;
  const int* na;      // per batch: the node whose rank bounds the rows
  const int* nbn;     // per batch: the node whose rank bounds the columns
  const int* rank;    // ranks by node id
  double den;         // 1 / (-2 h h)
};

struct GemmArgs {
  int M, N, K, batch;
  Operand A, B;
  OperandW C;
  double alpha, beta;
  int tri;  // 1: skip CTA tiles strictly above the diagonal of C (n0 >= m0 + BM); 2 (EPI 0,
            // M == N, BM a multiple of BN): also store the transpose of every tile strictly
            // below the diagonal (n0 + BN <= m0) -- a symmetric result from the tiles on
            // and below the diagonal (10 of 16 with 64 x 64 tiles)
  // EPI == 0: the beta term reads Cin instead of C when Cin.ptr is set (an
  // out-of-place C = alpha*AB + beta*Cin), and addI adds the identity
  // (C = alpha*AB + beta*Cin + I): the node assembly forms S = I - Y X and
  // E = P_r^T - Y P_l^T without initializing Aug first
  Operand Cin;
  int addI;
  GaussEpi ge;
  Operand E;  // EPI == 2: right factor of the epilogue product
  KrrEpi ke;  // EPI == 3
  CoupEpi ce;  // EPI == 4
  // TMA operand tiles (set by the host launcher for op(A) = A with strided,
  // 16-byte aligned batches): 3-D tensor maps; A and B^T as (K, rows, batch)
  // with boxes of 16 x rows and the 128-byte swizzle, B (K x N) as (N, K,
  // batch) with unswizzled boxes of 8 x 16
  int use_tma;
  CUtensorMap tma_a, tma_b;
};

template <int BM, int BN, int WM, int WN, bool TA, bool TB, int STAGES>
struct GemmCfg {
  static constexpr int BK = 16;
  static constexpr int THREADS = WM * WN * 32;
  static constexpr int WTM = BM / WM, WTN = BN / WN;
  static constexpr int MT = WTM / 8, NT = WTN / 8;
  static constexpr int A_ROWS = TA ? BK : BM, A_COLS = TA ? BM : BK, A_LD = A_COLS + 4;
  static constexpr int B_ROWS = TB ? BN : BK, B_COLS = TB ? BK : BN, B_LD = B_COLS + 4;
  static constexpr int A_STAGE = A_ROWS * A_LD, B_STAGE = B_ROWS * B_LD;
  static constexpr size_t SMEM = (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double);
  // EPI == 2 reuses the pipeline buffers for the staged tile and E
  static constexpr int T_LD = BN + 4;
  static constexpr size_t SMEM_EPI2 = (size_t)(BM + BN) * T_LD * sizeof(double);
  static_assert(A_LD % 16 == 4 && B_LD % 16 == 4, "conflict-free fragment loads need ld = 4 mod 16");
};

// ---- TMA (cp.async.bulk.tensor) + mbarrier helpers ----
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_inval(uint32_t bar) { asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(bar)); }
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// box (16 doubles of K) x rows at (k0, r0, batch) of the 3-D map into dst (1024-byte aligned)
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int k0, int r0, int b, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(k0), "r"(r0), "r"(b), "r"(bar)
      : "memory");
}
// element (r, k) of a 16-wide row-major tile stored with the 128-byte swizzle
// (16-byte chunk c of row r at chunk c ^ (r & 7)), in doubles from the tile base
__device__ __forceinline__ int swz128(int r, int k) { return r * 16 + ((((k >> 1) ^ (r & 7)) << 1) | (k & 1)); }

template <int ROWS, int COLS, int LD, int THREADS>
__device__ __forceinline__ void load_tile(double* dst, const double* src, int64_t ld, int r0, int c0,
                                          int rlim, int clim) {
  // ROWS x COLS tile of a row-major matrix, 16-byte chunks (2 doubles).
  constexpr int CPR = COLS / 2;
  constexpr int CHUNKS = ROWS * CPR;
#pragma unroll
  for (int c = threadIdx.x; c < CHUNKS; c += THREADS) {
    const int r = c / CPR, cc = (c % CPR) * 2;
    const int gr = r0 + r, gc = c0 + cc;
    const bool ok = (gr < rlim) && (gc < clim);
    const double* s = ok ? src + (int64_t)gr * ld + gc : src;
    cp_async16(dst + r * LD + cc, s, ok ? 16 : 0);
  }
}

// One BM x BN output tile (m0, n0) of batch entry b.
template <int BM, int BN, int WM, int WN, bool TA, bool TB, int STAGES, int EPI = 0>
__device__ __forceinline__ void gemm_tile(const GemmArgs& g, int b, int m0, int n0, double* smem) {
  using Cfg = GemmCfg<BM, BN, WM, WN, TA, TB, STAGES>;
  constexpr int BK = Cfg::BK;
  double* As = smem;
  double* Bs = smem + STAGES * Cfg::A_STAGE;
  if (g.tri && n0 >= m0 + BM) return;
  const double* A = g.A.at(b);
  const double* B = g.B.at(b);
  double* C = g.C.at(b);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm0 = (warp / WN) * Cfg::WTM, wn0 = (warp % WN) * Cfg::WTN;
  const int gq = lane >> 2, tq = lane & 3;

  double acc[Cfg::MT][Cfg::NT][2];
#pragma unroll
  for (int i = 0; i < Cfg::MT; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int KT = (g.K + BK - 1) / BK;
  bool tma_done = false;
  if constexpr (!TA) {
    if (g.use_tma) {
      // TMA ring: thread 0 arms a stage's mbarrier with its byte count and issues
      // the A and B boxes; every warp waits on the barrier's phase, computes, and
      // the barrier at the top of the next step frees the stage for its refill.
      const uint32_t sbase = (smem_u32(smem) + 1023u) & ~1023u;
      constexpr uint32_t A_BYTES = BM * BK * 8, B_BYTES = BN * BK * 8;
      const uint32_t bar0 = sbase + STAGES * (A_BYTES + B_BYTES);
      const double* sgen = smem + (sbase - smem_u32(smem)) / 8;  // generic pointer of sbase
      if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < STAGES; ++s) mbar_init(bar0 + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      }
      __syncthreads();
      auto issue_tma = [&](int stage, int kt) {
        const uint32_t bar = bar0 + 8 * stage;
        mbar_expect_tx(bar, A_BYTES + B_BYTES);
        tma_load_3d(sbase + stage * (A_BYTES + B_BYTES), &g.tma_a, kt * BK, m0, b, bar);
        if constexpr (TB) {
          tma_load_3d(sbase + stage * (A_BYTES + B_BYTES) + A_BYTES, &g.tma_b, kt * BK, n0, b, bar);
        } else {  // B is K x N: BN / 8 boxes of 8 columns x 16 rows, unswizzled
#pragma unroll
          for (int q = 0; q < BN / 8; ++q)
            tma_load_3d(sbase + stage * (A_BYTES + B_BYTES) + A_BYTES + q * 8 * BK * 8, &g.tma_b, n0 + q * 8, kt * BK, b,
                        bar);
        }
      };
      if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < STAGES - 1; ++s)
          if (s < KT) issue_tma(s, s);
      }
      for (int kt = 0; kt < KT; ++kt) {
        const int stage = kt % STAGES;
        __syncthreads();  // every warp is done with the stage refilled below
        if (threadIdx.x == 0) {
          const int nk = kt + STAGES - 1;
          if (nk < KT) issue_tma(nk % STAGES, nk);
        }
        mbar_wait(bar0 + 8 * stage, (uint32_t)((kt / STAGES) & 1));
        const double* as = sgen + stage * (A_BYTES + B_BYTES) / 8;
        const double* bs = as + A_BYTES / 8;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
          double af[Cfg::MT], bf[Cfg::NT];
#pragma unroll
          for (int i = 0; i < Cfg::MT; ++i) af[i] = as[swz128(wm0 + i * 8 + gq, kk + tq)];
#pragma unroll
          for (int j = 0; j < Cfg::NT; ++j) {
            const int c = wn0 + j * 8 + gq, k = kk + tq;
            // TB: N x 16 rows, 128-byte swizzle; else 8-column boxes [c / 8][k][c % 8]
            // (64-byte rows: the warp's four k rows fill two distinct bank halves twice)
            bf[j] = TB ? bs[swz128(c, k)] : bs[(c >> 3) * (8 * BK) + k * 8 + (c & 7)];
          }
#pragma unroll
          for (int i = 0; i < Cfg::MT; ++i)
#pragma unroll
            for (int j = 0; j < Cfg::NT; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
      }
      __syncthreads();  // all stages consumed: the barriers' memory may be reused
      if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < STAGES; ++s) mbar_inval(bar0 + 8 * s);
      }
      __syncthreads();
      tma_done = true;
    }
  }
  if (!tma_done) {
  auto issue = [&](int stage, int kt) {
    const int k0 = kt * BK;
    double* as = As + stage * Cfg::A_STAGE;
    double* bs = Bs + stage * Cfg::B_STAGE;
    if (!TA)
      load_tile<BM, BK, Cfg::A_LD, Cfg::THREADS>(as, A, g.A.ld, m0, k0, g.M, g.K);
    else
      load_tile<BK, BM, Cfg::A_LD, Cfg::THREADS>(as, A, g.A.ld, k0, m0, g.K, g.M);
    if (!TB)
      load_tile<BK, BN, Cfg::B_LD, Cfg::THREADS>(bs, B, g.B.ld, k0, n0, g.K, g.N);
    else
      load_tile<BN, BK, Cfg::B_LD, Cfg::THREADS>(bs, B, g.B.ld, n0, k0, g.N, g.K);
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) issue(s, s);
    cp_async_commit();
  }

  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      if (nk < KT) issue(nk % STAGES, nk);
      cp_async_commit();
    }
    const double* as = As + (kt % STAGES) * Cfg::A_STAGE;
    const double* bs = Bs + (kt % STAGES) * Cfg::B_STAGE;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[Cfg::MT], bf[Cfg::NT];
#pragma unroll
      for (int i = 0; i < Cfg::MT; ++i) {
        const int r = wm0 + i * 8 + gq, k = kk + tq;
        af[i] = TA ? as[k * Cfg::A_LD + r] : as[r * Cfg::A_LD + k];
      }
#pragma unroll
      for (int j = 0; j < Cfg::NT; ++j) {
        const int c = wn0 + j * 8 + gq, k = kk + tq;
        bf[j] = TB ? bs[c * Cfg::B_LD + k] : bs[k * Cfg::B_LD + c];
      }
#pragma unroll
      for (int i = 0; i < Cfg::MT; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::NT; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
  }
  const double alpha = g.alpha, beta = g.beta;
  if constexpr (EPI == 2) {
    constexpr int TL = Cfg::T_LD;
    static_assert(TL % 16 == 4, "conflict-free fragment loads");
    __syncthreads();  // every warp is done with the pipeline buffers
    double* Ts = smem;            // BM x BN updated tile
    double* Es = smem + BM * TL;  // BN x BN, E[c][k]
    const double* E = g.E.at(b);
    for (int e = threadIdx.x; e < BN * BN / 2; e += Cfg::THREADS) {
      const int r = e / (BN / 2), c = (e % (BN / 2)) * 2;
      *reinterpret_cast<double2*>(Es + r * TL + c) = *reinterpret_cast<const double2*>(E + (int64_t)r * g.E.ld + c);
    }
#pragma unroll
    for (int i = 0; i < Cfg::MT; ++i) {
      const int rl = wm0 + i * 8 + gq, r = m0 + rl;
#pragma unroll
      for (int j = 0; j < Cfg::NT; ++j) {
        const int cl = wn0 + j * 8 + 2 * tq;
        double2 v = make_double2(alpha * acc[i][j][0], alpha * acc[i][j][1]);
        if (beta != 0.0 && r < g.M) {
          const double2 ov = *reinterpret_cast<const double2*>(C + (int64_t)r * g.C.ld + n0 + cl);
          v.x = fma(beta, ov.x, v.x);
          v.y = fma(beta, ov.y, v.y);
        }
        *reinterpret_cast<double2*>(Ts + rl * TL + cl) = v;
        acc[i][j][0] = acc[i][j][1] = 0.0;
      }
    }
    __syncthreads();
    // E is lower triangular (E[c][k] = 0 for k > c): output columns
    // [c0, c0 + 8) need only k < c0 + 8 (warp-uniform bounds; the skipped
    // products are exact zeros)
#pragma unroll
    for (int kk = 0; kk < BN; kk += 4) {
      if (kk >= wn0 + Cfg::WTN) break;
      double af[Cfg::MT], bf[Cfg::NT];
#pragma unroll
      for (int i = 0; i < Cfg::MT; ++i) af[i] = Ts[(wm0 + i * 8 + gq) * TL + kk + tq];
#pragma unroll
      for (int j = 0; j < Cfg::NT; ++j) bf[j] = Es[(wn0 + j * 8 + gq) * TL + kk + tq];
#pragma unroll
      for (int j = 0; j < Cfg::NT; ++j) {
        if (kk >= wn0 + j * 8 + 8) continue;
#pragma unroll
        for (int i = 0; i < Cfg::MT; ++i) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
    }
#pragma unroll
    for (int i = 0; i < Cfg::MT; ++i) {
      const int r = m0 + wm0 + i * 8 + gq;
      if (r >= g.M) continue;
#pragma unroll
      for (int j = 0; j < Cfg::NT; ++j) {
        const int c = n0 + wn0 + j * 8 + 2 * tq;
        *reinterpret_cast<double2*>(C + (int64_t)r * g.C.ld + c) = make_double2(acc[i][j][0], acc[i][j][1]);
      }
    }
    return;
  }
  if constexpr (EPI == 3) {
    __syncthreads();  // pipeline buffers become the cross-warp row reduction
    double* red = smem;  // BM x WN
#pragma unroll
    for (int i = 0; i < Cfg::MT; ++i) {
      const int rl = wm0 + i * 8 + gq, r = m0 + rl;
      const double xr = (r < g.M) ? g.ke.xx[r] : 0.0;
      double sacc = 0.0;
#pragma unroll
      for (int j = 0; j < Cfg::NT; ++j) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int c = n0 + wn0 + j * 8 + 2 * tq + u;
          if (r < g.M && c < g.N) {
            const double sq = fmax(xr + g.ke.yy[c] - 2.0 * acc[i][j][u], 0.0);
            sacc = fma(exp(sq * g.ke.den), g.ke.w[c], sacc);
          }
        }
      }
      sacc += __shfl_xor_sync(0xffffffffu, sacc, 1);
      sacc += __shfl_xor_sync(0xffffffffu, sacc, 2);
      if (tq == 0) red[rl * WN + (warp % WN)] = sacc;
    }
    __syncthreads();
    for (int rl = threadIdx.x; rl < BM; rl += Cfg::THREADS) {
      const int r = m0 + rl;
      if (r >= g.M) continue;
      double s = 0.0;
#pragma unroll
      for (int w2 = 0; w2 < WN; ++w2) s += red[rl * WN + w2];
      g.ke.partial[(int64_t)blockIdx.x * g.M + r] = s;
    }
    return;
  }
  if constexpr (EPI == 4) {
    double cf[12];
    exp_coeffs(cf);
    const int ra = g.ce.rank[g.ce.na[b]], rb = g.ce.rank[g.ce.nbn[b]];
    const double* xa = g.ce.xa + (int64_t)b * g.ce.xs;
    const double* xb = g.ce.xb + (int64_t)b * g.ce.xs;
#pragma unroll
    for (int i = 0; i < Cfg::MT; ++i) {
      const int r = m0 + wm0 + i * 8 + gq;
      if (r >= g.M) continue;
      const double xr = (r < ra) ? xa[r] : 0.0;
#pragma unroll
      for (int j = 0; j < Cfg::NT; ++j) {
        const int c = n0 + wn0 + j * 8 + 2 * tq;
        if (c >= g.N) continue;
        double o[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int cc = c + u;
          o[u] = (r < ra && cc < rb) ? exp_neg(fmax(xr + xb[cc] - 2.0 * acc[i][j][u], 0.0) * g.ce.den, cf) : 0.0;
        }
        *reinterpret_cast<double2*>(C + (int64_t)r * g.C.ld + c) = make_double2(o[0], o[1]);
      }
    }
    return;
  }
  double den = 0.0, lam = 0.0;
  int bsz = 0, bbeg = 0;
  const double* Cin = (EPI == 0 && g.Cin.ptr) ? g.Cin.at(b) : nullptr;
  (void)Cin;
  if (EPI == 1) {
    den = 1.0 / (-2.0 * g.ge.h * g.ge.h);  // multiply by the reciprocal: one rounding in the exponent
    lam = *g.ge.lam;
    bsz = g.ge.size[b];
    bbeg = g.ge.begin[b];
  }
  if constexpr (EPI == 1) {
    // tiles strictly below the diagonal and inside the leaf (120 of the 136
    // lower tiles of a full 1024-point leaf): no per-element cases
    if (n0 + BN <= m0 && m0 + BM <= bsz) {
      double cf[12];
      exp_coeffs(cf);
      double xc[Cfg::NT][2];
#pragma unroll
      for (int j = 0; j < Cfg::NT; ++j) {
        xc[j][0] = g.ge.xx[bbeg + n0 + wn0 + j * 8 + 2 * tq];
        xc[j][1] = g.ge.xx[bbeg + n0 + wn0 + j * 8 + 2 * tq + 1];
      }
#pragma unroll
      for (int i = 0; i < Cfg::MT; ++i) {
        const int r = m0 + wm0 + i * 8 + gq;
        const double xr = g.ge.xx[bbeg + r];
#pragma unroll
        for (int j = 0; j < Cfg::NT; ++j) {
          const int c = n0 + wn0 + j * 8 + 2 * tq;
          double2 v;
          v.x = exp_neg(fmax(xr + xc[j][0] - 2.0 * acc[i][j][0], 0.0) * den, cf);
          v.y = exp_neg(fmax(xr + xc[j][1] - 2.0 * acc[i][j][1], 0.0) * den, cf);
          *reinterpret_cast<double2*>(C + (int64_t)r * g.C.ld + c) = v;
        }
      }
      return;
    }
  }
#pragma unroll
  for (int i = 0; i < Cfg::MT; ++i) {
    const int r = m0 + wm0 + i * 8 + gq;
    if (r >= g.M) continue;
    double xr = 0.0;
    if (EPI == 1 && r < bsz) xr = g.ge.xx[bbeg + r];
#pragma unroll
    for (int j = 0; j < Cfg::NT; ++j) {
      const int c = n0 + wn0 + j * 8 + 2 * tq;
      if (c >= g.N) continue;
      double2* p = reinterpret_cast<double2*>(C + (int64_t)r * g.C.ld + c);
      double2 v;
      if (EPI == 1) {
        double o[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int cc = c + u;
          if (cc > r) o[u] = 0.0;
          else if (r >= bsz || cc >= bsz) o[u] = (r == cc) ? 1.0 : 0.0;
          else if (r == cc) o[u] = 1.0 + lam;
          else {
            const double sq = fmax(xr + g.ge.xx[bbeg + cc] - 2.0 * acc[i][j][u], 0.0);
            o[u] = exp_neg(sq * den);
          }
        }
        v.x = o[0];
        v.y = o[1];
      } else {
        v.x = alpha * acc[i][j][0];
        v.y = alpha * acc[i][j][1];
        if (beta != 0.0) {
          const double2 ov = Cin ? *reinterpret_cast<const double2*>(Cin + (int64_t)r * g.Cin.ld + c) : *p;
          v.x = fma(beta, ov.x, v.x);
          v.y = fma(beta, ov.y, v.y);
        }
        if (g.addI) {
          if (r == c) v.x += 1.0;
          if (r == c + 1) v.y += 1.0;
        }
      }
      *p = v;
      if constexpr (EPI == 0) {
        if (g.tri == 2 && n0 + BN <= m0) {  // a tile strictly below the diagonal: its transpose lies in skipped tiles
          C[(int64_t)c * g.C.ld + r] = v.x;
          C[(int64_t)(c + 1) * g.C.ld + r] = v.y;
        }
      }
      if constexpr (EPI == 5) {  // SYRK: tiles below the diagonal also write their mirror image
        if (n0 < m0) {
          C[(int64_t)c * g.C.ld + r] = v.x;
          C[(int64_t)(c + 1) * g.C.ld + r] = v.y;
        }
      }
    }
  }
}

template <int BM, int BN, int WM, int WN, bool TA, bool TB, int STAGES, int EPI = 0>
__global__ void __launch_bounds__(WM* WN * 32) k_gemm(const __grid_constant__ GemmArgs g) {
  extern __shared__ __align__(16) double smem[];
  pdl_wait();
  gemm_tile<BM, BN, WM, WN, TA, TB, STAGES, EPI>(g, blockIdx.z, blockIdx.y * BM, blockIdx.x * BN, smem);
}

// Up to kGroupMax independent batched GEMMs of the same shape (M, N, K, batch)
// and transposes in one launch: grid.z = batch x problems. The node assembly
// of the block formulation issues its four independent products per stage
// this way (factorize.cu), one launch instead of four dependent ones.
constexpr int kGroupMax = 4;
struct GemmGroup {
  GemmArgs p[kGroupMax];
  int count;
};

template <int BM, int BN, int WM, int WN, bool TA, bool TB, int STAGES, int EPI = 0>
__global__ void __launch_bounds__(WM* WN * 32) k_gemm_group(const __grid_constant__ GemmGroup gg) {
  extern __shared__ __align__(16) double smem[];
  pdl_wait();
  const int batch = gg.p[0].batch;
  const int pi = blockIdx.z / batch, b = blockIdx.z - pi * batch;
  gemm_tile<BM, BN, WM, WN, TA, TB, STAGES, EPI>(gg.p[pi], b, blockIdx.y * BM, blockIdx.x * BN, smem);
}

// Host launcher: picks a tile shape for the problem; all dims must be even,
// leading dimensions even and base pointers 16-byte aligned.
cudaError_t gemm(const GemmArgs& g, bool ta, bool tb, cudaStream_t st);
// Leaf Gaussian blocks through the Gram GEMM with the EPI == 1 epilogue
// (lower-triangular tiles only).
cudaError_t gemm_gauss(const GemmArgs& g, cudaStream_t st);
// 64 x 64 outputs with long K (op(B) = B^T), 8 warps per tile.
cudaError_t gemm_small_tile(const GemmArgs& g, cudaStream_t st);
// C = alpha * A A^T, symmetric output written in full (EPI == 5): M == N, op(B) = B^T with B = A.
cudaError_t gemm_syrk(const GemmArgs& g, cudaStream_t st);
// Panel update with the panel TRSM folded in (EPI == 2): N must be 64, op(B) = B^T.
cudaError_t gemm_update_trsm(const GemmArgs& g, cudaStream_t st);
// gg.count problems of one shape (M, N, K, batch, alpha/beta per problem), no
// transposes, EPI 0, in one launch.
cudaError_t gemm_group(const GemmGroup& gg, cudaStream_t st);
// Coupling blocks (EPI == 4): op(B) = B^T (the gathered skeleton coordinates
// of both operands row-major, K = the padded dimension).
cudaError_t gemm_group_coupling(const GemmGroup& gg, cudaStream_t st);
// Gaussian cross-kernel row sums (EPI == 3), op(B) = B^T: partial sums per
// 64-column tile; returns the number of column tiles through *tiles.
cudaError_t gemm_krr(const GemmArgs& g, int* tiles, cudaStream_t st);

}  // namespace ks
