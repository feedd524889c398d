// Persistent per-node LU for the narrow (latency-bound) top levels of the tree.
//
// Reference: the internal-node step of factorize (solver.py:138-165): LU with
// partial pivoting of Z (linalg.py:199-213), then H = P G Z^-1 P^T. The GPU
// factors the augmented matrix [[Z, P^T], [-P G, 0]] (T x T, pivots among the
// first t_pad rows); its trailing block is H. The recursive
// launch sequence used for wide levels (capi.cu rlu: ~120 dependent launches
// per level) is replaced here by ONE cooperative launch per level:
//
//   * each CTA owns a W-column slab of one node's matrix, resident in shared
//     memory for the whole factorization (T x (W+1) doubles, <= 204 KB);
//   * step j (columns [jW, jW+W)) is factored by the CTA owning slab j: the
//     candidate rows in registers (lu_panel.cuh), published (rows [jW, t_pad))
//     with a release flag; then the augmented rows (never pivots) are
//     eliminated and published behind a second flag, off the path from one
//     panel to the next;
//   * every other CTA acquires the flag, applies the step's row interchanges to
//     its slab (LAPACK convention: also to the finished L columns), and, for
//     slabs right of the panel, U12 = L11^-1 A12 and the trailing update
//     A22 -= L21 U12 on the fp64 tensor pipe (DMMA m8n8k4, L21 streamed from L2);
//   * slab j+1 updates its candidate rows right after step j and starts the
//     next panel while the other slabs are still updating (look-ahead of one
//     step); its augmented rows catch up after that panel;
//   * after the last step the slabs are written back in place (same layout as
//     the launch sequence: L\U of Pi Z, U12 = L^-1 Pi P^T, L21aug, Schur block)
//     and the H slabs write sym(H) for the parent (solver.py:163).
// The 1-norm of Z for the condition estimate (linalg.py:176) is taken from the
// slabs before the first step. Waits are bounded (a watchdog sets an error
// word instead of hanging the GPU).
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"
#include "lu_panel.cuh"

namespace ks {

// KS_SLAB_TRACE=1: %globaltimer stamps of node 0 of the last traced launch,
// [slab][step][phase] (phase 0 acquired / panel start, 1 moves done / columns
// done, 2 U12 done / augmented rows done, 3 update done / published)
__device__ long long* g_slab_ts = nullptr;
constexpr int kTsSlabs = 128, kTsSteps = 64;

namespace {

__device__ __forceinline__ long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// all threads of the CTA: wait until *p >= target (false: watchdog expired)
__device__ bool cta_wait(const unsigned* p, unsigned target, unsigned* err, int* s_ok) {
  __syncthreads();
  if (threadIdx.x == 0) {
    int ok = 1;
    if (ld_acquire(p) < target) {
      const long long t0 = clock64();
      while (ld_acquire(p) < target) {
        if (clock64() - t0 > (1LL << 32)) {  // ~2 s: something is broken
          atomicExch(err, 1u);
          ok = 0;
          break;
        }
      }
    }
    *s_ok = ok;
  }
  __syncthreads();
  return *s_ok != 0;
}

// rows [c0, TP) of the slab (all SW columns) permuted by the step's NP row
// interchanges (spiv[i] = pivot of row c0+i, relative to c0): each touched row
// is followed through the swap sequence; all loads, one barrier, all stores.
template <int NP, int SW, int NT, int LD>
__device__ __forceinline__ void slab_moves(double* Sl, int c0, const int* spiv, int* msrc, int* mdst) {
  if (threadIdx.x < 2 * NP) {
    const int x = threadIdx.x < NP ? (int)threadIdx.x : spiv[threadIdx.x - NP];
    int f = x;
#pragma unroll 8
    for (int i = 0; i < NP; ++i) {
      const int p = spiv[i];
      f = (f == i) ? p : (f == p ? i : f);
    }
    msrc[threadIdx.x] = x;
    mdst[threadIdx.x] = f;
  }
  __syncthreads();
  constexpr int NE = 2 * NP * SW;
  constexpr int E = (NE + NT - 1) / NT;
  double v[E];
#pragma unroll
  for (int u = 0; u < E; ++u) {
    const int e = threadIdx.x + u * NT;
    if (e < NE) v[u] = Sl[(c0 + msrc[e / SW]) * LD + e % SW];
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < E; ++u) {
    const int e = threadIdx.x + u * NT;
    if (e < NE) {
      const int m = e / SW;
      if (msrc[m] != mdst[m]) Sl[(c0 + mdst[m]) * LD + e % SW] = v[u];
    }
  }
  __syncthreads();
}

// Sl[r][cc + n] -= sum_k A[r][ac + k] * Sl[ur + k][cc + n] for rows [r0, rend),
// k < KW, n < NC: warp tiles of 16 rows x NC columns on DMMA. A is the slab
// itself (ASM: shared memory, ld LD) or a published panel (global, ld lda).
template <int KW, int NC, int NT, int LD, bool ASM>
__device__ __forceinline__ void tile_update(double* Sl, int cc, const double* A, int64_t lda, int ac, int ur, int r0,
                                            int rend) {
  constexpr int KS = KW / 4, NN = NC / 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  double bf[KS][NN];
#pragma unroll
  for (int ks = 0; ks < KS; ++ks)
#pragma unroll
    for (int n = 0; n < NN; ++n) bf[ks][n] = Sl[(ur + ks * 4 + tq) * LD + cc + n * 8 + gq];
  const int ntiles = (rend - r0) / 16;
  for (int t = warp; t < ntiles; t += NT / 32) {
    const int r = r0 + t * 16;
    double af[2][KS];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int row = r + m * 8 + gq, col = ac + ks * 4 + tq;
        af[m][ks] = ASM ? -Sl[row * LD + col] : -__ldcg(A + (int64_t)row * lda + col);
      }
    double acc[2][NN][2];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int n = 0; n < NN; ++n) {
        acc[m][n][0] = Sl[(r + m * 8 + gq) * LD + cc + n * 8 + 2 * tq];
        acc[m][n][1] = Sl[(r + m * 8 + gq) * LD + cc + n * 8 + 2 * tq + 1];
      }
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int n = 0; n < NN; ++n) dmma884(acc[m][n][0], acc[m][n][1], af[m][ks], bf[ks][n]);
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int n = 0; n < NN; ++n) {
        Sl[(r + m * 8 + gq) * LD + cc + n * 8 + 2 * tq] = acc[m][n][0];
        Sl[(r + m * 8 + gq) * LD + cc + n * 8 + 2 * tq + 1] = acc[m][n][1];
      }
  }
}

// Sl rows [c0, c0+KW), columns [cc, cc+NC) := L^-1 (...), L unit lower KW x KW
// at Lm (ld LLD, shared memory): one thread per column.
template <int KW, int NC, int LD, int LLD>
__device__ __forceinline__ void tile_trsm(double* Sl, int c0, int cc, const double* Lm) {
  if (threadIdx.x < NC) {
    double x[KW];
#pragma unroll
    for (int i = 0; i < KW; ++i) x[i] = Sl[(c0 + i) * LD + cc + threadIdx.x];
#pragma unroll
    for (int i = 1; i < KW; ++i) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int q = 0; q + 3 < i; q += 4) {
        s0 = fma(Lm[i * LLD + q], x[q], s0);
        s1 = fma(Lm[i * LLD + q + 1], x[q + 1], s1);
        s2 = fma(Lm[i * LLD + q + 2], x[q + 2], s2);
        s3 = fma(Lm[i * LLD + q + 3], x[q + 3], s3);
      }
#pragma unroll
      for (int q = i & ~3; q < i; ++q) s0 = fma(Lm[i * LLD + q], x[q], s0);
      x[i] -= (s0 + s1) + (s2 + s3);
    }
#pragma unroll
    for (int i = 0; i < KW; ++i) Sl[(c0 + i) * LD + cc + threadIdx.x] = x[i];
  }
}

}  // namespace

// SW: slab width (columns per CTA); PW: panel width (columns per step, SW/PW
// steps per slab: the second panel of a slab is updated by its own CTA from
// shared memory right after the first); RPT: candidate rows per thread.
template <int SW, int PW, int RPT, int NT>
__global__ void __launch_bounds__(NT, 1)
    k_lu_slab(NodeBatch nb, double* Hout, int64_t h_stride, int write_h, unsigned* sync, unsigned* err, int groups) {
  constexpr int LD = SW + 1;  // odd row stride: conflict-free row-per-thread access
  constexpr int NW = NT / 32;
  constexpr int HV = SW / PW;  // steps per slab
  static_assert(HV == 1 || HV == 2, "slab = 1 or 2 panels");
  const int T = nb.T, TP = nb.t_pad, S = nb.s_pad;
  const int G = T / SW, nzs = TP / SW, nst = TP / PW;
  const int slab = blockIdx.x % G;
  const int col0 = slab * SW;
  extern __shared__ __align__(16) double smem[];
  double* Sl = smem;                    // T x LD: this CTA's slab
  double* L11 = smem + (size_t)T * LD;  // PW x (PW+1): unit-lower diagonal block of the step
  __shared__ PanelShared<NW, PW> ps;
  __shared__ double urcp[SW];  // the pivots' reciprocals of this slab's panels
  __shared__ int spiv[PW], msrc[2 * PW], mdst[2 * PW];
  __shared__ int s_ok;
  long long* ts = g_slab_ts;
  auto stamp = [&](int k, int j, int ph) {
    if (ts && k == 0 && threadIdx.x == 0 && slab < kTsSlabs && j < kTsSteps) ts[(slab * kTsSteps + j) * 4 + ph] = gtime();
  };
  for (int k = blockIdx.x / G; k < nb.count; k += groups) {
    double* A = nb.Aug + (int64_t)k * T * T;
    unsigned* sy = sync + 4 * k;
    int* pivk = nb.piv + (int64_t)k * TP;
    __syncthreads();
    for (int e = threadIdx.x; e < T * SW; e += NT) {
      const int r = e / SW, c = e % SW;
      Sl[r * LD + c] = A[(int64_t)r * T + col0 + c];
    }
    __syncthreads();
    if (slab < nzs) {  // ||Z||_1 over this slab's columns (rows < t_pad), linalg.py:176
      constexpr int NG = NT / SW;
      double* red = &ps.cand[0][0][0];  // 2*NW*PW >= NG*SW doubles
      static_assert(2 * NW * PW >= NG * SW, "scratch");
      const int c = threadIdx.x % SW, g = threadIdx.x / SW;
      double sacc = 0.0;
      for (int r = g; r < TP; r += NG) sacc += fabs(Sl[r * LD + c]);
      red[g * SW + c] = sacc;
      __syncthreads();
      if (threadIdx.x < 32) {
        double t = 0.0;
        if (threadIdx.x < SW)
          for (int gg = 0; gg < NG; ++gg) t += red[gg * SW + threadIdx.x];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t = fmax(t, __shfl_xor_sync(0xffffffffu, t, o));
        if (threadIdx.x == 0) atomicMax(reinterpret_cast<unsigned long long*>(nb.norm1 + k), __double_as_longlong(t));
      }
      __syncthreads();  // the scratch is the panel's candidate buffer
    }
    // Augmented rows lag behind: aug_done = steps whose update has been applied
    // to this slab's augmented rows (the columns right of that step's panel).
    // They never pivot and no panel needs them, so they are caught up off the
    // panel-to-panel path (before this slab's own eliminations and at the end).
    int aug_done = 0;
    auto aug_catch_up = [&](int upto) -> bool {
      for (int t = aug_done; t < upto; ++t) {
        const int ow = t / HV, ct = t * PW;
        if (ow < slab) {
          if (!cta_wait(sy + 3, (unsigned)(t + 1), err, &s_ok)) return false;
          tile_update<PW, SW, NT, LD, false>(Sl, 0, A, T, ct, ct, TP, T);
        } else if (ow == slab && (t % HV) + 1 < HV) {  // own left panel -> the right half
          if constexpr (HV > 1) {
            __syncthreads();
            tile_update<PW, SW - PW, NT, LD, true>(Sl, PW, nullptr, 0, 0, ct, TP, T);
          }
        }
      }
      aug_done = max(aug_done, upto);
      __syncthreads();
      return true;
    };
    for (int j = 0; j < nst; ++j) {
      const int c0 = j * PW;
      const int owner = j / HV;
      if (slab == owner) {
        // ---- this slab's HV panels: candidate rows first, published step by step ----
        for (int hh = 0; hh < HV; ++hh) {
          const int jj = j + hh, cj = jj * PW, pc = hh * PW;
          __syncthreads();  // the previous step's update of this slab is complete
          if (hh > 0) {
            // own previous panel (columns [0, PW)): U12 and the candidate rows of
            // this half, from shared memory
            tile_trsm<PW, PW, LD, LD>(Sl, cj - PW, PW, Sl + (size_t)(cj - PW) * LD);
            __syncthreads();
            tile_update<PW, PW, NT, LD, true>(Sl, PW, nullptr, 0, 0, cj - PW, cj, TP);
            __syncthreads();
          }
          stamp(k, jj, 0);
          const int rows = TP - cj;
          {
            double a[RPT][PW];
            int pos[RPT];
            bool done[RPT];
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
              const int r = threadIdx.x + i * NT;
              pos[i] = r;
              done[i] = (r >= rows);
#pragma unroll
              for (int q = 0; q < PW; ++q) a[i][q] = (r < rows) ? Sl[(cj + r) * LD + pc + q] : 0.0;
            }
            const int nact = panel_warps(rows, NT);
            if ((int)(threadIdx.x >> 5) < nact)
              panel_columns<PW, RPT, NT, (PW <= 16 ? PW : 16)>(a, pos, done, ps, Sl + (size_t)cj * LD + pc, LD, rows,
                                                               pivk + cj, cj, nb.info + k, cj, nact);
          }
          __syncthreads();
          stamp(k, jj, 1);
          if (threadIdx.x < PW) {
            spiv[threadIdx.x] = pivk[cj + threadIdx.x] - cj;
            urcp[pc + threadIdx.x] = ps.urcp[threadIdx.x];
          }
          __syncthreads();
          slab_moves<PW, SW, NT, LD>(Sl, cj, spiv, msrc, mdst);
          for (int e = threadIdx.x; e < (TP - cj) * PW; e += NT) {
            const int r = cj + e / PW, c = e % PW;
            A[(int64_t)r * T + col0 + pc + c] = Sl[r * LD + pc + c];
          }
          __threadfence();
          __syncthreads();
          if (threadIdx.x == 0) st_release(sy, (unsigned)(jj + 1));
          stamp(k, jj, 2);
        }
        // ---- then their augmented rows ----
        for (int hh = 0; hh < HV; ++hh) {
          const int jj = j + hh, cj = jj * PW, pc = hh * PW;
          if (!aug_catch_up(jj)) return;
          for (int r = TP + threadIdx.x; r < T; r += NT) {
            double x[PW];
#pragma unroll
            for (int q = 0; q < PW; ++q) x[q] = Sl[r * LD + pc + q];
#pragma unroll
            for (int kk = 0; kk < PW; ++kk) {
              const double l = x[kk] * urcp[pc + kk];
              x[kk] = l;
#pragma unroll
              for (int q = kk + 1; q < PW; ++q) x[q] = fma(-l, Sl[(cj + kk) * LD + pc + q], x[q]);
            }
#pragma unroll
            for (int q = 0; q < PW; ++q) Sl[r * LD + pc + q] = x[q];
          }
          __syncthreads();
          for (int e = threadIdx.x; e < (T - TP) * PW; e += NT) {
            const int r = TP + e / PW, c = e % PW;
            A[(int64_t)r * T + col0 + pc + c] = Sl[r * LD + pc + c];
          }
          __threadfence();
          __syncthreads();
          if (threadIdx.x == 0) st_release(sy + 3, (unsigned)(jj + 1));
          stamp(k, jj, 3);
        }
        j += HV - 1;
        continue;
      }
      // ---- any other slab: acquire step j ----
      if (!cta_wait(sy, (unsigned)(j + 1), err, &s_ok)) return;
      stamp(k, j, 0);
      if (threadIdx.x < PW) spiv[threadIdx.x] = __ldcg(pivk + c0 + threadIdx.x) - c0;
      __syncthreads();
      slab_moves<PW, SW, NT, LD>(Sl, c0, spiv, msrc, mdst);
      stamp(k, j, 1);
      if (slab < owner) continue;  // finished L columns: the interchanges only
      for (int e = threadIdx.x; e < PW * PW; e += NT) {
        const int i = e / PW, q = e % PW;
        L11[i * (PW + 1) + q] = __ldcg(A + (int64_t)(c0 + i) * T + c0 + q);
      }
      __syncthreads();
      tile_trsm<PW, SW, LD, PW + 1>(Sl, c0, 0, L11);
      __syncthreads();
      stamp(k, j, 2);
      tile_update<PW, SW, NT, LD, false>(Sl, 0, A, T, c0, c0, c0 + PW, TP);  // candidate rows
      // augmented rows one step behind, except on the slab that owns the next
      // panel (it catches up after its panels)
      const bool lookahead = (j + 1 < nst) && ((j + 1) / HV == slab);
      if (!lookahead && !aug_catch_up(j)) return;
      __syncthreads();
      stamp(k, j, 3);
    }
    if (!aug_catch_up(nst)) return;
    // ---- every CTA of the node is past the last step: write the slab back ----
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(sy + 1, 1u);
    }
    if (!cta_wait(sy + 1, (unsigned)G, err, &s_ok)) return;
    for (int e = threadIdx.x; e < T * SW; e += NT) {
      const int r = e / SW, c = e % SW;
      A[(int64_t)r * T + col0 + c] = Sl[r * LD + c];
    }
    if (write_h && slab >= nzs) {  // H = sym(trailing block) -> Hout[node] (solver.py:163)
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) atomicAdd(sy + 2, 1u);
      if (!cta_wait(sy + 2, (unsigned)(G - nzs), err, &s_ok)) return;
      double* hh = Hout + (int64_t)nb.node[k] * h_stride;
      for (int e = threadIdx.x; e < S * SW; e += NT) {
        const int i = e / SW, jj = e % SW, j2 = col0 - TP + jj;
        hh[(int64_t)i * S + j2] = 0.5 * (Sl[(TP + i) * LD + jj] + __ldcg(A + (int64_t)(TP + j2) * T + TP + i));
      }
    }
  }
}

// ---------------------------------------------------------------------------
// 32-column LU panel of the launch sequence (wide levels), factored as two
// 16-column halves in shared memory by one CTA per node: the second half is
// updated from the first (TRSM + DMMA tile update) inside the kernel, which
// replaces two panel launches, a 16-wide TRSM launch and a 16-wide GEMM launch
// of the recursion (capi.cu rlu) per 32 columns. Same pivot rule and output
// layout as two k_lu_panel2 launches with their merge; the row interchanges
// are applied to every column outside the panel.
// ---------------------------------------------------------------------------
template <int NT>
__global__ void __launch_bounds__(NT, 1) k_lu_panel32(NodeBatch nb, int c0) {
  constexpr int PW = 16, SW = 32, LD = SW + 1, NW = NT / 32;
  pdl_wait();
  const int k = blockIdx.x;
  const int T = nb.T, TP = nb.t_pad;
  const int nr = T - c0;          // panel rows [c0, T), relative index
  const int nz = TP - c0;         // candidate rows [0, nz)
  double* A = nb.Aug + (int64_t)k * T * T;
  int* pivk = nb.piv + (int64_t)k * TP;
  extern __shared__ __align__(16) double smem[];
  double* Sl = smem;  // nr x LD
  __shared__ PanelShared<NW, PW> ps;
  __shared__ double urcp[SW];
  __shared__ int spiv[SW], msrc[2 * SW], mdst[2 * SW];
  for (int e = threadIdx.x; e < nr * SW; e += NT) {
    const int r = e / SW, c = e % SW;
    Sl[r * LD + c] = A[(int64_t)(c0 + r) * T + c0 + c];
  }
  __syncthreads();
  for (int hh = 0; hh < 2; ++hh) {
    const int cj = hh * PW;  // relative first row/column of this half
    if (hh > 0) {
      tile_trsm<PW, PW, LD, LD>(Sl, 0, PW, Sl);
      __syncthreads();
      tile_update<PW, PW, NT, LD, true>(Sl, PW, nullptr, 0, 0, 0, PW, nz);
      __syncthreads();
    }
    const int rows = nz - cj;
    {
      double a[1][PW];
      int pos[1];
      bool done[1];
      const int r = threadIdx.x;
      pos[0] = r;
      done[0] = (r >= rows);
#pragma unroll
      for (int q = 0; q < PW; ++q) a[0][q] = (r < rows) ? Sl[(cj + r) * LD + cj + q] : 0.0;
      const int nact = panel_warps(rows, NT);
      if ((int)(threadIdx.x >> 5) < nact)
        panel_columns<PW, 1, NT, PW>(a, pos, done, ps, Sl + (size_t)cj * LD + cj, LD, rows, pivk + c0 + cj, c0 + cj,
                                     nb.info + k, c0 + cj, nact);
    }
    __syncthreads();
    if (threadIdx.x < PW) {
      spiv[threadIdx.x] = pivk[c0 + cj + threadIdx.x] - (c0 + cj);
      urcp[cj + threadIdx.x] = ps.urcp[threadIdx.x];
    }
    __syncthreads();
    slab_moves<PW, SW, NT, LD>(Sl, cj, spiv, msrc, mdst);
  }
  // augmented rows: first half, its update of the second half, second half
  for (int hh = 0; hh < 2; ++hh) {
    const int cj = hh * PW;
    if (hh > 0) {
      tile_update<PW, PW, NT, LD, true>(Sl, PW, nullptr, 0, 0, 0, nz, nr);
      __syncthreads();
    }
    for (int r = nz + threadIdx.x; r < nr; r += NT) {
      double x[PW];
#pragma unroll
      for (int q = 0; q < PW; ++q) x[q] = Sl[r * LD + cj + q];
#pragma unroll
      for (int kk = 0; kk < PW; ++kk) {
        const double l = x[kk] * urcp[cj + kk];
        x[kk] = l;
#pragma unroll
        for (int q = kk + 1; q < PW; ++q) x[q] = fma(-l, Sl[(cj + kk) * LD + cj + q], x[q]);
      }
#pragma unroll
      for (int q = 0; q < PW; ++q) Sl[r * LD + cj + q] = x[q];
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < nr * SW; e += NT) {
    const int r = e / SW, c = e % SW;
    A[(int64_t)(c0 + r) * T + c0 + c] = Sl[r * LD + c];
  }
  // the 32 interchanges for every column outside the panel (rows [c0, TP)):
  // touched rows followed through the swap sequence, all loads, then stores
  if (threadIdx.x < SW) spiv[threadIdx.x] = pivk[c0 + threadIdx.x] - c0;
  __syncthreads();
  if (threadIdx.x < 2 * SW) {
    const int x = threadIdx.x < SW ? (int)threadIdx.x : spiv[threadIdx.x - SW];
    int f = x;
    for (int i = 0; i < SW; ++i) {
      const int p = spiv[i];
      f = (f == i) ? p : (f == p ? i : f);
    }
    msrc[threadIdx.x] = (f != x) ? x : -1;
    mdst[threadIdx.x] = f;
  }
  __syncthreads();
  const int npair = (T - SW) / 2;
  constexpr int PER = 12;
  for (int e0 = 0; e0 < 2 * SW * npair; e0 += PER * NT) {
    double2 v[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = e0 + u * NT + threadIdx.x;
      if (e < 2 * SW * npair) {
        const int m = e / npair, x2 = 2 * (e % npair);
        const int col = x2 < c0 ? x2 : x2 + SW;
        if (msrc[m] >= 0) v[u] = *reinterpret_cast<const double2*>(A + (int64_t)(c0 + msrc[m]) * T + col);
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = e0 + u * NT + threadIdx.x;
      if (e < 2 * SW * npair) {
        const int m = e / npair, x2 = 2 * (e % npair);
        const int col = x2 < c0 ? x2 : x2 + SW;
        if (msrc[m] >= 0) *reinterpret_cast<double2*>(A + (int64_t)(c0 + mdst[m]) * T + col) = v[u];
      }
    }
    __syncthreads();
  }
}

bool lu_panel32_ok(const NodeBatch& nb) {
  return nb.t_pad <= 512 && nb.T % 32 == 0 && (size_t)nb.T * 33 * 8 <= 200 * 1024;
}

void launch_lu_panel32(const NodeBatch& nb, int c0, cudaStream_t st) {
  const size_t smem = (size_t)(nb.T - c0) * 33 * sizeof(double);
  ensure_smem(k_lu_panel32<512>, 200 * 1024);
  launch_pdl(k_lu_panel32<512>, dim3(nb.count), dim3(512), smem, st, nb, c0);
}

namespace {

template <int SW, int PW, int RPT>
int launch_slab_t(const NodeBatch& nb, double* H, int64_t hs, bool write_h, unsigned* sync, unsigned* err,
                  cudaStream_t st) {
  constexpr int NT = 512;
  const size_t smem = ((size_t)nb.T * (SW + 1) + (size_t)PW * (PW + 1)) * sizeof(double);
  auto kern = k_lu_slab<SW, PW, RPT, NT>;
  if (ensure_smem(kern, smem) != cudaSuccess) return -1;
  int per_sm = 0, dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem);
  const int max_active = per_sm * sms;  // co-resident CTAs: the cooperative launch's ceiling
  const int G = nb.T / SW;
  const int groups = std::min(nb.count, max_active / G);
  if (groups < 1) return -1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(groups * G);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // slabs of a node wait on each other
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, nb, H, hs, write_h ? 1 : 0, sync, err, groups) == cudaSuccess ? 0 : -2;
}

}  // namespace

// W = 32 while a 32-column slab fits (T <= 800: configs 1-4), else 16 (T <= 1600).
int slab_width(const NodeBatch& nb) {
  const char* e = std::getenv("KS_SLAB_W");  // 16: force 16-column slabs where they fit
  if (e && std::atoi(e) == 16 && nb.T % 16 == 0 && nb.t_pad <= 1024 && (size_t)(nb.T + 16) * 17 * 8 <= 212 * 1024)
    return 16;
  if (nb.T % 32 == 0 && nb.t_pad <= 512 && (size_t)(nb.T + 32) * 33 * 8 <= 212 * 1024) return 32;
  if (nb.T % 16 == 0 && nb.t_pad <= 1024 && (size_t)(nb.T + 16) * 17 * 8 <= 212 * 1024) return 16;
  return 0;
}

static long long* slab_ts_buf() {
  static long long* p = nullptr;
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("KS_SLAB_TRACE");
    on = (e && e[0] == '1') ? 1 : 0;
    if (on) {
      cudaMalloc(&p, sizeof(long long) * kTsSlabs * kTsSteps * 4);
      cudaMemset(p, 0, sizeof(long long) * kTsSlabs * kTsSteps * 4);
      cudaMemcpyToSymbol(g_slab_ts, &p, sizeof(p));
    }
  }
  return p;
}

int launch_lu_slab(const NodeBatch& nb, double* H, int64_t h_stride, bool write_h, unsigned* sync, unsigned* err,
                   cudaStream_t st) {
  slab_ts_buf();
  const int w = slab_width(nb);
  const char* e = std::getenv("KS_SLAB_PW");  // 32: one 32-column panel per slab step
  const bool pw32 = e && std::atoi(e) == 32;
  if (w == 32) return pw32 ? launch_slab_t<32, 32, 1>(nb, H, h_stride, write_h, sync, err, st)
                           : launch_slab_t<32, 16, 1>(nb, H, h_stride, write_h, sync, err, st);
  if (w == 16) return nb.t_pad <= 512 ? launch_slab_t<16, 16, 1>(nb, H, h_stride, write_h, sync, err, st)
                                      : launch_slab_t<16, 16, 2>(nb, H, h_stride, write_h, sync, err, st);
  return -1;
}

}  // namespace ks

#include "../../include/invaskit_probe.h"

// Probe hook: copies the stamps of the last traced level (KS_SLAB_TRACE=1).
extern "C" int ks_slab_trace(long long* out, int64_t cap) {
  long long* p = ks::slab_ts_buf();
  if (!p) return 0;
  const int64_t n = std::min<int64_t>(cap, (int64_t)ks::kTsSlabs * ks::kTsSteps * 4);
  cudaMemcpy(out, p, sizeof(long long) * n, cudaMemcpyDeviceToHost);
  return (int)n;
}
