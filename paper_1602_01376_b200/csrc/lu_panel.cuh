// Column loop of a W-column LU panel with partial pivoting (linalg.py:199-213),
// shared by the per-launch panel kernel (k_lu_panel2) and the persistent
// per-node LU (k_lu_slab, lu_slab.cu).
//
// The panel's candidate rows live in registers: thread t holds physical rows
// t + i*NT (i < RPT). Rows never move inside the loop; each thread tracks its
// rows' LOGICAL positions (the reference's swap sequence, swaps[k] = p). The
// per-column critical path is what bounds the top levels of the tree, so the
// step is arranged to keep it short:
//   * pivot search on a 32-bit key (hi word of |v| + 1; 0 = not a candidate):
//     one redux + one ballot decide a warp's (and then the CTA's) winner unless
//     two keys tie on the hi word, when the low word and then the logical
//     position decide (np.argmax: first occurrence);
//   * every thread starts 1/a[k] for its best candidate before the search, so
//     the winner publishes the pivot's reciprocal with its key and row; the
//     division overlaps the reduction instead of following the barrier;
//   * one barrier per column (records double-buffered by column parity).
// Multipliers are a * (1/pivot) (the reciprocal correctly rounded). The
// caller must synchronize before reading ps.urcp.
#pragma once

#include "common.cuh"

namespace ks {

struct __align__(16) PivRec {
  unsigned hi, lo;
  int pos, pad;
  double rcp, pad2;
};

template <int NW, int W>
struct PanelShared {
  double cand[2][NW][W];  // per-warp candidate pivot rows, by column parity
  PivRec rec[2][NW];      // per-warp winner records
  double urcp[W];         // 1 / pivot of each column (for rows eliminated later)
};

// winner lane of a warp for (key hi, lo, logical position): max hi, then max
// lo, then min position
__device__ __forceinline__ int warp_winner3(unsigned h, unsigned l, int p) {
  const unsigned mh = __reduce_max_sync(0xffffffffu, h);
  const unsigned m = __ballot_sync(0xffffffffu, h == mh);
  if (__popc(m) == 1) return __ffs(m) - 1;
  const unsigned ml = __reduce_max_sync(0xffffffffu, h == mh ? l : 0u);
  const bool t = (h == mh && l == ml);
  const unsigned mp = __reduce_min_sync(0xffffffffu, t ? (unsigned)p : 0x7fffffffu);
  return __ffs(__ballot_sync(0xffffffffu, t && (unsigned)p == mp)) - 1;
}

// Eliminates columns [0, W) of the register panel. Finished CB-column blocks
// of physical row r go to fbase[r * fstride + kb + j] (shared memory).
// piv[kk] = piv_base + logical pivot position; *info = info_base + kk + 1 at
// the first zero pivot column (SingularMatrixError, linalg.py:205-206).
// Only the first nact warps (those holding candidate rows) take part; they
// synchronize on named barrier 1. The caller skips the call on the others and
// synchronizes the whole CTA afterwards.
__device__ __forceinline__ int panel_warps(int rows, int nt) { return (min(rows, nt) + 31) / 32; }

template <int W, int RPT, int NT, int CB = 4>
__device__ __forceinline__ void panel_columns(double (&a)[RPT][W], int (&pos)[RPT], bool (&done)[RPT],
                                              PanelShared<NT / 32, W>& ps, double* fbase, int fstride, int rows,
                                              int* piv, int piv_base, int* info, int info_base, int nact) {
  constexpr int NW = NT / 32;
  constexpr int NONE = 0x7fffffff;
  static_assert(NW <= 32 && W % CB == 0 && W <= 32, "panel shape");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int my_piv = 0, first_sing = -1;
  double my_rcp = 0.0;
#pragma unroll 1
  for (int kb = 0; kb < W; kb += CB) {
#pragma unroll
    for (int c = 0; c < CB; ++c) {
      const int kk = kb + c;
      const int buf = c & 1;
      // 1) this thread's best candidate and its reciprocal (started early)
      unsigned bh = 0u, bl = 0u;
      int bp = NONE, bi = -1;
      double bvv = 1.0;
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const double v = fabs(a[i][c]);
        const unsigned h = (unsigned)__double2hiint(v) + 1u, l = (unsigned)__double2loint(v);
        if (!done[i] && (h > bh || (h == bh && (l > bl || (l == bl && pos[i] < bp))))) {
          bh = h; bl = l; bp = pos[i]; bi = i; bvv = a[i][c];
        }
      }
      const double rc = 1.0 / bvv;
      // 2) the warp's winner publishes its row, key and reciprocal
      const int wl = warp_winner3(bh, bl, bp);
      if (lane == wl) {
#pragma unroll
        for (int i = 0; i < RPT; ++i)
          if (i == bi) {
#pragma unroll
            for (int j = c + 1; j < W; ++j) ps.cand[buf][warp][j] = a[i][j];
          }
        PivRec q;
        q.hi = bh; q.lo = bl; q.pos = bp; q.pad = 0; q.rcp = rc; q.pad2 = 0.0;
        ps.rec[buf][warp] = q;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(nact * 32) : "memory");
      // 3) the CTA's winner (every warp redundantly)
      unsigned qh = 0u, ql = 0u;
      int qp = NONE;
      double qr = 0.0;
      if (lane < nact) {
        const PivRec& q = ps.rec[buf][lane];
        qh = q.hi; ql = q.lo; qp = q.pos; qr = q.rcp;
      }
      const int ww = warp_winner3(qh, ql, qp);
      const int bpos = __shfl_sync(0xffffffffu, qp, ww);
      const double rcp = __shfl_sync(0xffffffffu, qr, ww);
      // |pivot| == 0 (or NaN) <=> 1/pivot is not finite: the reference raises
      // SingularMatrixError; all keys then tie and the winner is the row at
      // logical position kk. (A subnormal pivot below 2^-1024 counts too.)
      const bool singular = !(fabs(rcp) < INFINITY);
      // the column's outputs stay in registers until the loop ends (lane kk%32
      // of every warp keeps them), off the per-column critical path
      if (lane == (kk & 31)) { my_piv = bpos; my_rcp = rcp; }
      if (singular && first_sing < 0) first_sing = kk;
      // 4) logical swap kk <-> bpos; eliminate the other candidates
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const bool cd = !done[i];
        const bool is_piv = cd && pos[i] == bpos;
        if (cd) pos[i] = is_piv ? kk : (pos[i] == kk ? bpos : pos[i]);
        done[i] = done[i] || is_piv;
        if (cd && !is_piv && !singular) {
          const double l = a[i][c] * rcp;
          a[i][c] = l;
#pragma unroll
          for (int j = c + 1; j < W; ++j) a[i][j] = fma(-l, ps.cand[buf][ww][j], a[i][j]);
        }
      }
    }
    // block finished: flush its CB columns, shift the register window
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int r = threadIdx.x + i * NT;
      if (r < rows) {
#pragma unroll
        for (int j = 0; j < CB; ++j) fbase[r * fstride + kb + j] = a[i][j];
      }
#pragma unroll
      for (int j = 0; j < W; ++j) a[i][j] = (j + CB < W) ? a[i][j + CB] : 0.0;
    }
  }
  // W <= 32: warp 0's lanes hold the columns' pivots and reciprocals
  if (warp == 0 && lane < W) {
    piv[lane] = piv_base + my_piv;
    ps.urcp[lane] = my_rcp;
  }
  if (threadIdx.x == 0 && first_sing >= 0 && *info == 0) *info = info_base + first_sing + 1;
}

}  // namespace ks
