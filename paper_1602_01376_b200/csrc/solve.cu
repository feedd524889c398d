// ks_solve (+ the sharded solve phases) and ks_matvec: the O(N) telescoping
// solve on the stored factors (solver.py:192-237 restated) and the
// compressed operator (compress.py:352-411). Every call runs in a workspace of
// its own (SolveWs), so concurrent calls on one handle are safe.
#include "handle.h"

using namespace ksr;

namespace {

// ---- per-call workspaces ----
// Idle workspaces are reused first by the same stream (no wait), then any whose
// last use has completed; otherwise, up to kMaxIdleWs workspaces are created,
// and beyond that the call waits (on the device) for the least recently
// released one. A workspace is never shared by two calls in flight on the host.
constexpr size_t kMaxIdleWs = 4;

int ws_fit(ks_factor* f, SolveWs* w, int64_t q) {
  if (q <= w->q_cap) return KS_OK;
  if (w->done) KS_CUDA(cudaEventSynchronize(w->done));
  w->z.release(); w->c.release(); w->tin.release(); w->y.release(); w->wtmp.release(); w->bdev.release();
  w->xdev.release();
  KS_CUDA(w->z.alloc((size_t)f->leaf_nodes.size() * f->m_pad * q));
  KS_CUDA(w->c.alloc((size_t)std::max<int64_t>(f->n_nodes * f->s_pad * q, 1)));
  KS_CUDA(w->tin.alloc((size_t)std::max<int64_t>(f->n_nodes * f->s_pad * q, 1)));
  KS_CUDA(w->y.alloc((size_t)std::max<int64_t>((int64_t)f->n_int * f->zt * q, 1)));
  KS_CUDA(w->wtmp.alloc((size_t)std::max<int64_t>((int64_t)f->n_int * f->zt * q, 1)));
  KS_CUDA(w->bdev.alloc((size_t)f->n * q));
  KS_CUDA(w->xdev.alloc((size_t)f->n * q));
  w->q_cap = q;
  return KS_OK;
}

int ws_acquire(ks_factor* f, int64_t q, cudaStream_t st, SolveWs** out) {
  SolveWs* w = nullptr;
  {
    std::lock_guard<std::mutex> lk(f->ws_mu);
    SolveWs* any = nullptr;
    for (auto& u : f->ws) {
      if (u->busy || u.get() == f->shard_ws) continue;
      if (u->last == st) { w = u.get(); break; }
      if (!any && (!u->done || cudaEventQuery(u->done) == cudaSuccess)) any = u.get();
    }
    if (!w) w = any;
    if (!w) {
      size_t idle = 0;
      for (auto& u : f->ws) idle += (!u->busy && u.get() != f->shard_ws);
      if (idle >= kMaxIdleWs) {
        for (auto& u : f->ws)
          if (!u->busy && u.get() != f->shard_ws) { w = u.get(); break; }
      } else {
        f->ws.emplace_back(new SolveWs());
        w = f->ws.back().get();
      }
    }
    w->busy = true;
  }
  int rc = KS_OK;
  if (!w->done) {
    cudaError_t e = cudaEventCreateWithFlags(&w->done, cudaEventDisableTiming);
    if (e != cudaSuccess) rc = fail(KS_ERR_CUDA, "workspace event: %s", cudaGetErrorString(e));
  } else if (w->last != st) {
    cudaError_t e = cudaStreamWaitEvent(st, w->done, 0);  // its previous user's work on another stream
    if (e != cudaSuccess) rc = fail(KS_ERR_CUDA, "workspace wait: %s", cudaGetErrorString(e));
  }
  if (!rc) rc = ws_fit(f, w, q);
  if (rc) {
    std::lock_guard<std::mutex> lk(f->ws_mu);
    w->busy = false;
    return rc;
  }
  w->launches = 0;
  *out = w;
  return KS_OK;
}

void ws_release(ks_factor* f, SolveWs* w, cudaStream_t st) {
  cudaEventRecord(w->done, st);
  std::lock_guard<std::mutex> lk(f->ws_mu);
  w->last = st;
  w->busy = false;
  f->last_ws = w;
  f->launches[1] = w->launches.load();
}

// the sharded solve phases keep one workspace across ks_solve_up / top / down
int shard_ws(ks_factor* f, int64_t q, SolveWs** out) {
  {
    std::lock_guard<std::mutex> lk(f->ws_mu);
    if (!f->shard_ws) {
      f->ws.emplace_back(new SolveWs());
      f->shard_ws = f->ws.back().get();
    }
  }
  if (int rc = ws_fit(f, f->shard_ws, q)) return rc;
  f->last_ws = f->shard_ws;
  *out = f->shard_ws;
  return KS_OK;
}

// ---- multi-RHS path (q >= kGemmSolveQ): factors applied as DMMA GEMMs ----
constexpr int64_t kGemmSolveQ = 8;

// op(T)^-1 B for an n x n triangle T (ld lda, batch stride sa) and B (n x ncols,
// ld ldb, batch stride sb): recursive halves, GEMM for the off-diagonal block,
// k_trsm_rhs at 8/16/32/64.
static int gemm_trsm(Launcher& L, bool upper, bool unit, const double* A, int64_t lda, int64_t sa, double* B,
                     int64_t ldb, int64_t sb, int n, int ncols, int batch) {
  if (n == 64 || n == 32 || n == 16 || n == 8) {
    ks::launch_trsm_rhs(n, upper, unit, A, lda, sa, B, ldb, sb, ncols, batch, L.st);
    ++*L.count;
    return L.check("trsm_rhs");
  }
  const int h = (n > 64) ? (int)roundup(n / 2, 8) : (n > 32 ? 32 : (n > 16 ? 16 : 8));
  int rc;
  if (!upper) {
    if ((rc = gemm_trsm(L, upper, unit, A, lda, sa, B, ldb, sb, h, ncols, batch))) return rc;
    rc = L.gemm(mk(n - h, ncols, h, batch, Operand{A + (int64_t)h * lda, lda, sa, nullptr}, Operand{B, ldb, sb, nullptr},
                   OperandW{B + (int64_t)h * ldb, ldb, sb, nullptr}, -1.0, 1.0), false, false);
    if (rc) return rc;
    return gemm_trsm(L, upper, unit, A + (int64_t)h * lda + h, lda, sa, B + (int64_t)h * ldb, ldb, sb, n - h, ncols,
                     batch);
  }
  if ((rc = gemm_trsm(L, upper, unit, A + (int64_t)h * lda + h, lda, sa, B + (int64_t)h * ldb, ldb, sb, n - h, ncols,
                      batch)))
    return rc;
  rc = L.gemm(mk(h, ncols, n - h, batch, Operand{A + h, lda, sa, nullptr}, Operand{B + (int64_t)h * ldb, ldb, sb, nullptr},
                 OperandW{B, ldb, sb, nullptr}, -1.0, 1.0), false, false);
  if (rc) return rc;
  return gemm_trsm(L, upper, unit, A, lda, sa, B, ldb, sb, h, ncols, batch);
}

// Leaf triangular solves on q right-hand sides, recursively by row halves so
// the off-diagonal updates are large GEMMs (rows [r0+h, r0+n) against the
// solved half) instead of 64-row strips; 64-row diagonal blocks go through
// their stored inverses (inv, from the leaf factorization).
static int leaf_fwd_rec(ks_factor* f, SolveWs* w, Launcher& L, int r0, int n, int q) {
  const int nl = (int)f->leaf_nodes.size(), M = f->m_pad;
  const int64_t AS = (int64_t)f->R * M, ZS = (int64_t)M * q;
  if (n == 64)
    return L.gemm(mk(64, q, 64, nl, Operand{f->inv.p + (int64_t)(r0 / 64) * 4096, 64, (int64_t)M * 64, nullptr},
                     Operand{w->z.p + (int64_t)r0 * q, q, ZS, nullptr}, OperandW{w->z.p + (int64_t)r0 * q, q, ZS, nullptr},
                     1.0, 0.0), false, false);
  const int h = (int)roundup(n / 2, 64);
  if (int rc = leaf_fwd_rec(f, w, L, r0, h, q)) return rc;
  // z[r0+h, r0+n) -= L[r0+h : r0+n, r0 : r0+h] z[r0, r0+h)
  if (int rc = L.gemm(mk(n - h, q, h, nl, Operand{f->leafA.p + (int64_t)(r0 + h) * M + r0, M, AS, nullptr},
                         Operand{w->z.p + (int64_t)r0 * q, q, ZS, nullptr},
                         OperandW{w->z.p + (int64_t)(r0 + h) * q, q, ZS, nullptr}, -1.0, 1.0), false, false))
    return rc;
  return leaf_fwd_rec(f, w, L, r0 + h, n - h, q);
}

static int leaf_bwd_rec(ks_factor* f, SolveWs* w, Launcher& L, int r0, int n, int q) {
  const int nl = (int)f->leaf_nodes.size(), M = f->m_pad;
  const int64_t AS = (int64_t)f->R * M, ZS = (int64_t)M * q;
  if (n == 64)
    return L.gemm(mk(64, q, 64, nl, Operand{f->inv.p + (int64_t)(r0 / 64) * 4096, 64, (int64_t)M * 64, nullptr},
                     Operand{w->z.p + (int64_t)r0 * q, q, ZS, nullptr}, OperandW{w->z.p + (int64_t)r0 * q, q, ZS, nullptr},
                     1.0, 0.0), true, false);
  const int h = (int)roundup(n / 2, 64);
  if (int rc = leaf_bwd_rec(f, w, L, r0 + h, n - h, q)) return rc;
  // z[r0, r0+h) -= L[r0+h : r0+n, r0 : r0+h]^T z[r0+h, r0+n)
  if (int rc = L.gemm(mk(h, q, n - h, nl, Operand{f->leafA.p + (int64_t)(r0 + h) * M + r0, M, AS, nullptr},
                         Operand{w->z.p + (int64_t)(r0 + h) * q, q, ZS, nullptr},
                         OperandW{w->z.p + (int64_t)r0 * q, q, ZS, nullptr}, -1.0, 1.0), true, false))
    return rc;
  return leaf_bwd_rec(f, w, L, r0, h, q);
}

// up pass at the leaves: z = L^-1 b, c = L21 z
static int leaf_up_gemm(ks_factor* f, SolveWs* w, Launcher& L, const double* Bd, int q) {
  const ks::LeafBatch lb = f->leafbatch();
  const int nl = lb.count, M = f->m_pad, S = f->s_pad;
  const int64_t AS = lb.a_stride, ZS = (int64_t)M * q;
  ks::launch_leaf_gather(lb, Bd, q, w->z.p, q, L.st);
  ++*L.count;
  if (int rc = leaf_fwd_rec(f, w, L, 0, M, q)) return rc;
  if (S > 0 && f->n_nodes > 1)
    return L.gemm(mk(S, q, M, nl, Operand{f->leafA.p + (int64_t)M * M, M, AS, nullptr}, Operand{w->z.p, q, ZS, nullptr},
                     OperandW{w->c.p, q, (int64_t)S * q, lb.node}, 1.0, 0.0), false, false);
  return KS_OK;
}

// down pass at the leaves: x = L^-T (z - L21^T t)
static int leaf_down_gemm(ks_factor* f, SolveWs* w, Launcher& L, double* Xd, int q) {
  const ks::LeafBatch lb = f->leafbatch();
  const int nl = lb.count, M = f->m_pad, S = f->s_pad;
  const int64_t AS = lb.a_stride, ZS = (int64_t)M * q;
  if (S > 0 && f->n_nodes > 1) {
    if (int rc = L.gemm(mk(M, q, S, nl, Operand{f->leafA.p + (int64_t)M * M, M, AS, nullptr},
                           Operand{w->tin.p, q, (int64_t)S * q, lb.node}, OperandW{w->z.p, q, ZS, nullptr}, -1.0, 1.0),
                        true, false))
      return rc;
  }
  if (int rc = leaf_bwd_rec(f, w, L, 0, M, q)) return rc;
  ks::launch_leaf_scatter(lb, w->z.p, Xd, q, q, L.st);
  ++*L.count;
  return KS_OK;
}

// up pass at one level (block formulation, kernels.cuh NodeBatch):
//   r1 = B c_r (kept in y's first half), r2 = B^T c_l - Y r1, y2 = L^-1 Pi r2,
//   c = P cc - (P_l H_l) r1 + L21 y2
static int node_up_gemm(ks_factor* f, SolveWs* w, Launcher& L, const ks::NodeBatch& nb, bool root, int q) {
  const int S = nb.s_pad, T = nb.T, ZT = nb.zt, cnt = nb.count;
  const int64_t SS = (int64_t)S * S, XS = 2 * SS, TT = (int64_t)T * T, CS = (int64_t)S * q, YS = (int64_t)ZT * q;
  const int64_t PS = (int64_t)S * ZT;
  double* wv = w->wtmp.p + (int64_t)nb.first * YS;
  double* y = w->y.p + (int64_t)nb.first * YS;
  double* r1 = y;
  double* y2 = y + (int64_t)S * q;
  int rc = L.gemm(mk(S, q, S, cnt, Operand{nb.Bc, S, SS, nullptr}, Operand{w->c.p, q, CS, nb.right},
                     OperandW{r1, q, YS, nullptr}, 1.0, 0.0), false, false);
  if (rc) return rc;
  rc = L.gemm(mk(S, q, S, cnt, Operand{nb.Bc, S, SS, nullptr}, Operand{w->c.p, q, CS, nb.left},
                 OperandW{wv + (int64_t)S * q, q, YS, nullptr}, 1.0, 0.0), true, false);
  if (rc) return rc;
  rc = L.gemm(mk(S, q, S, cnt, Operand{nb.XY + SS, S, XS, nullptr}, Operand{r1, q, YS, nullptr},
                 OperandW{wv + (int64_t)S * q, q, YS, nullptr}, -1.0, 1.0), false, false);
  if (rc) return rc;
  ks::launch_permute_rows(nb, w->wtmp.p, w->y.p, q, L.st);
  ++*L.count;
  if ((rc = gemm_trsm(L, false, true, nb.Aug, T, TT, y2, q, YS, S, q, cnt))) return rc;
  if (root) return KS_OK;
  rc = L.gemm(mk(S, q, S, cnt, Operand{nb.Pn, ZT, PS, nullptr}, Operand{w->c.p, q, CS, nb.left},
                 OperandW{w->c.p, q, CS, nb.node}, 1.0, 0.0), false, false);
  if (rc) return rc;
  rc = L.gemm(mk(S, q, S, cnt, Operand{nb.Pn + S, ZT, PS, nullptr}, Operand{w->c.p, q, CS, nb.right},
                 OperandW{w->c.p, q, CS, nb.node}, 1.0, 1.0), false, false);
  if (rc) return rc;
  rc = L.gemm(mk(S, q, S, cnt, Operand{nb.PHl, S, SS, nullptr}, Operand{r1, q, YS, nullptr},
                 OperandW{w->c.p, q, CS, nb.node}, -1.0, 1.0), false, false);
  if (rc) return rc;
  return L.gemm(mk(S, q, S, cnt, Operand{nb.Aug + (int64_t)S * T, T, TT, nullptr}, Operand{y2, q, YS, nullptr},
                   OperandW{w->c.p, q, CS, nb.node}, 1.0, 1.0), false, false);
}

// down pass at one level: y2 += U12 t, r1 += P_l^T t (not at the root);
// w2 = U^-1 y2, w1 = r1 - X w2; the children receive w1 and w2
static int node_down_gemm(ks_factor* f, SolveWs* w, Launcher& L, const ks::NodeBatch& nb, bool root, int q) {
  const int S = nb.s_pad, T = nb.T, ZT = nb.zt, cnt = nb.count;
  const int64_t SS = (int64_t)S * S, XS = 2 * SS, TT = (int64_t)T * T, CS = (int64_t)S * q, YS = (int64_t)ZT * q;
  const int64_t PS = (int64_t)S * ZT;
  double* y = w->y.p + (int64_t)nb.first * YS;
  double* r1 = y;
  double* y2 = y + (int64_t)S * q;
  int rc;
  if (!root) {
    rc = L.gemm(mk(S, q, S, cnt, Operand{nb.Aug + S, T, TT, nullptr}, Operand{w->tin.p, q, CS, nb.node},
                   OperandW{y2, q, YS, nullptr}, 1.0, 1.0), false, false);
    if (rc) return rc;
    rc = L.gemm(mk(S, q, S, cnt, Operand{nb.Pn, ZT, PS, nullptr}, Operand{w->tin.p, q, CS, nb.node},
                   OperandW{r1, q, YS, nullptr}, 1.0, 1.0), true, false);
    if (rc) return rc;
  }
  if ((rc = gemm_trsm(L, true, false, nb.Aug, T, TT, y2, q, YS, S, q, cnt))) return rc;
  rc = L.gemm(mk(S, q, S, cnt, Operand{nb.XY, S, XS, nullptr}, Operand{y2, q, YS, nullptr},
                 OperandW{r1, q, YS, nullptr}, -1.0, 1.0), false, false);
  if (rc) return rc;
  ks::launch_split_u(nb, w->y.p, w->tin.p, q, L.st);
  ++*L.count;
  return KS_OK;
}

// LU-fallback leaves overwrite their Cholesky-path results (c at the leaf, x rows)
static int fb_up(ks_factor* f, SolveWs* w, const double* Bd, int64_t q, cudaStream_t st) {
  if (f->fb_leaf.empty()) return KS_OK;
  const size_t need = f->fb_leaf.size() * (size_t)f->m_pad * q;
  if (w->fb_y.n < need) {
    w->fb_y.release();
    KS_CUDA(w->fb_y.alloc(need));
  }
  ks::launch_fb_up(f->fb_batch(), f->fb_begin.p, f->fb_size.p, Bd, q, w->fb_y.p, w->c.p, (int)q, st);
  KS_CUDA(cudaGetLastError());
  return KS_OK;
}

static int fb_down(ks_factor* f, SolveWs* w, double* Xd, int64_t q, cudaStream_t st) {
  if (f->fb_leaf.empty()) return KS_OK;
  ks::launch_fb_down(f->fb_batch(), f->fb_begin.p, f->fb_size.p, w->fb_y.p, w->tin.p, Xd, q, (int)q, f->n_nodes > 1,
                     st);
  KS_CUDA(cudaGetLastError());
  return KS_OK;
}

static void trace_mark(ks_factor* f, cudaStream_t st, const char* what) {
  if (!trace_on()) return;
  std::atomic<int64_t> none{0};
  Launcher L{f, st, &none};
  L.check(what);
}

static void trace_build_report(ks_factor* f) {
  if (!trace_on() || f->trace_n < 2) return;
  cudaDeviceSynchronize();
  std::vector<std::pair<std::string, std::pair<int, double>>> agg;
  for (int i = 1; i < f->trace_n; ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, f->trace_ev[i - 1], f->trace_ev[i]);
    std::string nm = (f->trace_tag[i] < 0 ? std::string("leaf ") : "L" + std::to_string(f->trace_tag[i]) + " ") +
                     f->trace_name[i];
    bool found = false;
    for (auto& a : agg)
      if (a.first == nm) { a.second.first++; a.second.second += ms; found = true; }
    if (!found) agg.push_back({nm, {1, (double)ms}});
  }
  std::string rep;
  char line[160];
  for (auto& a : agg) {
    std::snprintf(line, sizeof line, "%-24s %5d x %10.3f ms\n", a.first.c_str(), a.second.first, a.second.second);
    rep += line;
  }
  f->trace_report = rep;
}

// Solve phases. Shard-local rows are [loc_begin, loc_end) of tree order; the
// kernels index B and X by absolute tree position, so local buffers are passed
// with a virtual base (ptr - loc_begin * q).
static int solve_up(ks_factor* f, SolveWs* w, const double* Bd, int64_t q, cudaStream_t st) {
  if (q >= kGemmSolveQ && (q & 1) == 0) {  // DMMA tiles need an even q
    Launcher L{f, st, &w->launches};
    if (int rc = leaf_up_gemm(f, w, L, Bd, (int)q)) return rc;
    if (int rc = fb_up(f, w, Bd, q, st)) return rc;
    for (int lev = 0; lev < f->n_local_levels; ++lev)
      if (int rc = node_up_gemm(f, w, L, f->nodebatch(lev), f->levels[lev][0] == 0, (int)q)) return rc;
    KS_CUDA(cudaGetLastError());
    return KS_OK;
  }
  ks::SolveBufs sb{(int)q, w->z.p, w->c.p, w->tin.p, w->y.p};
  f->cur_tag = -1;
  trace_mark(f, st, "start");
  ks::launch_leaf_fwd(f->leafbatch(), Bd, q, sb, st);
  if (int rc = fb_up(f, w, Bd, q, st)) return rc;
  ++w->launches;
  trace_mark(f, st, "leaf_fwd");
  for (int lev = 0; lev < f->n_local_levels; ++lev) {
    f->cur_tag = lev;
    ks::launch_node_up(f->nodebatch(lev), sb, f->levels[lev][0] == 0, st);
    ++w->launches;
    trace_mark(f, st, "node_up");
  }
  KS_CUDA(cudaGetLastError());
  return KS_OK;
}

static int solve_top(ks_factor* f, SolveWs* w, int64_t q, cudaStream_t st) {
  if (q >= kGemmSolveQ && (q & 1) == 0) {  // DMMA tiles need an even q
    Launcher L{f, st, &w->launches};
    const int nlev = (int)f->levels.size();
    for (int lev = f->n_local_levels; lev < nlev; ++lev)
      if (int rc = node_up_gemm(f, w, L, f->nodebatch(lev), f->levels[lev][0] == 0, (int)q)) return rc;
    for (int lev = nlev - 1; lev >= f->n_local_levels; --lev)
      if (int rc = node_down_gemm(f, w, L, f->nodebatch(lev), f->levels[lev][0] == 0, (int)q)) return rc;
    KS_CUDA(cudaGetLastError());
    return KS_OK;
  }
  ks::SolveBufs sb{(int)q, w->z.p, w->c.p, w->tin.p, w->y.p};
  const int nlev = (int)f->levels.size();
  for (int lev = f->n_local_levels; lev < nlev; ++lev) {
    ks::launch_node_up(f->nodebatch(lev), sb, f->levels[lev][0] == 0, st);
    ++w->launches;
  }
  for (int lev = nlev - 1; lev >= f->n_local_levels; --lev) {
    f->cur_tag = lev;
    ks::launch_node_down(f->nodebatch(lev), sb, f->levels[lev][0] == 0, st);
    ++w->launches;
    trace_mark(f, st, "node_down");
  }
  KS_CUDA(cudaGetLastError());
  return KS_OK;
}

static int solve_down(ks_factor* f, SolveWs* w, double* Xd, int64_t q, cudaStream_t st) {
  if (q >= kGemmSolveQ && (q & 1) == 0) {  // DMMA tiles need an even q
    Launcher L{f, st, &w->launches};
    for (int lev = f->n_local_levels - 1; lev >= 0; --lev)
      if (int rc = node_down_gemm(f, w, L, f->nodebatch(lev), f->levels[lev][0] == 0, (int)q)) return rc;
    if (int rc = leaf_down_gemm(f, w, L, Xd, (int)q)) return rc;
    if (int rc = fb_down(f, w, Xd, q, st)) return rc;
    KS_CUDA(cudaGetLastError());
    return KS_OK;
  }
  ks::SolveBufs sb{(int)q, w->z.p, w->c.p, w->tin.p, w->y.p};
  for (int lev = f->n_local_levels - 1; lev >= 0; --lev) {
    f->cur_tag = lev;
    ks::launch_node_down(f->nodebatch(lev), sb, f->levels[lev][0] == 0, st);
    ++w->launches;
    trace_mark(f, st, "node_down");
  }
  f->cur_tag = -1;
  ks::launch_leaf_bwd(f->leafbatch(), Xd, q, sb, f->n_nodes > 1, st);
  if (int rc = fb_down(f, w, Xd, q, st)) return rc;
  ++w->launches;
  trace_mark(f, st, "leaf_bwd");
  KS_CUDA(cudaGetLastError());
  return KS_OK;
}


}  // namespace

extern "C" {

int ks_solve(ks_factor* f, const double* B, double* X, int64_t q, void* stream) {
  if (!f) return fail(KS_ERR_INVALID, "null handle");
  if (!f->factored) return fail(KS_ERR_INVALID, "handle is not factored");
  if (f->shard_root != 0) return fail(KS_ERR_INVALID, "sharded handle: use ks_solve_up / ks_solve_top / ks_solve_down");
  if (q < 0) return fail(KS_ERR_INVALID, "q must be >= 0");
  if (q == 0) return KS_OK;
  if (!B || !X) return fail(KS_ERR_INVALID, "null B or X");
  KS_CUDA(cudaSetDevice(f->device));
  cudaStream_t st = (cudaStream_t)stream;
  SolveWs* w = nullptr;
  if (int rc = ws_acquire(f, q, st, &w)) return rc;
  if (trace_on()) f->trace_n = 0;
  PhaseTimer tm(f->profiling, st, 2);
  tm.mark(0);
  const bool bdev = is_device_ptr(B), xdev = is_device_ptr(X);
  const double* Bd = B;
  double* Xd = X;
  const size_t bytes = (size_t)f->n * q * sizeof(double);
  auto run = [&]() -> int {
    if (!bdev) {
      KS_CUDA(cudaMemcpyAsync(w->bdev.p, B, bytes, cudaMemcpyHostToDevice, st));
      Bd = w->bdev.p;
    }
    if (!xdev) Xd = w->xdev.p;
    if (int rc = solve_up(f, w, Bd, q, st)) return rc;
    if (int rc = solve_top(f, w, q, st)) return rc;
    if (int rc = solve_down(f, w, Xd, q, st)) return rc;
    if (!xdev) KS_CUDA(cudaMemcpyAsync(X, Xd, bytes, cudaMemcpyDeviceToHost, st));
    tm.mark(1);
    return KS_OK;
  };
  const int rc = run();
  ws_release(f, w, st);
  if (rc) return rc;
  if (!xdev || !bdev) KS_CUDA(cudaStreamSynchronize(st));
  trace_build_report(f);
  if (f->profiling) {
    KS_CUDA(cudaStreamSynchronize(st));
    f->phase_ms[5] = tm.between(0, 1);
  }
  return KS_OK;
}

int ks_solve_up(ks_factor* f, const double* B_local, int64_t q, void* stream) {
  if (!f || !f->local_factored) return fail(KS_ERR_INVALID, "shard is not factored");
  if (q <= 0 || !B_local) return fail(KS_ERR_INVALID, "need q >= 1 and a device B");
  KS_CUDA(cudaSetDevice(f->device));
  SolveWs* w = nullptr;
  if (int rc = shard_ws(f, q, &w)) return rc;
  w->launches = 0;
  const int rc = solve_up(f, w, B_local - f->loc_begin * q, q, (cudaStream_t)stream);
  f->launches[1] = w->launches.load();
  return rc;
}

int ks_solve_top(ks_factor* f, int64_t q, void* stream) {
  if (!f || !f->factored) return fail(KS_ERR_INVALID, "handle is not factored (ks_factorize_top)");
  SolveWs* w = f->shard_ws;
  if (q <= 0 || !w || q > w->q_cap) return fail(KS_ERR_INVALID, "ks_solve_top needs q >= 1 and a prior ks_solve_up with the same q");
  KS_CUDA(cudaSetDevice(f->device));
  return solve_top(f, w, q, (cudaStream_t)stream);
}

int ks_solve_down(ks_factor* f, double* X_local, int64_t q, void* stream) {
  if (!f || !f->factored) return fail(KS_ERR_INVALID, "handle is not factored");
  if (q <= 0 || !X_local) return fail(KS_ERR_INVALID, "need q >= 1 and a device X");
  SolveWs* w = f->shard_ws;
  if (!w || q > w->q_cap) return fail(KS_ERR_INVALID, "ks_solve_down needs a prior ks_solve_up with the same q");
  KS_CUDA(cudaSetDevice(f->device));
  return solve_down(f, w, X_local - f->loc_begin * q, q, (cudaStream_t)stream);
}

// Skeleton-sized exchange buffers of one node (device pointers): 0 = H
// (s_pad x s_pad), 1 = c (up-pass skeleton weights, s_pad x q), 2 = t (incoming
// down-pass vector, s_pad x q). dir 0 copies out of the handle, 1 into it.
int ks_node_exchange(ks_factor* f, int which, int64_t node, double* dev, int64_t q, int dir, void* stream) {
  if (!f || !dev || node < 0 || node >= f->n_nodes || which < 0 || which > 2)
    return fail(KS_ERR_INVALID, "bad exchange arguments");
  KS_CUDA(cudaSetDevice(f->device));
  double* buf;
  size_t count;
  if (which == 0) {
    buf = f->hbuf.p + node * (int64_t)f->s_pad * f->s_pad;
    count = (size_t)f->s_pad * f->s_pad;
  } else {
    SolveWs* w = f->shard_ws;
    if (!w || q <= 0 || q > w->q_cap) return fail(KS_ERR_INVALID, "solve buffers hold q <= %lld", (long long)(w ? w->q_cap : 0));
    buf = (which == 1 ? w->c.p : w->tin.p) + node * (int64_t)f->s_pad * q;
    count = (size_t)f->s_pad * q;
  }
  if (dir == 0)
    KS_CUDA(cudaMemcpyAsync(dev, buf, count * sizeof(double), cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  else
    KS_CUDA(cudaMemcpyAsync(buf, dev, count * sizeof(double), cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return KS_OK;
}

int ks_shard_info(const ks_factor* f, int64_t* out, int64_t cap) {
  // [shard_root, shard_level, loc_begin, loc_end, s_pad, n_peers, peers...]
  if (!f || !out) return fail(KS_ERR_INVALID, "null argument");
  std::vector<int64_t> v{f->shard_root, f->shard_level, f->loc_begin, f->loc_end, f->s_pad, (int64_t)f->peers.size()};
  for (int64_t p : f->peers) v.push_back(p);
  for (int64_t i = 0; i < (int64_t)v.size() && i < cap; ++i) out[i] = v[i];
  return (int)v.size();
}

// Y = K~ W, the compressed operator (hss_matvec, compress.py:352-411), on the
// handle's resident inputs and coupling blocks (needs a factorized handle).
int ks_matvec(ks_factor* f, const double* W, double* Y, int64_t q, void* stream) {
  if (!f || !f->factored) return fail(KS_ERR_INVALID, "handle is not factored");
  if (f->shard_root != 0) return fail(KS_ERR_INVALID, "matvec on a sharded handle is not supported");
  if (q < 0) return fail(KS_ERR_INVALID, "q must be >= 0");
  if (q == 0) return KS_OK;
  if (!W || !Y) return fail(KS_ERR_INVALID, "null W or Y");
  KS_CUDA(cudaSetDevice(f->device));
  cudaStream_t st = (cudaStream_t)stream;
  SolveWs* w = nullptr;
  if (int rc = ws_acquire(f, q, st, &w)) return rc;
  const bool wdev = is_device_ptr(W), ydev = is_device_ptr(Y);
  auto run = [&]() -> int {
    if (q > w->mv_q) {
      w->mv_c.release(); w->mv_inc.release(); w->mv_tot.release();
      const size_t cnt = (size_t)std::max<int64_t>(f->n_nodes * f->s_pad * q, 1);
      KS_CUDA(w->mv_c.alloc(cnt));
      KS_CUDA(w->mv_inc.alloc(cnt));
      KS_CUDA(w->mv_tot.alloc(cnt));
      w->mv_q = q;
    }
    const size_t vb = (size_t)f->n_nodes * f->s_pad * q * sizeof(double);
    KS_CUDA(cudaMemsetAsync(w->mv_c.p, 0, vb, st));
    KS_CUDA(cudaMemsetAsync(w->mv_inc.p, 0, vb, st));
    KS_CUDA(cudaMemsetAsync(w->mv_tot.p, 0, vb, st));
    const size_t bytes = (size_t)f->n * q * sizeof(double);
    const double* Wd = W;
    double* Yd = Y;
    if (!wdev) {
      KS_CUDA(cudaMemcpyAsync(w->bdev.p, W, bytes, cudaMemcpyHostToDevice, st));
      Wd = w->bdev.p;
    }
    if (!ydev) Yd = w->xdev.p;
    const ks::DevTree dt = f->devtree();
    const ks::LeafBatch lb = f->leafbatch();
    const int S = f->s_pad, nlev = (int)f->levels.size();
    if (S > 0) ks::launch_mv_up_leaf(dt, lb, Wd, q, w->mv_c.p, S, (int)q, st);
    for (int lev = 0; lev < nlev; ++lev) ks::launch_mv_up_node(dt, f->nodebatch(lev), w->mv_c.p, S, (int)q, st);
    for (int lev = 0; lev < nlev; ++lev)
      ks::launch_mv_couple(dt, f->nodebatch(lev), w->mv_c.p, w->mv_inc.p, S, (int)q, st);
    for (int lev = nlev - 1; lev >= 0; --lev)
      ks::launch_mv_down(dt, f->nodebatch(lev), w->mv_inc.p, w->mv_tot.p, S, (int)q, f->levels[lev][0] != 0, st);
    ks::launch_mv_leaf(dt, lb, Wd, q, w->mv_tot.p, Yd, S, (int)q, nlev > 0, st);
    KS_CUDA(cudaGetLastError());
    if (!ydev) KS_CUDA(cudaMemcpyAsync(Y, Yd, bytes, cudaMemcpyDeviceToHost, st));
    return KS_OK;
  };
  const int rc = run();
  const int64_t keep = f->launches[1];
  ws_release(f, w, st);
  f->launches[1] = keep;  // the launch counter reports solves only
  if (rc) return rc;
  if (!ydev || !wdev) KS_CUDA(cudaStreamSynchronize(st));
  return KS_OK;
}

}  // extern "C"
