// ks_factorize / ks_factorize_top: the factorization schedule. Leaves in
// groups on their own streams (Gaussian blocks, left-looking Cholesky of the
// [[A],[P]] trapezoid, SYRK H), then the internal levels deepest first (coupling,
// augmented LU, Schur block H), condition estimates on side streams; replayed
// as a CUDA graph from the second call on (solver.py:92-189).
#include "handle.h"

using namespace ksr;

namespace {

// Enqueue the whole factorization on `st` (no host synchronization inside, so
// the sequence can be captured into a CUDA graph). Leaf Cholesky failures are
// recorded on the device and handled by the caller afterwards.
// Leaves [l0, l1): left-looking Cholesky of the (m+s) x m trapezoids in 64-column
// panels (panel update GEMM, 64x64 POTRF + inverse, panel TRSM as GEMM with the
// inverse), then H = L21 L21^T (solver.py:123-135).
// Leaves [l0, l1): K(X_leaf, X_leaf) + lam I (lower triangle) and the P rows of
// the trapezoid [[A], [P]].
// wait_p: on the first factorization, the upload milestone of these leaves' P
// blocks (the Gaussian blocks need only the points, so they start before it)
// defer_p: the P rows are copied later (enqueue_leaf_chol's split form)
static int enqueue_leaf_assemble(ks_factor* f, Launcher& L, int l0, int l1, cudaEvent_t wait_p = nullptr,
                                 bool defer_p = false) {
  if (l1 <= l0) return KS_OK;
  const ks::DevTree dt = f->devtree();
  const ks::LeafBatch all = f->leafbatch();
  ks::LeafBatch lb = all;
  lb.count = l1 - l0;
  lb.node = all.node + l0;
  lb.begin = all.begin + l0;
  lb.size = all.size + l0;
  lb.A = all.A + (int64_t)l0 * all.a_stride;
  const int M = f->m_pad;
  if ((f->d & 1) == 0) {
    // a DMMA Gram GEMM with the Gaussian epilogue
    GemmArgs g = mk(M, M, (int)f->d, lb.count, Operand{f->coords.p, f->d, f->d, lb.begin},
                    Operand{f->coords.p, f->d, f->d, lb.begin}, OperandW{lb.A, M, lb.a_stride, nullptr}, 1.0, 0.0);
    g.ge = ks::GaussEpi{f->xx.p, lb.begin, lb.size, f->lam_dev.p, f->h};
    ++L.count[0];
    cudaError_t e = (f->knobs.ablate & 8) ? cudaSuccess : ks::gemm_gauss(g, L.st);
    if (e != cudaSuccess) return fail(KS_ERR_CUDA, "leaf gauss gemm: %s", cudaGetErrorString(e));
    if (!defer_p) {
      if (wait_p) KS_CUDA(cudaStreamWaitEvent(L.st, wait_p, 0));
      ks::launch_leaf_copy_p(dt, lb, L.st);
    }
  } else {
    if (wait_p) KS_CUDA(cudaStreamWaitEvent(L.st, wait_p, 0));
    ks::launch_leaf_assemble(dt, lb, f->lam_dev.p, L.st);
  }
  L.count[0] += 1;
  return L.check("leaf_assemble");
}

// KS_UNFUSED_LEAF_TRSM=1: separate update and TRSM GEMMs per leaf panel (A/B check)

// split (the first factorization, while the leaves' P is still on its way):
// the panels factor the m x m block A alone (rows [0, m)), the P rows are
// copied in once their upload milestone wait_p has passed, and then L21 =
// P L^-T is formed panel by panel from the stored diagonal inverses (the same
// left-looking update + TRSM epilogue, on the P rows only). The Cholesky of
// every leaf then needs only the points and overlaps the upload of P.
static int enqueue_leaf_chol(ks_factor* f, Launcher& L, int l0, int l1, bool split = false,
                             cudaEvent_t wait_p = nullptr) {
  const ks::LeafBatch all = f->leafbatch();
  ks::LeafBatch lb = all;
  lb.count = l1 - l0;
  lb.node = all.node + l0;
  lb.begin = all.begin + l0;
  lb.size = all.size + l0;
  lb.A = all.A + (int64_t)l0 * all.a_stride;
  const int nl = lb.count;
  const int M = f->m_pad, S = f->s_pad, R = f->R;
  const int64_t AS = lb.a_stride;
  double* leafA = lb.A;
  double* inv = f->inv.p + (int64_t)l0 * M * 64;
  int* info = f->leaf_info.p + l0;
  cudaStream_t st = L.st;
  const bool fused = !f->knobs.unfused_leaf_trsm;
  const int R_eff = split ? M : R;  // rows the panels carry
  for (int j0 = 0; j0 < M; j0 += 64) {
    const Operand Einv{inv + (int64_t)(j0 / 64) * 64 * 64, 64, (int64_t)M * 64, nullptr};
    if (j0 > 0) {  // left-looking update of the panel (all rows, or just its diagonal block)
      Operand A{leafA + (int64_t)j0 * M, M, AS, nullptr};
      Operand B{leafA + (int64_t)j0 * M, M, AS, nullptr};
      OperandW C{leafA + (int64_t)j0 * M + j0, M, AS, nullptr};
      if (fused) {
        ++L.count[0];
        cudaError_t e = (f->knobs.ablate & 2) ? cudaSuccess : ks::gemm_small_tile(mk(64, 64, j0, nl, A, B, C, -1.0, 1.0), st);
        if (e != cudaSuccess) return fail(KS_ERR_CUDA, "leaf diagonal update: %s", cudaGetErrorString(e));
        if (int rc = L.check("leaf_update_diag")) return rc;
      } else {
        int rc = L.gemm(mk(R_eff - j0, 64, j0, nl, A, B, C, -1.0, 1.0), false, true, "leaf_update");
        if (rc) return rc;
      }
    }
    if (!(f->knobs.ablate & 1)) ks::launch_potrf64(lb, j0, inv, info, st);
    ++L.count[0];
    if (int rc = L.check("potrf64")) return rc;
    if (R_eff - j0 - 64 > 0) {
      OperandW C{leafA + (int64_t)(j0 + 64) * M + j0, M, AS, nullptr};
      if (fused && j0 > 0) {
        // rows below the diagonal block: update and TRSM (x L_jj^-T) in one GEMM
        Operand A{leafA + (int64_t)(j0 + 64) * M, M, AS, nullptr};
        Operand B{leafA + (int64_t)j0 * M, M, AS, nullptr};
        GemmArgs g = mk(R_eff - j0 - 64, 64, j0, nl, A, B, C, -1.0, 1.0);
        g.E = Einv;
        ++L.count[0];
        cudaError_t e = (f->knobs.ablate & 4) ? cudaSuccess : ks::gemm_update_trsm(g, st);
        if (e != cudaSuccess) return fail(KS_ERR_CUDA, "leaf update+trsm gemm: %s", cudaGetErrorString(e));
        if (int rc = L.check("leaf_update_trsm")) return rc;
      } else {
        Operand A{leafA + (int64_t)(j0 + 64) * M + j0, M, AS, nullptr};
        int rc = L.gemm(mk(R_eff - j0 - 64, 64, 64, nl, A, Einv, C, 1.0, 0.0), false, true, "leaf_trsm");
        if (rc) return rc;
      }
    }
  }
  if (split && R > M) {
    // the P rows: copy them in (after their upload), then L21 = P L^-T
    if (wait_p) KS_CUDA(cudaStreamWaitEvent(st, wait_p, 0));
    ks::launch_leaf_copy_p(f->devtree(), lb, st);
    ++L.count[0];
    const int S_rows = R - M;
    for (int j0 = 0; j0 < M; j0 += 64) {
      const Operand Einv{inv + (int64_t)(j0 / 64) * 64 * 64, 64, (int64_t)M * 64, nullptr};
      OperandW C{leafA + (int64_t)M * M + j0, M, AS, nullptr};
      if (j0 == 0) {
        Operand A{leafA + (int64_t)M * M, M, AS, nullptr};
        if (int rc = L.gemm(mk(S_rows, 64, 64, nl, A, Einv, C, 1.0, 0.0), false, true, "leaf_p_trsm")) return rc;
      } else {
        Operand A{leafA + (int64_t)M * M, M, AS, nullptr};
        Operand B{leafA + (int64_t)j0 * M, M, AS, nullptr};
        GemmArgs g = mk(S_rows, 64, j0, nl, A, B, C, -1.0, 1.0);
        g.E = Einv;
        ++L.count[0];
        cudaError_t e = ks::gemm_update_trsm(g, st);
        if (e != cudaSuccess) return fail(KS_ERR_CUDA, "leaf P update+trsm gemm: %s", cudaGetErrorString(e));
        if (int rc = L.check("leaf_p_update_trsm")) return rc;
      }
    }
  }
  if (S > 0 && f->n_int > 0 && !(f->knobs.ablate & 16)) {
    Operand A{leafA + (int64_t)M * M, M, AS, nullptr};
    OperandW C{f->hbuf.p, S, (int64_t)S * S, lb.node};
    // SYRK: tiles on and below the diagonal, mirrored by the epilogue (H exactly
    // symmetric, so the reference's 0.5 (H + H^T) is the identity on it)
    ++L.count[0];
    cudaError_t e = ks::gemm_syrk(mk(S, S, M, nl, A, A, C, 1.0, 0.0), st);
    if (e != cudaSuccess) return fail(KS_ERR_CUDA, "leaf syrk: %s", cudaGetErrorString(e));
    if (int rc = L.check("leaf_syrk")) return rc;
  }
  KS_CUDA(cudaGetLastError());
  return KS_OK;
}

static int enqueue_levels(ks_factor* f, cudaStream_t st, Launcher& L, int lev0, int lev1, int deferred_before = 0);
static int enqueue_level_body(ks_factor* f, Launcher& L, const ks::NodeBatch& nb, bool is_root_level, int plan_count = -1);
static ks::NodeBatch sub_batch(const ks::NodeBatch& nb, int off, int cnt);
static int plan_batch(const ks_factor* f, int level_count);
// subtree pipelining (ks_factor::npipe) in this factorization: the default 4
// node groups, not under the per-level profiler or the tracer (their level
// boundaries would blur); KS_PIPE=0 disables it
static bool pipelined(const ks_factor* f, int G) {
  if (!f->knobs.pipe) return false;
  return f->npipe > 0 && G == ks_factor::kLeafChunks && !f->profiling && !trace_on();
}

// node groups per phase (KS_GROUPS, default 2; tracing forces 1 so per-launch
// events stay on one stream)
static int n_groups(const ks_factor* f) { return trace_on() ? 1 : f->knobs.groups; }

static int enqueue_factorization(ks_factor* f, cudaStream_t st) {
  Launcher L{f, st, &f->launches[0]};
  const ks::DevTree dt = f->devtree();
  const ks::LeafBatch lb = f->leafbatch();
  const int nl = lb.count;
  auto mark = [&](cudaEvent_t e) -> int {
    if (f->profiling) KS_CUDA(cudaEventRecord(e, st));
    return KS_OK;
  };
  f->cur_tag = -1;
  if (int rc = mark(f->ev_phase[0])) return rc;
  KS_CUDA(cudaMemsetAsync(f->leaf_info.p, 0, sizeof(int) * nl, st));
  if (f->n_int) KS_CUDA(cudaMemsetAsync(f->int_info.p, 0, sizeof(int) * f->n_int, st));
  if (f->lu_sync.p) KS_CUDA(cudaMemsetAsync(f->lu_sync.p + (int64_t)4 * f->n_int, 0, sizeof(unsigned), st));
  // ---- leaves: assemble [[K + lam I], [P]] and factor, leaves split into
  // independent groups on their own streams; on the first factorization each
  // group waits only for the uploads of its own P blocks
  if (f->upload_pending) KS_CUDA(cudaStreamWaitEvent(st, f->ev_up_coords, 0));
  if (int rc = L.check("start")) return rc;
  bool pipe = false, early = false;
  int n_early = 0, np = 0;  // np: levels pipelined per subtree in this factorization
  if (int rc = mark(f->ev_phase[1])) return rc;
  {
    const int G = (nl >= 2 * 64) ? n_groups(f) : 1;
    pipe = pipelined(f, G);
    if (pipe) np = f->npipe;
    early = pipe && f->knobs.hager_early && !trace_on();
    n_early = early ? G : 0;
    if (G > 1) {
      KS_CUDA(cudaEventRecord(f->gfork, st));
      for (int g = 0; g < G; ++g) KS_CUDA(cudaStreamWaitEvent(f->gst[g], f->gfork, 0));
    }
    for (int g = 0; g < G; ++g) {
      const int l0 = (int)((int64_t)nl * g / G), l1 = (int)((int64_t)nl * (g + 1) / G);
      cudaStream_t gs = (G > 1) ? f->gst[g] : st;
      cudaEvent_t wait_p = nullptr;
      if (f->upload_pending && l1 > l0) {
        int c = 0;  // the upload chunk holding this group's last leaf
        while ((int64_t)nl * (c + 1) / ks_factor::kLeafChunks <= l1 - 1) ++c;
        wait_p = f->ev_up_leaf[c];
      }
      Launcher Lg{f, gs, &f->launches[0]};
      // while the uploads are in flight, factor A before P has arrived
      const bool split = wait_p != nullptr && (f->d & 1) == 0 && f->n_int > 0 && f->knobs.split_leaf;
      if (int rc = enqueue_leaf_assemble(f, Lg, l0, l1, wait_p, split)) return rc;
      if (int rc = enqueue_leaf_chol(f, Lg, l0, l1, split, wait_p)) return rc;
      if (pipe) {  // this subtree's nodes of the deepest np levels, on the same stream
        for (int lev = 0; lev < np; ++lev) {
          if (f->upload_pending)
            KS_CUDA(cudaStreamWaitEvent(gs, f->ev_up_sublev[(size_t)g * f->npipe + lev], 0));
          f->cur_tag = lev;
          const ks::NodeBatch nb = f->nodebatch(lev);
          const int c = nb.count / G;
          const ks::NodeBatch sb = sub_batch(nb, g * c, c);
          if (int rc = enqueue_level_body(f, Lg, sb, false, plan_batch(f, nb.count))) return rc;
          if (early) {  // this subtree's estimates at once, beside its next level
            KS_CUDA(cudaEventRecord(f->hfork[g], gs));
            KS_CUDA(cudaStreamWaitEvent(f->hst[g], f->hfork[g], 0));
            ks::launch_hager(dt, sb, f->dinv.p, f->lut.p, std::max(1, f->knobs.hager_ctas / G), f->hst[g]);
            L.count[0] += ks::hager_launches(sb);
          }
        }
        f->cur_tag = -1;
      }
    }
    if (G > 1)
      for (int g = 0; g < G; ++g) {
        KS_CUDA(cudaEventRecord(f->gjoin[g], f->gst[g]));
        KS_CUDA(cudaStreamWaitEvent(st, f->gjoin[g], 0));
      }
  }
  KS_CUDA(cudaGetLastError());
  if (int rc = mark(f->ev_phase[2])) return rc;
  if (int rc = mark(f->ev_phase[3])) return rc;
  // ---- the shard's internal levels, deepest first (the pipelined ones are
  // done; their condition estimates are still to be launched) ----
  if (int rc = enqueue_levels(f, st, L, np, f->n_local_levels, (pipe && !early) ? np : 0))
    return rc;
  for (int g = 0; g < n_early; ++g) {
    KS_CUDA(cudaEventRecord(f->hjoin[g], f->hst[g]));
    KS_CUDA(cudaStreamWaitEvent(st, f->hjoin[g], 0));
  }
  if (int rc = mark(f->ev_phase[4])) return rc;
  return KS_OK;
}

// Levels with at most KS_SLAB_MAX (default 4) nodes run the persistent
// per-node LU (lu_slab.cu); KS_SLAB_MAX=0 keeps the launch sequence everywhere.
static bool use_slab(const ks_factor* f, const ks::NodeBatch& nb, int plan_count) {
  return plan_count <= f->knobs.slab_max && f->lu_sync.p && ks::slab_width(nb) > 0;
}

// The LU variant of a node (persistent LU / spine / plain recursion) follows
// the batch size the REPLAYED schedule gives the node's level (a wide level's
// node group, a narrow level whole), not the size of the sub-batch at hand:
// the first factorization pipelines deeper (smaller sub-batches) and must give
// the same bits as every later one.
static int plan_batch(const ks_factor* f, int level_count) {
  return level_count >= 64 ? std::max(1, level_count / n_groups(f)) : level_count;
}

// batches of at most KS_SPINE_MAX (default 16) nodes carry the P^T columns
// through the recursive LU (rlu ext)

// One level's node work on L's stream for the node sub-batch nb, in the block
// formulation (kernels.cuh NodeBatch, node_kernels.cu): the coupling B, then
//   X = B H_r, Y = B^T H_l                      (Z = I + W G = [[I, X], [Y, I]], solver.py:142-148)
//   Aug = [[S, E], [F, C]] = [[I - Y X, P_r^T - Y P_l^T], [P_l H_l X - P_r H_r, P_l H_l P_l^T]]
// as DMMA GEMMs, ||Z||_1, then the LU of Aug's first s_pad columns with pivots
// among S's rows (linalg.py:199-213 on the Schur complement of Z's identity
// block) whose trailing block is H = P G Z^-1 P^T (solver.py:154-164).
static int enqueue_level_body(ks_factor* f, Launcher& L, const ks::NodeBatch& nb, bool is_root_level, int plan_count) {
  if (plan_count < 0) plan_count = nb.count;
  const ks::DevTree dt = f->devtree();
  const int S = nb.s_pad, T = nb.T, ZT = nb.zt;
  const int64_t TT = (int64_t)T * T, SS = (int64_t)S * S, XS = 2 * SS, PS = (int64_t)S * ZT;
  const int cnt = nb.count;
  cudaStream_t st = L.st;
  const int abl = f->knobs.ablate;
  if (abl & 1024) return KS_OK;
  if (!(abl & 32)) ks::launch_coupling(dt, nb, st);
  ++L.count[0];
  if (f->need_p_layout) {  // the padded P and P^T copies: once per handle
    ks::launch_p_layout(dt, nb, st);
    L.count[0] += 2;
  }
  int rc = L.check("coupling/p_layout");
  if (rc) return rc;
  double* Xb = nb.XY;
  double* Yb = nb.XY + SS;
  double* Sb = nb.Aug;
  double* Eb = nb.Aug + S;
  double* Fb = nb.Aug + (int64_t)S * T;
  double* Cb = nb.Aug + (int64_t)S * T + S;
  // stage 1 (independent products, one launch; H is exactly symmetric, so it
  // is read row-major as the right factor):
  //   X = B H_r,  Y = B^T H_l,  P_l H_l
  // stage 2 (one launch; S and E are written out of place, nothing of Aug is
  // initialized beforehand):
  //   S = I - Y X,  E = P_r^T - Y P_l^T,  C = (P_l H_l) P_l^T
  // stage 3:
  //   F = P_l H_l X - P_r H_r = -E^T H_r   (F^T = X^T H_l P_l^T - H_r P_r^T = H_r (Y P_l^T - P_r^T):
  //   one product instead of two)
  {
    ks::GemmGroup g1{};
    g1.count = 3;
    g1.p[0] = mk(S, S, S, cnt, Operand{nb.Bc, S, SS, nullptr}, Operand{f->hbuf.p, S, SS, nb.right},
                 OperandW{Xb, S, XS, nullptr}, 1.0, 0.0);
    g1.p[1] = mk(S, S, S, cnt, Operand{nb.BcT, S, SS, nullptr}, Operand{f->hbuf.p, S, SS, nb.left},
                 OperandW{Yb, S, XS, nullptr}, 1.0, 0.0);
    g1.p[2] = mk(S, S, S, cnt, Operand{nb.Pn, ZT, PS, nullptr}, Operand{f->hbuf.p, S, SS, nb.left},
                 OperandW{nb.PHl, S, SS, nullptr}, 1.0, 0.0);
    ++L.count[0];
    if (abl & 64) {
    } else if (cudaError_t e = ks::gemm_group(g1, st)) return fail(KS_ERR_CUDA, "assembly stage 1: %s", cudaGetErrorString(e));
    if ((rc = L.check("assembly1"))) return rc;
    const int64_t PTS = (int64_t)ZT * S;
    ks::GemmGroup g2{};
    g2.count = 3;
    g2.p[0] = mk(S, S, S, cnt, Operand{Yb, S, XS, nullptr}, Operand{Xb, S, XS, nullptr}, OperandW{Sb, T, TT, nullptr},
                 -1.0, 0.0);
    g2.p[0].addI = 1;
    g2.p[1] = mk(S, S, S, cnt, Operand{Yb, S, XS, nullptr}, Operand{nb.PT, S, PTS, nullptr},
                 OperandW{Eb, T, TT, nullptr}, -1.0, 1.0);
    g2.p[1].Cin = Operand{nb.PT + SS, S, PTS, nullptr};  // P_r^T
    g2.p[2] = mk(S, S, S, cnt, Operand{nb.PHl, S, SS, nullptr}, Operand{nb.PT, S, PTS, nullptr},
                 OperandW{Cb, T, TT, nullptr}, 1.0, 0.0);
    g2.p[2].tri = 2;  // C = P_l H_l P_l^T is symmetric: tiles on and below the diagonal, mirrored
    ++L.count[0];
    if (abl & 64) {
    } else if (cudaError_t e = ks::gemm_group(g2, st)) return fail(KS_ERR_CUDA, "assembly stage 2: %s", cudaGetErrorString(e));
    if ((rc = L.check("assembly2"))) return rc;
    if (!(abl & 64)) {
      if ((rc = L.gemm(mk(S, S, S, cnt, Operand{Eb, T, TT, nullptr}, Operand{f->hbuf.p, S, SS, nb.right},
                          OperandW{Fb, T, TT, nullptr}, -1.0, 0.0), true, false, "assembly3")))
        return rc;
    }
  }
  ks::launch_znorm1(nb, st);  // ||Z||_1 for the condition estimate (linalg.py:176)
  ++L.count[0];
  if ((rc = L.check("znorm1"))) return rc;
  if (abl & 128) return KS_OK;
  if (use_slab(f, nb, plan_count)) {
    // narrow level: the whole LU, U12, Schur block and H in one cooperative launch
    // (its own ||.||_1 of the slabs goes to a scratch word: Z's norm is znorm1's)
    ks::NodeBatch sb = nb;
    sb.norm1 = f->norm1_slab.p + nb.first;
    KS_CUDA(cudaMemsetAsync(sb.norm1, 0, sizeof(double) * cnt, st));
    unsigned* sy = f->lu_sync.p + (int64_t)4 * nb.first;
    KS_CUDA(cudaMemsetAsync(sy, 0, sizeof(unsigned) * 4 * cnt, st));
    if (ks::launch_lu_slab(sb, f->hbuf.p, SS, !is_root_level, sy, f->lu_sync.p + (int64_t)4 * f->n_int, st))
      return fail(KS_ERR_CUDA, "persistent LU launch failed: %s", cudaGetErrorString(cudaGetLastError()));
    ++L.count[0];
    if (int rc2 = L.check("lu_slab")) return rc2;
    ks::launch_compose_perm(nb, st);
    ++L.count[0];
    KS_CUDA(cudaGetLastError());
    return KS_OK;
  }
  // LU of S's columns with pivots restricted to S's rows. Small batches carry
  // the E columns on the right spine of the recursion (U12 = L^-1 Pi E and the
  // Schur block H come out of the merges: fewer dependent launches); large
  // batches keep the separate U12 TRSM and Schur GEMM (higher tensor-pipe rate).
  int pend[4] = {0, 0, 0, 0};
  const int TP = nb.t_pad;
  const bool spine = plan_count <= f->knobs.spine_max;
  if ((rc = rlu(L, nb, 0, TP, f->pw, pend, spine ? S : 0))) return rc;
  if (!spine) {
    if ((rc = trsm_ul(L, nb, 0, TP, TP, S))) return rc;
    // H = C - F S^-1 E is symmetric like C: the same 10 of 16 tiles, mirrored
    GemmArgs gs = mk(S, S, TP, cnt, Operand{Fb, T, TT, nullptr}, Operand{Eb, T, TT, nullptr},
                     OperandW{Cb, T, TT, nullptr}, -1.0, 1.0);
    gs.tri = 2;
    if ((rc = L.gemm(gs, false, false, "schur"))) return rc;
  }
  ks::launch_compose_perm(nb, st);
  ++L.count[0];
  if (!is_root_level) {
    ks::launch_extract_h(nb, f->hbuf.p, SS, st);
    ++L.count[0];
    if (int rc2 = L.check("extract_h")) return rc2;
  }
  KS_CUDA(cudaGetLastError());
  return KS_OK;
}

static ks::NodeBatch sub_batch(const ks::NodeBatch& nb, int off, int cnt) {
  const int S = nb.s_pad, T = nb.T, TP = nb.t_pad;
  ks::NodeBatch s = nb;
  s.count = cnt;
  s.first = nb.first + off;
  s.node = nb.node + off;
  s.left = nb.left + off;
  s.right = nb.right + off;
  s.Aug = nb.Aug + (int64_t)off * T * T;
  s.XY = nb.XY + (int64_t)off * 2 * S * S;
  s.PHl = nb.PHl + (int64_t)off * S * S;
  s.Bc = nb.Bc + (int64_t)off * S * S;
  s.BcT = nb.BcT + (int64_t)off * S * S;
  s.PT = nb.PT + (int64_t)off * nb.zt * S;
  if (nb.XS) {
    s.XS = nb.XS + (int64_t)off * nb.zt * nb.dk;
    s.XN = nb.XN + (int64_t)off * nb.zt;
  }
  s.Pn = nb.Pn + (int64_t)off * S * nb.zt;
  s.piv = nb.piv + (int64_t)off * TP;
  s.norm1 = nb.norm1 + off;
  s.cond = nb.cond + off;
  s.info = nb.info + off;
  s.moves = nb.moves + (int64_t)off * (2 * 64 + 1);
  s.pm = nb.pm + (int64_t)off * TP;
  s.scratch = nb.scratch + (int64_t)off * 32 * 64;
  return s;
}

// SMs the overlapped condition estimates may occupy (of 148); KS_HAGER_CTAS overrides

// KS_HAGER_FLUSH=n: launch the deferred estimates at the first level with <= n
// nodes (default 0: the first narrow level, < 64 nodes)

// KS_HAGER_SPLIT=0: narrow levels' estimates queue on `side` like the wide ones

// Internal levels [lev0, lev1) of the plan (deepest first); wide levels split
// into node groups on the group streams. Condition estimates run on the side
// stream (they only feed diagnostics), joined at the end. The estimates of the
// wide (HBM-heavy) levels wait for the first narrow level, whose latency-bound
// launches leave most SMs idle, instead of competing with the next wide level.
static int enqueue_levels(ks_factor* f, cudaStream_t st, Launcher& L, int lev0, int lev1, int deferred_before) {
  const ks::DevTree dt = f->devtree();
  auto mark = [&](cudaEvent_t e) -> int {
    if (f->profiling) KS_CUDA(cudaEventRecord(e, st));
    return KS_OK;
  };
  std::vector<int> deferred;  // levels whose estimate is not launched yet
  for (int lv = 0; lv < deferred_before; ++lv) deferred.push_back(lv);
  bool used_side = false, used_side2 = false;
  auto flush = [&]() -> int {
    if (deferred.empty()) return KS_OK;
    if (trace_on()) {  // inline, so the trace times each estimate
      for (int lv : deferred) {
        f->cur_tag = lv;
        ks::launch_hager(dt, f->nodebatch(lv), f->dinv.p, f->lut.p, 1 << 30, st);
        L.count[0] += ks::hager_launches(f->nodebatch(lv));
        if (int rc = L.check("hager")) return rc;
      }
      deferred.clear();
      return KS_OK;
    }
    KS_CUDA(cudaEventRecord(f->ev_fork, st));
    KS_CUDA(cudaStreamWaitEvent(f->side, f->ev_fork, 0));
    used_side = true;
    for (int lv : deferred) {
      ks::launch_hager(dt, f->nodebatch(lv), f->dinv.p, f->lut.p, f->knobs.hager_ctas, f->side);
      L.count[0] += ks::hager_launches(f->nodebatch(lv));
    }
    deferred.clear();
    KS_CUDA(cudaGetLastError());
    return KS_OK;
  };
  for (int lev = lev0; lev < lev1; ++lev) {
    f->cur_tag = (int)lev;
    if (f->upload_pending) KS_CUDA(cudaStreamWaitEvent(st, f->ev_up_level[lev], 0));
    const ks::NodeBatch nb = f->nodebatch((int)lev);
    const bool is_root_level = (f->levels[lev][0] == 0);
    const bool wide = nb.count >= 64;
    if (f->knobs.hager_flush > 0 ? nb.count <= f->knobs.hager_flush : !wide)
      if (int rc = flush()) return rc;
    const int G = wide ? n_groups(f) : 1;
    if (G == 1) {
      if (int rc = enqueue_level_body(f, L, nb, is_root_level)) return rc;
    } else {
      KS_CUDA(cudaEventRecord(f->gfork, st));
      for (int g = 0; g < G; ++g) {
        KS_CUDA(cudaStreamWaitEvent(f->gst[g], f->gfork, 0));
        const int o0 = (int)((int64_t)nb.count * g / G), o1 = (int)((int64_t)nb.count * (g + 1) / G);
        Launcher Lg{f, f->gst[g], &f->launches[0]};
        if (int rc = enqueue_level_body(f, Lg, sub_batch(nb, o0, o1 - o0), is_root_level))
          return rc;
        KS_CUDA(cudaEventRecord(f->gjoin[g], f->gst[g]));
        KS_CUDA(cudaStreamWaitEvent(st, f->gjoin[g], 0));
      }
    }
    // condition estimate off the critical path: a narrow level's right away
    // on side2 (one CTA per node), a wide level's deferred (see above)
    if (!wide && !trace_on() && f->knobs.hager_split) {
      KS_CUDA(cudaEventRecord(f->ev_fork2, st));
      KS_CUDA(cudaStreamWaitEvent(f->side2, f->ev_fork2, 0));
      used_side2 = true;
      ks::launch_hager(dt, nb, f->dinv.p, f->lut.p, nb.count, f->side2);
      L.count[0] += ks::hager_launches(nb);
      KS_CUDA(cudaGetLastError());
    } else {
      deferred.push_back(lev);
      if (f->knobs.hager_flush > 0 ? nb.count <= f->knobs.hager_flush : !wide)
        if (int rc = flush()) return rc;
    }
    if (int rc2 = mark(f->ev_level[lev])) return rc2;
  }
  if (int rc = flush()) return rc;
  if (used_side) {
    KS_CUDA(cudaEventRecord(f->ev_join, f->side));
    KS_CUDA(cudaStreamWaitEvent(st, f->ev_join, 0));
  }
  if (used_side2) {
    KS_CUDA(cudaEventRecord(f->ev_join2, f->side2));
    KS_CUDA(cudaStreamWaitEvent(st, f->ev_join2, 0));
  }
  return KS_OK;
}

// The reference raises at the first failing node in its processing order
// (levels bottom-up, ids ascending): singular LU (linalg.py:205-206), then the
// condition estimate above 1e14 (solver.py:150-152).
static int check_nodes(ks_factor* f, int k0, int k1) {
  for (int k = k0; k < k1; ++k) {
    if (f->int_info_h[k])
      return fail(KS_ERR_SINGULAR, "node %d: zero pivot column at elimination step %d", f->int_nodes[k],
                  f->int_info_h[k] - 1);
    const double cnd = f->cond_h[k];
    if (!(cnd <= kCondHard))
      return fail(KS_ERR_ILL_COND, "reduced system at node %d is numerically singular (1-norm condition estimate %.3e)",
                  f->int_nodes[k], cnd);
  }
  return KS_OK;
}


// Non-SPD leaves: LU with partial pivoting of [[A, -P^T], [P, 0]] for the
// first m_pad pivots (dense_factor(..., "lu-partial-pivot"), solver.py:127-130);
// the Schur complement is H = P A^-1 P^T (solver.py:134-135).
// device storage of the LU-fallback leaves listed in f->fb_leaf
static int fb_alloc_impl(ks_factor* f) {
  const int nf = (int)f->fb_leaf.size();
  const int M = f->m_pad;
  const int T = M + ((f->n_nodes > 1) ? f->s_pad : 0);
  f->fb_aug.release(); f->fb_piv.release(); f->fb_info.release(); f->fb_moves.release(); f->fb_pm.release();
  f->fb_node.release(); f->fb_begin.release(); f->fb_size.release(); f->fb_norm1.release(); f->fb_cond.release();
  f->fb_T = T;
  std::vector<int> nd, bg, sz;
  for (int li : f->fb_leaf) {
    const int v = f->leaf_nodes[li];
    nd.push_back(v);
    bg.push_back((int)f->begin[v]);
    sz.push_back((int)(f->end[v] - f->begin[v]));
  }
  KS_CUDA(f->fb_aug.alloc((size_t)nf * T * T));
  KS_CUDA(f->fb_piv.alloc((size_t)nf * M));
  KS_CUDA(f->fb_info.alloc(nf));
  KS_CUDA(f->fb_moves.alloc((size_t)nf * (2 * 64 + 1)));
  KS_CUDA(f->fb_pm.alloc((size_t)nf * M));
  KS_CUDA(f->fb_norm1.alloc(nf));
  KS_CUDA(f->fb_cond.alloc(nf));
  KS_CUDA(f->fb_node.upload(nd));
  KS_CUDA(f->fb_begin.upload(bg));
  KS_CUDA(f->fb_size.upload(sz));
  return KS_OK;
}

static int factor_fallback_leaves(ks_factor* f, cudaStream_t st) {
  const int nf = (int)f->fb_leaf.size();
  const int M = f->m_pad;
  const int S = (f->n_nodes > 1) ? f->s_pad : 0;
  const int T = M + S;
  if (nf == 0) return KS_OK;
  if (T != f->fb_T || f->fb_node.n != (size_t)nf)
    if (int rc = fb_alloc_impl(f)) return rc;
  const ks::NodeBatch fb = f->fb_batch();
  Launcher L{f, st, &f->launches[0]};
  KS_CUDA(cudaMemsetAsync(f->fb_info.p, 0, sizeof(int) * nf, st));
  ks::launch_fb_assemble(f->devtree(), fb, f->fb_begin.p, f->fb_size.p, f->lam_dev.p, st);
  int pend[4] = {0, 0, 0, 0};
  int rc = rlu(L, fb, 0, M, T <= 1024 ? 16 : 8, pend, S);  // the -P^T columns on the spine: H comes out of it
  if (rc) return rc;
  if (S > 0) ks::launch_extract_h(fb, f->hbuf.p, (int64_t)f->s_pad * f->s_pad, st);
  ks::launch_compose_perm(fb, st);
  KS_CUDA(cudaGetLastError());
  std::vector<int> info(nf, 0);
  KS_CUDA(cudaMemcpyAsync(info.data(), f->fb_info.p, sizeof(int) * nf, cudaMemcpyDeviceToHost, st));
  KS_CUDA(cudaStreamSynchronize(st));
  for (int k = 0; k < nf; ++k)
    if (info[k])  // linalg.py:205-206 inside the fallback (solver.py:129)
      return fail(KS_ERR_SINGULAR, "leaf %d: zero pivot column at elimination step %d", f->leaf_nodes[f->fb_leaf[k]],
                  info[k] - 1);
  return KS_OK;
}


}  // namespace

namespace ksr {
int fb_alloc(ks_factor* f) { return fb_alloc_impl(f); }
}  // namespace ksr

extern "C" {

int ks_factorize(ks_factor* f, double lam, void* stream) {
  if (!f) return fail(KS_ERR_INVALID, "null handle");
  if (!std::isfinite(lam) || lam < 0.0) return fail(KS_ERR_INVALID, "need lambda >= 0 and finite, got %g", lam);
  KS_CUDA(cudaSetDevice(f->device));
  cudaStream_t st = (cudaStream_t)stream;
  f->lam = lam;
  f->factored = false;
  f->launches[0] = 0;
  f->trace_n = 0;
  const int nl = (int)f->leaf_nodes.size();
  KS_CUDA(cudaMemcpyAsync(f->lam_dev.p, &f->lam, sizeof(double), cudaMemcpyHostToDevice, st));
  // CUDA graph of the ~1000-launch sequence: from the second factorization on
  // (KS_GRAPH=1, default), always (2) or never (0); tracing runs eagerly.
  f->need_p_layout = !f->p_layout_local;
  const int gm = (trace_on() || debug_sync() || f->profiling) ? 0 : f->knobs.graph;
  const bool use_graph = gm == 2 || (gm == 1 && f->n_factorizations > 0);
  if (use_graph && f->upload_pending) {  // a graph does not capture waits on the upload stream
    KS_CUDA(cudaStreamSynchronize(f->upl));
    f->upload_pending = false;
  }
  if (use_graph) {
    if (!f->graph_exec || f->graph_profiling != f->profiling) {
      if (f->graph_exec) { cudaGraphExecDestroy(f->graph_exec); f->graph_exec = nullptr; }
      cudaGraph_t g = nullptr;
      KS_CUDA(cudaStreamBeginCapture(f->cap, cudaStreamCaptureModeThreadLocal));
      int rc = enqueue_factorization(f, f->cap);
      cudaError_t ce = cudaStreamEndCapture(f->cap, &g);
      if (rc) { if (g) cudaGraphDestroy(g); return rc; }
      KS_CUDA(ce);
      KS_CUDA(cudaGraphInstantiate(&f->graph_exec, g, 0));
      cudaGraphDestroy(g);
      f->graph_profiling = f->profiling;
      f->graph_launches = f->launches[0];
    }
    KS_CUDA(cudaGraphLaunch(f->graph_exec, st));
    f->launches[0] = f->graph_launches;
  } else {
    int rc = enqueue_factorization(f, st);
    if (rc) return rc;
    if (f->upload_pending) {  // everything after this point sees every upload
      KS_CUDA(cudaStreamWaitEvent(st, f->ev_up_all, 0));
      f->upload_pending = false;
    }
  }
  ++f->n_factorizations;
  f->p_layout_local = true;
  if (f->knobs.ablate) {  // timing experiment: nothing below is meaningful
    KS_CUDA(cudaStreamSynchronize(st));
    return KS_OK;
  }
  // leaf Cholesky failures (NotSPD) -> LU fallback for those leaves (solver.py:125-131)
  f->leaf_info_h.assign(nl, 0);
  KS_CUDA(cudaMemcpyAsync(f->leaf_info_h.data(), f->leaf_info.p, sizeof(int) * nl, cudaMemcpyDeviceToHost, st));
  KS_CUDA(cudaStreamSynchronize(st));
  f->fallback.clear();
  std::vector<int> failed;
  const bool force = f->knobs.force_leaf_lu;
  for (int i = 0; i < nl; ++i)
    if (f->leaf_info_h[i] || force) {
      f->fallback.push_back(f->leaf_nodes[i]);
      failed.push_back(i);
    }
  if (failed != f->fb_leaf) {
    f->fb_leaf = failed;
    f->fb_T = 0;  // re-plan the fallback buffers
  }
  if (!failed.empty()) {
    // LU for those leaves, then the internal levels again on the corrected H
    if (int rc = factor_fallback_leaves(f, st)) return rc;
    if (f->n_int) KS_CUDA(cudaMemsetAsync(f->int_info.p, 0, sizeof(int) * f->n_int, st));
    Launcher L{f, st, &f->launches[0]};
    if (int rc = enqueue_levels(f, st, L, 0, f->n_local_levels)) return rc;
  }
  // ---- diagnostics and errors (solver.py:150-152, 175-188) ----
  f->int_info_h.assign(f->n_int, 0);
  f->cond_h.assign(f->n_int, 0.0);
  if (f->n_int) {
    KS_CUDA(cudaMemcpyAsync(f->int_info_h.data(), f->int_info.p, sizeof(int) * f->n_int, cudaMemcpyDeviceToHost, st));
    KS_CUDA(cudaMemcpyAsync(f->cond_h.data(), f->cond.p, sizeof(double) * f->n_int, cudaMemcpyDeviceToHost, st));
  }
  unsigned watchdog = 0;
  if (f->lu_sync.p)
    KS_CUDA(cudaMemcpyAsync(&watchdog, f->lu_sync.p + (int64_t)4 * f->n_int, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  KS_CUDA(cudaStreamSynchronize(st));
  if (watchdog) return fail(KS_ERR_CUDA, "persistent LU: a node's slabs stopped making progress (watchdog)");
  if (f->profiling) {
    auto el = [](cudaEvent_t a, cudaEvent_t b) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, a, b);
      return (double)ms;
    };
    f->phase_ms[0] = el(f->ev_phase[0], f->ev_phase[1]);
    f->phase_ms[1] = el(f->ev_phase[1], f->ev_phase[2]);
    f->phase_ms[2] = el(f->ev_phase[2], f->ev_phase[3]);
    f->phase_ms[3] = el(f->ev_phase[3], f->ev_phase[4]);
    f->phase_ms[4] = el(f->ev_phase[0], f->ev_phase[4]);
    f->level_ms.assign(f->n_local_levels, 0.0);
    for (int i = 0; i < f->n_local_levels; ++i)
      f->level_ms[i] = el(i == 0 ? f->ev_phase[3] : f->ev_level[i - 1], f->ev_level[i]);
  }
  if (trace_on() && f->trace_n > 1) {
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
    rep += "-- last 120 launches --\n";
    for (int i = std::max(1, f->trace_n - 120); i < f->trace_n; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, f->trace_ev[i - 1], f->trace_ev[i]);
      std::snprintf(line, sizeof line, "%-18s %8.1f us\n", f->trace_name[i], ms * 1e3);
      rep += line;
    }
    f->trace_report = rep;
  }
  const int k1 = f->n_local_levels < (int)f->levels.size() ? f->level_first[f->n_local_levels] : f->n_int;
  if (int rc = check_nodes(f, 0, k1)) return rc;
  f->local_factored = true;
  f->factored = (f->n_local_levels == (int)f->levels.size());
  return KS_OK;
}

int ks_factorize_top(ks_factor* f, void* stream) {
  if (!f) return fail(KS_ERR_INVALID, "null handle");
  if (!f->local_factored) return fail(KS_ERR_INVALID, "factor the shard (ks_factorize) first");
  KS_CUDA(cudaSetDevice(f->device));
  cudaStream_t st = (cudaStream_t)stream;
  Launcher L{f, st, &f->launches[0]};
  f->need_p_layout = !f->p_layout_top;
  if (int rc = enqueue_levels(f, st, L, f->n_local_levels, (int)f->levels.size())) return rc;
  f->p_layout_top = true;
  const int k0 = f->n_local_levels < (int)f->levels.size() ? f->level_first[f->n_local_levels] : f->n_int;
  if (f->n_int > k0) {
    KS_CUDA(cudaMemcpyAsync(f->int_info_h.data() + k0, f->int_info.p + k0, sizeof(int) * (f->n_int - k0),
                            cudaMemcpyDeviceToHost, st));
    KS_CUDA(cudaMemcpyAsync(f->cond_h.data() + k0, f->cond.p + k0, sizeof(double) * (f->n_int - k0),
                            cudaMemcpyDeviceToHost, st));
  }
  KS_CUDA(cudaStreamSynchronize(st));
  if (int rc = check_nodes(f, k0, f->n_int)) return rc;
  f->factored = true;
  return KS_OK;
}

}  // extern "C"
