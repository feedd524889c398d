// Internal header of the host runtime behind the C ABI (include/invaskit.h):
// the factor handle, device buffers, per-solve workspaces, the launch helper
// and the tuning switches. Translation units:
//   runtime.cu    errors, device memory pool, tuning switches, launch helpers
//                 (recursive LU / TRSM sequences), ks_destroy
//   create.cu     ks_create / ks_create_shard: validation, level plan, uploads
//   factorize.cu  ks_factorize / ks_factorize_top: the level schedule
//   solve.cu      ks_solve (+ shard phases), ks_matvec, per-call workspaces
//   diag.cu       diagnostics, debug views, profiling, test hooks, krr matvec
//   persist.cu    operator / factor files (container.h)
#pragma once

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/invaskit.h"
#include "gemm.cuh"
#include "kernels.cuh"

namespace ksr {

// ---- errors: a thread-local message behind every non-zero return code ----
int fail(int code, const char* fmt, ...);
const std::string& last_error_msg();

#define KS_CUDA(x)                                                                                    \
  do {                                                                                                \
    cudaError_t e_ = (x);                                                                             \
    if (e_ != cudaSuccess)                                                                            \
      return ::ksr::fail(KS_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
  } while (0)

constexpr double kCondHard = 1e14;  // solver.py:50
constexpr double kCondWarn = 1e10;  // solver.py:51

inline int64_t roundup(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

// ---- tuning switches, read from the environment. The
// per-handle ones are snapshot when the handle is created, so a process can
// run handles with different settings (the parity tests do). ----
struct Knobs {
  int slab_max = 4;            // KS_SLAB_MAX: levels with <= this many nodes run the persistent LU
  int spine_max = 16;          // KS_SPINE_MAX: batches <= this carry P^T on the recursive LU's spine
  int groups = 8;              // KS_GROUPS: leaf groups / subtree streams
  bool pipe = true;            // KS_PIPE=0: join the groups after the leaves
  int pipe_min = 16;           // KS_PIPE_MIN: nodes per subtree for a level to be pipelined
  int panel_w = 0;             // KS_PANEL_W: 32 / 8 override the register-panel width
  bool fused_merge = false;    // KS_FUSED_MERGE=1: TRSM + update merge in one launch (slower)
  bool unfused_leaf_trsm = false;  // KS_UNFUSED_LEAF_TRSM=1: separate leaf update and TRSM GEMMs
  bool split_leaf = true;      // KS_SPLIT_LEAF=0: the first factorization waits for the leaves' P up front
  int hager_ctas = 96;         // KS_HAGER_CTAS: CTAs of the deferred wide-level estimates
  int hager_flush = 0;         // KS_HAGER_FLUSH: start the deferred estimates at levels <= n nodes
  bool hager_split = true;     // KS_HAGER_SPLIT=0: narrow-level estimates queue with the wide ones
  bool hager_early = false;    // KS_HAGER_EARLY=1: a pipelined level's estimates right after each subtree's level
  bool force_leaf_lu = false;  // KS_FORCE_LEAF_LU=1: test hook, every leaf takes the LU path
  int graph = 1;               // KS_GRAPH: 1 graph replay from the 2nd factorization, 2 always, 0 never
  int ablate = 0;              // KS_ABLATE: timing experiment, skip pieces of the schedule (results are garbage; tools/ablate.py)
};
Knobs read_knobs();
// process-wide debugging switches
bool trace_on();     // KS_TRACE=1: an event after every launch (per-kernel times)
bool debug_sync();   // KS_DEBUG_SYNC=1: synchronize after every launch
bool host_timing();  // KS_HOST_TIMING=1: host phases of ks_create on stderr
double host_ms();

// ---- device memory: the stream-ordered pool of the handle's device ----
cudaError_t pool_alloc(void** p, size_t bytes);
cudaError_t pool_alloc_async(void** p, size_t bytes, cudaStream_t st);  // stream-ordered, caller frees with cudaFreeAsync
void pool_free(void* p);
void pool_trim();  // give unused pool memory back to the driver (ks_destroy)

template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaError_t alloc(size_t count) {
    n = count;
    if (count == 0) return cudaSuccess;
    return pool_alloc(reinterpret_cast<void**>(&p), count * sizeof(T));
  }
  cudaError_t upload(const std::vector<T>& v) {
    cudaError_t e = alloc(v.size());
    if (e != cudaSuccess || v.empty()) return e;
    return cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
  }
  void release() {
    if (p) pool_free(p);
    p = nullptr;
    n = 0;
  }
};

bool is_device_ptr(const void* p);

// ---- per-call solve workspace. The factor is immutable after ks_factorize;
// every solve / matvec takes a workspace of its own from the handle's pool, so
// concurrent calls (several host threads, or several streams) never share
// intermediates (SPEC concurrency model: solves on a shared factor are safe).
struct SolveWs {
  int64_t q_cap = 0;
  DBuf<double> z, c, tin, y, wtmp, bdev, xdev, fb_y;  // solve intermediates, q_cap columns
  int64_t mv_q = 0;
  DBuf<double> mv_c, mv_inc, mv_tot;                  // hss_matvec intermediates
  cudaEvent_t done = nullptr;     // recorded on the last user's stream when it released the workspace
  cudaStream_t last = nullptr;    // that stream
  bool busy = false;
  std::atomic<int64_t> launches{0};  // kernel launches of the call using it
  void release_all() {
    z.release(); c.release(); tin.release(); y.release(); wtmp.release(); bdev.release(); xdev.release();
    fb_y.release(); mv_c.release(); mv_inc.release(); mv_tot.release();
    q_cap = mv_q = 0;
  }
};

}  // namespace ksr

struct ks_factor {
  int device = 0;
  ksr::Knobs knobs;
  int64_t n = 0, d = 0, n_nodes = 0;
  std::vector<int64_t> begin, end, left, right, rank, level;
  // plan
  std::vector<int> leaf_nodes;                 // leaf index -> node
  std::vector<std::vector<int>> levels;        // internal nodes per level, deepest first
  std::vector<int> level_first;                // internal index of each level's first node
  std::vector<int> int_nodes;                  // internal index -> node
  int n_int = 0;
  // subtree sharding (multi-GPU): this handle factors the subtree of shard_root
  // ("local" levels) and, after the level-k exchange, the levels above it ("top")
  int64_t shard_root = 0;
  int shard_level = 0;
  int n_local_levels = 0;
  // subtree pipelining: the deepest npipe levels split into kLeafChunks
  // subtrees, each factored on its own stream right after its own leaves
  // (children of a subtree's nodes lie in the same subtree one level down)
  int npipe = 0;
  int64_t loc_begin = 0, loc_end = 0;   // tree-order rows owned by the shard
  std::vector<int64_t> peers;           // nodes at the shard level (all shards' roots)
  bool local_factored = false;
  // padded shapes: leaf m_pad, rank s_pad; the node LU view has t_pad = s_pad pivot
  // rows and order T = 2 s_pad; zt = 2 s_pad is the order of the padded Z
  int m_pad = 0, s_pad = 0, t_pad = 0, T = 0, zt = 0, R = 0, pw = 32;
  // device tables
  ksr::DBuf<double> coords, xx;   // coords: n + m_pad rows (zero tail), tree order
  ksr::DBuf<int> rank_d, skel_pos;
  ksr::DBuf<int64_t> skel_off, coeff_off;
  ksr::DBuf<double> coeff;
  ksr::DBuf<int> leaf_node, leaf_begin, leaf_size, leaf_info;
  ksr::DBuf<int> int_node, int_left, int_right, int_info, piv, moves, pm;
  ksr::DBuf<double> lu_scratch;
  ksr::DBuf<unsigned> lu_sync;  // persistent-LU flags: 4 words per internal node + the watchdog word
  ksr::DBuf<double> dinv;  // condition estimator: diagonal-block inverses of every node's Z factors
  ksr::DBuf<double> lut;   // condition estimator: column-major copies of every node's Z factors (t_pad <= 512)
  ksr::DBuf<double> leafA, inv, hbuf, aug, bc, pn, norm1, cond;
  ksr::DBuf<double> xy, phl;      // per internal node: X = B H_r and Y = B^T H_l; P_l H_l (the solve's up pass)
  ksr::DBuf<double> bt, pt;       // per internal node: B^T, P^T (operands of the assembly GEMMs)
  ksr::DBuf<double> xs, xn;       // GEMM-form coupling (large d): gathered skeleton coordinates, norms
  int dk = 0;                     // their padded dimension (0: difference-form coupling kernel)
  ksr::DBuf<double> norm1_slab;   // scratch for the persistent LU's own column norms
  // solve workspaces (solve.cu): a pool of per-call workspaces; the sharded
  // solve phases (ks_solve_up / top / down, ks_node_exchange) keep theirs across calls
  std::mutex ws_mu;
  std::vector<std::unique_ptr<ksr::SolveWs>> ws;
  ksr::SolveWs* shard_ws = nullptr;
  ksr::SolveWs* last_ws = nullptr;  // the workspace of the last solve (debug views)
  double h = 1.0;
  double lam = 0.0;
  bool factored = false;
  cudaStream_t side = nullptr, cap = nullptr;
  // independent node groups run on their own streams so latency-bound kernels
  // (POTRF, LU panels, TRSM) of one group overlap the GEMMs of another
  static constexpr int kGroups = 8;  // stream slots; KS_GROUPS picks how many are used (default 8)
  cudaStream_t gst[kGroups] = {};
  cudaEvent_t gfork = nullptr, gjoin[kGroups] = {};
  // per-group condition-estimate streams (KS_HAGER_EARLY)
  cudaStream_t hst[kGroups] = {};
  cudaEvent_t hfork[kGroups] = {}, hjoin[kGroups] = {};
  cudaEvent_t ev_phase[5] = {};
  std::vector<cudaEvent_t> ev_level;
  cudaGraphExec_t graph_exec = nullptr;
  bool graph_profiling = false;
  int64_t graph_launches = 0;
  int64_t n_factorizations = 0;
  // the padded P and P^T copies of the internal nodes (pn, pt) depend only on the
  // operator: laid out by the first factorization of the local / top levels
  bool p_layout_local = false, p_layout_top = false, need_p_layout = true;
  ksr::DBuf<double> lam_dev;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // narrow levels' condition estimates: their own stream, so they do not queue
  // behind the deferred wide-level batch on `side`
  cudaStream_t side2 = nullptr;
  cudaEvent_t ev_fork2 = nullptr, ev_join2 = nullptr;
  // uploads started by ks_create, consumed by the first factorization
  static constexpr int kLeafChunks = 8;
  cudaStream_t upl = nullptr;
  cudaEvent_t ev_up_coords = nullptr, ev_up_all = nullptr, ev_up_leaf[kLeafChunks] = {};
  std::vector<cudaEvent_t> ev_up_level;
  std::vector<cudaEvent_t> ev_up_sublev;  // [subtree][level < npipe]
  bool upload_pending = false;
  int64_t h2d_bytes = 0;  // host -> device bytes ks_create copied (operator inputs this handle reads)
  // diagnostics
  std::vector<int> leaf_info_h, int_info_h;
  std::vector<double> cond_h;
  std::vector<int64_t> fallback;
  // LU fallback leaves (non-SPD leaf blocks, solver.py:125-131)
  std::vector<int> fb_leaf;  // leaf indices
  int fb_T = 0;
  ksr::DBuf<double> fb_aug, fb_norm1, fb_cond;
  ksr::DBuf<int> fb_piv, fb_info, fb_moves, fb_pm, fb_node, fb_begin, fb_size;
  ks::NodeBatch fb_batch() const {
    ks::NodeBatch nb{};
    nb.count = (int)fb_leaf.size();
    nb.first = 0;
    nb.node = fb_node.p;
    nb.left = fb_node.p;
    nb.right = fb_node.p;
    nb.s_pad = fb_T - m_pad;
    nb.t_pad = m_pad;
    nb.T = fb_T;
    nb.zt = 0;
    nb.XY = nullptr;
    nb.PHl = nullptr;
    nb.BcT = nullptr;
    nb.PT = nullptr;
    nb.XS = nullptr;
    nb.XN = nullptr;
    nb.dk = 0;
    nb.Aug = fb_aug.p;
    nb.Bc = nullptr;
    nb.Pn = nullptr;
    nb.piv = fb_piv.p;
    nb.norm1 = fb_norm1.p;
    nb.cond = fb_cond.p;
    nb.info = fb_info.p;
    nb.moves = fb_moves.p;
    nb.pm = fb_pm.p;
    nb.scratch = nullptr;
    return nb;
  }
  // profiling
  bool profiling = false;
  double phase_ms[6] = {0, 0, 0, 0, 0, 0};
  std::vector<double> level_ms;
  // KS_TRACE=1: an event after every launch on the main stream; consecutive
  // deltas are per-kernel device times (including launch gaps). Debugging only:
  // not meant for concurrent calls on one handle.
  std::vector<cudaEvent_t> trace_ev;
  std::vector<const char*> trace_name;
  std::vector<int> trace_tag;
  int cur_tag = -1;  // -1 leaves, else internal level index
  int trace_n = 0;
  std::string trace_report;
  std::atomic<int64_t> launches[2] = {{0}, {0}};

  ks::DevTree devtree() const {
    ks::DevTree t;
    t.n = n;
    t.d = d;
    t.coords = coords.p;
    t.rank = rank_d.p;
    t.skel_off = skel_off.p;
    t.skel_pos = skel_pos.p;
    t.coeff_off = coeff_off.p;
    t.coeff = coeff.p;
    t.h = h;
    return t;
  }
  ks::LeafBatch leafbatch() const {
    ks::LeafBatch lb;
    lb.count = (int)leaf_nodes.size();
    lb.node = leaf_node.p;
    lb.begin = leaf_begin.p;
    lb.size = leaf_size.p;
    lb.m_pad = m_pad;
    lb.s_pad = s_pad;
    lb.A = leafA.p;
    lb.a_stride = (int64_t)R * m_pad;
    return lb;
  }
  ks::NodeBatch nodebatch(int lev) const {
    const int first = level_first[lev];
    ks::NodeBatch nb;
    nb.count = (int)levels[lev].size();
    nb.first = first;
    nb.node = int_node.p + first;
    nb.left = int_left.p + first;
    nb.right = int_right.p + first;
    nb.s_pad = s_pad;
    nb.t_pad = t_pad;
    nb.T = T;
    nb.zt = zt;
    nb.Aug = aug.p + (int64_t)first * T * T;
    nb.XY = xy.p + (int64_t)first * 2 * s_pad * s_pad;
    nb.PHl = phl.p + (int64_t)first * s_pad * s_pad;
    nb.Bc = bc.p + (int64_t)first * s_pad * s_pad;
    nb.BcT = bt.p + (int64_t)first * s_pad * s_pad;
    nb.PT = pt.p + (int64_t)first * zt * s_pad;
    nb.XS = dk ? xs.p + (int64_t)first * zt * dk : nullptr;
    nb.XN = dk ? xn.p + (int64_t)first * zt : nullptr;
    nb.dk = dk;
    nb.Pn = pn.p + (int64_t)first * s_pad * zt;
    nb.piv = piv.p + (int64_t)first * t_pad;
    nb.norm1 = norm1.p + first;
    nb.cond = cond.p + first;
    nb.info = int_info.p + first;
    nb.moves = moves.p + (int64_t)first * (2 * 64 + 1);
    nb.pm = pm.p + (int64_t)first * t_pad;
    nb.scratch = lu_scratch.p + (int64_t)first * 32 * 64;
    return nb;
  }
  void release_all() {
    coords.release(); xx.release(); rank_d.release(); skel_pos.release(); skel_off.release(); coeff_off.release();
    coeff.release(); leaf_node.release(); leaf_begin.release(); leaf_size.release(); leaf_info.release();
    int_node.release(); int_left.release(); int_right.release(); int_info.release(); piv.release(); moves.release();
    pm.release(); lu_scratch.release(); lu_sync.release(); dinv.release(); lut.release();
    leafA.release(); inv.release(); hbuf.release(); aug.release(); bc.release(); pn.release();
    norm1.release(); cond.release(); xy.release(); phl.release(); norm1_slab.release(); bt.release();
    pt.release(); xs.release(); xn.release();
    fb_aug.release(); fb_norm1.release(); fb_cond.release(); fb_piv.release(); fb_info.release();
    fb_moves.release(); fb_pm.release(); fb_node.release(); fb_begin.release(); fb_size.release();
    for (auto& w : ws) {
      w->release_all();
      if (w->done) cudaEventDestroy(w->done);
    }
    ws.clear();
    shard_ws = last_ws = nullptr;
  }
};

namespace ksr {

using ks::GemmArgs;
using ks::Operand;
using ks::OperandW;

inline GemmArgs mk(int M, int N, int K, int batch, Operand A, Operand B, OperandW C, double alpha, double beta) {
  GemmArgs g;
  g.M = M; g.N = N; g.K = K; g.batch = batch;
  g.A = A; g.B = B; g.C = C;
  g.alpha = alpha; g.beta = beta; g.tri = 0;
  g.E = Operand{nullptr, 0, 0, nullptr};
  g.Cin = Operand{nullptr, 0, 0, nullptr};
  g.addI = 0;
  return g;
}

// Launch bookkeeping on one stream: counts launches, and under KS_TRACE /
// KS_DEBUG_SYNC records an event after (or synchronizes on) every launch.
struct Launcher {
  ks_factor* f;
  cudaStream_t st;
  std::atomic<int64_t>* count;
  int check(const char* what);
  int gemm(const GemmArgs& g, bool ta, bool tb, const char* name = "gemm");
};

// B[r0:r0+w, c0:c0+ncols] := L^-1 B, L unit lower at (r0, r0) of each node's Aug.
int trsm_ul(Launcher& L, const ks::NodeBatch& nb, int r0, int w, int c0, int ncols);
// Recursive LU of columns [c0, c0+w) over rows [c0, T), pivots among rows < t_pad.
int rlu(Launcher& L, const ks::NodeBatch& nb, int c0, int w, int pw, int* pend, int ext = 0);

// create.cu
int create_impl(const ks_problem* p, int device, int64_t shard_root, ks_factor** out);
// factorize.cu
int fb_alloc(ks_factor* f);

struct PhaseTimer {
  bool on;
  cudaStream_t st;
  std::vector<cudaEvent_t> ev;
  PhaseTimer(bool on_, cudaStream_t s, int n) : on(on_), st(s) {
    if (!on) return;
    ev.resize(n);
    for (auto& e : ev) cudaEventCreate(&e);
  }
  void mark(int i) {
    if (on) cudaEventRecord(ev[i], st);
  }
  float between(int a, int b) {
    float ms = 0.f;
    if (on) cudaEventElapsedTime(&ms, ev[a], ev[b]);
    return ms;
  }
  ~PhaseTimer() {
    for (auto& e : ev) cudaEventDestroy(e);
  }
};

}  // namespace ksr
